"""Seeded plan corruptions reproducing the reference's bug taxonomy.

Same categories, site enumeration and mutation recipes as the reference
injector (pkg/src/planeq/faults.py:40-370), so a FaultSpec names the same
mutant in both implementations (tests compare mutants byte for byte):
missing_comm (rewire | dangle), wrong_primitive (all_reduce -> all_gather),
wrong_group (merge two disjoint sibling all_reduces), bad_partition (rotate a
chunk index), wrong_scaling (seed: scale x dp | avg: 1/dp after a replica
all_reduce), shuffled_microbatch (cross | cycle), dropped_microbatch (an
accumulator consumes one lane twice), bad_slice (shift one lineage range),
extra_op (scale a tensor by 2). Mutants round-trip through the serializer and
record plan.provenance["fault"].
"""

from __future__ import annotations

import random
from dataclasses import dataclass, field
from fractions import Fraction

from .errors import PlanEqError
from .graph import Graph, Node
from .plan import Plan, plan_from_dict, plan_to_dict

CATEGORIES = ("missing_comm", "wrong_primitive", "wrong_group", "bad_partition",
              "wrong_scaling", "shuffled_microbatch", "dropped_microbatch", "bad_slice")


@dataclass(frozen=True)
class FaultSpec:
    category: str
    site: str
    detail: dict = field(default_factory=dict)

    def to_dict(self) -> dict:
        return {"category": self.category, "site": self.site, "detail": self.detail}


def _origin(g: Graph, tid: str):
    return g.tensors[tid].meta.get("from")


def _find(g: Graph, nid: str) -> int:
    for i, n in enumerate(g.nodes):
        if n.id == nid:
            return i
    raise PlanEqError(f"fault site {nid!r} not found")


def _replace(g: Graph, nid: str, **kw):
    i = _find(g, nid)
    n = g.nodes[i]
    g.nodes[i] = Node(kw.get("id", n.id), kw.get("kind", n.kind), tuple(kw.get("inputs", n.inputs)),
                      tuple(kw.get("outputs", n.outputs)), kw.get("attrs", n.attrs), n.device, n.seq)


def _drop(g: Graph, nid: str):
    g.nodes = [n for n in g.nodes if n.id != nid]


def _rewire(g: Graph, old: str, new: str):
    for i, n in enumerate(g.nodes):
        if old in n.inputs:
            g.nodes[i] = Node(n.id, n.kind, tuple(new if t == old else t for t in n.inputs),
                              n.outputs, n.attrs, n.device, n.seq)
    g.outputs = [new if t == old else t for t in g.outputs]


def _rewire_lineage(plan: Plan, old: str, new: str):
    for entry in plan.lineage.values():
        entry.shards = tuple(type(s)(tensor=new, ranges=s.ranges) if s.tensor == old else s
                             for s in entry.shards)


def _same_lane_descendant(g: Graph, n: Node) -> str | None:
    """A tensor within 6 hops downstream of n on the same device and microbatch."""
    m = g.tensors[n.outputs[0]].microbatch
    want_shape = g.tensors[n.inputs[0]].shape
    cons = g.consumers_map()
    frontier = list(n.outputs)
    seen = set(frontier)
    for _hop in range(6):
        if not frontier:
            break
        nxt = []
        for tid in frontier:
            for cn in cons.get(tid, []):
                for out in cn.outputs:
                    if out in seen:
                        continue
                    seen.add(out)
                    t = g.tensors[out]
                    if t.device == n.device and t.microbatch == m and t.shape == want_shape:
                        return out
                    nxt.append(out)
        frontier = nxt
    return None


def list_sites(plan: Plan, category: str) -> list[FaultSpec]:
    g = plan.parallel
    if g is None:
        raise PlanEqError("plan has no parallel graph to corrupt")
    sites: list[FaultSpec] = []
    if category == "missing_comm":
        for n in g.nodes:
            if n.kind == "all_reduce":
                sites += [FaultSpec(category, n.id, {"variant": v}) for v in ("rewire", "dangle")]
    elif category == "wrong_primitive":
        sites = [FaultSpec(category, n.id, {"to": "all_gather"}) for n in g.nodes
                 if n.kind == "all_reduce"]
    elif category == "wrong_group":
        pairs: dict[tuple, list[Node]] = {}
        for n in g.nodes:
            if n.kind == "all_reduce":
                key = (_origin(g, n.outputs[0]), g.tensors[n.outputs[0]].microbatch, len(n.inputs))
                pairs.setdefault(key, []).append(n)
        for _key, nodes in sorted(pairs.items(), key=lambda kv: kv[1][0].id):
            found = next(((a, b) for i, a in enumerate(nodes) for b in nodes[i + 1:]
                          if set(a.attrs["group"]).isdisjoint(b.attrs["group"])), None)
            if found:
                sites.append(FaultSpec(category, found[0].id, {"merge_with": found[1].id}))
    elif category == "bad_partition":
        sites = [FaultSpec(category, n.id, {}) for n in g.nodes
                 if n.kind == "chunk" and int(n.attrs.get("parts", 1)) > 1]
    elif category == "wrong_scaling":
        for n in g.nodes:
            if n.kind == "scale" and n.attrs.get("norm") == "global_batch":
                sites.append(FaultSpec(category, n.id, {"variant": "seed"}))
            elif n.kind == "all_reduce" and n.id.startswith("dpar."):
                sites.append(FaultSpec(category, n.id, {"variant": "avg"}))
    elif category == "shuffled_microbatch":
        lanes: dict[tuple, list[Node]] = {}
        for n in g.nodes:
            if n.kind not in ("mul", "div", "matmul", "dropout", "silu_grad") or len(n.inputs) < 2:
                continue
            if g.tensors[n.outputs[0]].microbatch is None or \
                    g.tensors[n.inputs[1]].microbatch is None:
                continue
            lanes.setdefault((n.kind, n.device, _origin(g, n.outputs[0])), []).append(n)
        for _key, nodes in sorted(lanes.items(), key=lambda kv: kv[1][0].id):
            if len(nodes) >= 2:
                sites.append(FaultSpec(category, nodes[0].id, {"variant": "cross", "peer": nodes[1].id}))
        for n in g.nodes:
            if not n.outputs or not n.inputs or g.tensors[n.outputs[0]].microbatch is None:
                continue
            desc = _same_lane_descendant(g, n)
            if desc is not None:
                sites.append(FaultSpec(category, n.id, {"variant": "cycle", "tensor": desc}))
                break
    elif category == "dropped_microbatch":
        sites = [FaultSpec(category, n.id, {}) for n in g.nodes
                 if n.kind == "add" and n.id.startswith("mb.") and n.inputs[0] != n.inputs[1]]
    elif category == "bad_slice":
        for tid, entry in plan.lineage.items():
            hit = next(((i, a) for i, s in enumerate(entry.shards)
                        for a, (lo, _hi) in enumerate(s.ranges) if lo > 0), None)
            if hit is not None:
                sites.append(FaultSpec(category, tid, {"shard": hit[0], "axis": hit[1]}))
    elif category == "extra_op":
        cons = g.consumers_map()
        sites = [FaultSpec(category, tid, {}) for tid, t in g.tensors.items()
                 if cons.get(tid) and t.dtype == "real" and not t.meta.get("mask")]
    # -- extensions for the Llama/DeepSeek bug-injected configs (not in the reference)
    elif category == "wrong_allreduce_scaling":
        sites = [FaultSpec(category, n.id, {"factor": "1/tp"}) for n in g.nodes
                 if n.kind in ("all_reduce", "reduce_scatter") and
                 (n.id.startswith("ar.") or n.id.startswith("rs.") or n.id.startswith("tpar."))]
    elif category == "misordered_concat":
        sites = [FaultSpec(category, n.id, {"swap": [0, 1]}) for n in g.nodes
                 if n.kind in ("all_gather", "all_to_all") and len(n.inputs) >= 2]
    elif category == "dropped_partial_sum":
        sites = [FaultSpec(category, n.id, {"slot": len(n.inputs) - 1}) for n in g.nodes
                 if n.kind in ("all_reduce", "reduce_scatter") and len(n.inputs) >= 2]
    else:
        raise PlanEqError(f"unknown fault category {category!r}")
    return sites


def _insert_scale(g: Graph, tid: str, factor: Fraction, tag: str):
    """Route tid's value through scale(factor) so every reader sees the corruption."""
    t = g.tensors[tid]
    new = f"{tid}.{tag}"
    g.add_tensor(type(t)(id=new, shape=t.shape, role="intermediate", dtype=t.dtype,
                         device=t.device, microbatch=t.microbatch, meta=dict(t.meta)))
    seq = max((n.seq for n in g.nodes if n.device == t.device), default=0) + 1
    prod = next((n for n in g.nodes if tid in n.outputs), None)
    if prod is not None:
        _replace(g, prod.id, outputs=[new if x == tid else x for x in prod.outputs])
        src, dst = new, tid
    else:
        _rewire(g, tid, new)
        src, dst = tid, new
    g.add_node(Node(id=f"{tag}.{tid}", kind="scale", inputs=(src,), outputs=(dst,),
                    attrs={"factor": factor}, device=t.device, seq=seq))


def inject(plan: Plan, spec: FaultSpec) -> Plan:
    mutant = plan_from_dict(plan_to_dict(plan))
    g = mutant.parallel
    c = spec.category
    if c == "missing_comm":
        n = g.nodes[_find(g, spec.site)]
        _drop(g, n.id)
        if spec.detail.get("variant") == "rewire":
            for src, dst in zip(n.inputs, n.outputs):
                _rewire(g, dst, src)
                _rewire_lineage(mutant, dst, src)
                del g.tensors[dst]
    elif c == "wrong_primitive":
        n = g.nodes[_find(g, spec.site)]
        attrs = {k: v for k, v in n.attrs.items() if k != "op"}
        attrs["axis"] = 0
        _replace(g, n.id, kind="all_gather", attrs=attrs)
    elif c == "wrong_group":
        a = g.nodes[_find(g, spec.site)]
        b = g.nodes[_find(g, spec.detail["merge_with"])]
        attrs = dict(a.attrs)
        attrs["group"] = list(a.attrs["group"]) + list(b.attrs["group"])
        _replace(g, a.id, inputs=list(a.inputs) + list(b.inputs),
                 outputs=list(a.outputs) + list(b.outputs), attrs=attrs)
        _drop(g, b.id)
    elif c == "bad_partition":
        n = g.nodes[_find(g, spec.site)]
        attrs = dict(n.attrs)
        attrs["index"] = (int(attrs["index"]) + 1) % int(attrs["parts"])
        _replace(g, n.id, attrs=attrs)
    elif c == "wrong_scaling":
        n = g.nodes[_find(g, spec.site)]
        dp = max(int(mutant.config.get("cfg", {}).get("dp", 1)), 2)
        if spec.detail.get("variant") == "seed":
            attrs = dict(n.attrs)
            attrs["factor"] = Fraction(attrs["factor"]) * dp
            _replace(g, n.id, attrs=attrs)
        else:
            _insert_scale(g, n.outputs[0], Fraction(1, dp), "avg")
    elif c == "shuffled_microbatch":
        n = g.nodes[_find(g, spec.site)]
        if spec.detail.get("variant") == "cross":
            p = g.nodes[_find(g, spec.detail["peer"])]
            ni, pi = list(n.inputs), list(p.inputs)
            ni[1], pi[1] = pi[1], ni[1]
            _replace(g, n.id, inputs=ni)
            _replace(g, p.id, inputs=pi)
        else:
            ni = list(n.inputs)
            ni[0] = spec.detail["tensor"]
            _replace(g, n.id, inputs=ni)
    elif c == "dropped_microbatch":
        n = g.nodes[_find(g, spec.site)]
        _replace(g, n.id, inputs=(n.inputs[0], n.inputs[0]))
    elif c == "bad_slice":
        entry = mutant.lineage[spec.site]
        i, a = int(spec.detail["shard"]), int(spec.detail["axis"])
        s = entry.shards[i]
        lo, hi = s.ranges[a]
        ranges = s.ranges[:a] + ((lo - 1, hi - 1),) + s.ranges[a + 1:]
        entry.shards = entry.shards[:i] + (type(s)(tensor=s.tensor, ranges=ranges),) + \
            entry.shards[i + 1:]
    elif c == "extra_op":
        _insert_scale(g, spec.site, Fraction(2), "xop")
    elif c == "wrong_allreduce_scaling":
        # average instead of sum over the tensor group: every output scaled by 1/k
        n = g.nodes[_find(g, spec.site)]
        for out in n.outputs:
            _insert_scale(g, out, Fraction(1, len(n.inputs)), "avg")
    elif c == "misordered_concat":
        n = g.nodes[_find(g, spec.site)]
        i, j = spec.detail.get("swap", [0, 1])
        ins = list(n.inputs)
        ins[i], ins[j] = ins[j], ins[i]
        _replace(g, n.id, inputs=ins)
    elif c == "dropped_partial_sum":
        # one partial never reaches the collective: it contributes zero
        n = g.nodes[_find(g, spec.site)]
        _insert_scale(g, n.inputs[int(spec.detail["slot"])], Fraction(0), "drop")
    else:
        raise PlanEqError(f"unknown fault category {c!r}")
    mutant.provenance = dict(mutant.provenance)
    mutant.provenance["fault"] = spec.to_dict()
    return mutant


def random_structural_fault(plan: Plan, rng: random.Random) -> Plan:
    """One seeded, loadable, value-level corruption (soundness corpus)."""
    order = ["missing_comm", "wrong_group", "bad_partition", "wrong_scaling",
             "dropped_microbatch", "shuffled_microbatch", "bad_slice", "extra_op"]
    rng.shuffle(order)
    for category in order:
        sites = list_sites(plan, category)
        if category == "missing_comm":
            sites = [s for s in sites if s.detail.get("variant") == "rewire"]
        if category == "shuffled_microbatch":
            sites = [s for s in sites if s.detail.get("variant") == "cross"]
        if sites:
            return inject(plan, rng.choice(sites))
    raise PlanEqError("no fault site available in this plan")

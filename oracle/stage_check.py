"""TEST INFRASTRUCTURE ONLY. Per-stage discharge by witness evaluation on the CPU.

Restates, over F_p witness batches, what the reference does in
pkg/src/planeq/stages.py:267-389 (run_stage):
  * interface (stages.py:144-176): real logical inputs -> variables
    "v.<tid>.<i>"; integer inputs -> position enumeration; full lineage
    entries alias logical element values; partial groups get variables
    "ps.<shard>.<i>" for all members but the last, the last being the logical
    value minus the others;
  * both sub-DFGs evaluated node by node (oracle/evaluator.py);
  * obligations in the reference's order (stages.py:316-340);
  * a witness is valid iff every guarded operand is nonzero; the stage is
    refuted iff some valid witness breaks an obligation.

Stage construction (build_stages) is host code shared with the product; the
discharge below shares nothing with the product compiler or kernel.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import m31
from .evaluator import Ctx, eval_node


@dataclass
class OracleStageResult:
    target: str
    status: str                   # proven | refuted | unknown | par_div0 | log_div0
    obligations: int = 0
    valid: int = 0
    bad: int = 0
    first_bad: tuple[int, int] | None = None   # (witness, obligation)
    reason: str | None = None
    lhs: int | None = None
    rhs: int | None = None
    bad_mask: np.ndarray | None = field(default=None, repr=False)


def _iter_box(ranges):
    return np.ndindex(*[hi - lo for lo, hi in ranges])


def _slice(x: np.ndarray, ranges) -> np.ndarray:
    return x[tuple(slice(lo, hi) for lo, hi in ranges)]


def check_stage(plan, stage, owner: dict[str, str], seed: int, witnesses: np.ndarray) -> OracleStageResult:
    """Evaluate one stage on the given witness indices."""
    logical, parallel, lineage = plan.logical, plan.parallel, plan.lineage
    W = len(witnesses)
    ctx = Ctx(seed, W)
    boxes: dict[str, np.ndarray] = {}

    def box_of(tid):
        if tid in boxes:
            return boxes[tid]
        t = logical.tensors[tid]
        if t.dtype == "int":
            if t.meta.get("enum") != "position":
                raise ValueError(f"integer checkpoint {tid!r} has no enumerated values")
            v = np.arange(t.nelems(), dtype=np.int64).reshape(t.shape)
        else:
            v = m31.var_values(seed, f"v.{tid}", t.nelems(), witnesses).reshape(tuple(t.shape) + (W,))
        boxes[tid] = v
        return v

    env_l: dict[str, np.ndarray] = {}
    produced_l = {o for n in stage.logical_nodes for o in n.outputs}
    for tid in stage.l_inputs:
        if tid not in produced_l:
            env_l[tid] = box_of(tid)
    try:
        for n in stage.logical_nodes:
            outs = eval_node(n, [env_l[t] for t in n.inputs], [logical.shape(t) for t in n.outputs], ctx)
            for t, v in zip(n.outputs, outs):
                env_l[t] = v
    except ZeroDivisionError as e:
        return OracleStageResult(stage.target, "log_div0", reason=str(e))

    env_p: dict[str, np.ndarray] = {}
    produced_p = {o for n in stage.parallel_nodes for o in n.outputs}
    done = set()
    for st in stage.p_inputs:
        if st in produced_p:
            continue
        etid = owner[st]
        if etid in done:
            continue
        done.add(etid)
        entry = lineage[etid]
        box = box_of(etid)
        if entry.mode == "full":
            for s in entry.shards:
                env_p[s.tensor] = np.ascontiguousarray(_slice(box, s.ranges))
            continue
        groups: dict = {}
        for s in entry.shards:
            groups.setdefault(s.ranges, []).append(s)
        for ranges in sorted(groups):
            members = sorted(groups[ranges], key=lambda s: s.tensor)
            ext = tuple(hi - lo for lo, hi in ranges)
            n = int(np.prod(ext))
            rest = None
            for s in members[:-1]:
                v = m31.var_values(seed, f"ps.{s.tensor}", n, witnesses).reshape(ext + (W,))
                env_p[s.tensor] = v
                rest = v if rest is None else m31.add(rest, v)
            sl = np.ascontiguousarray(_slice(box, ranges))
            env_p[members[-1].tensor] = sl if rest is None else m31.sub(sl, rest)
    try:
        for n in stage.parallel_nodes:
            outs = eval_node(n, [env_p[t] for t in n.inputs], [parallel.shape(t) for t in n.outputs], ctx)
            for t, v in zip(n.outputs, outs):
                env_p[t] = v
    except ZeroDivisionError as e:
        return OracleStageResult(stage.target, "par_div0", reason=str(e))

    # obligations
    entry = lineage[stage.target]
    tgt = env_l[stage.target]
    lhs_list, rhs_list = [], []
    if entry.mode == "full":
        for s in entry.shards:
            lhs_list.append(_slice(tgt, s.ranges).reshape(-1, *([W] if tgt.dtype != np.int64 else [])))
            rhs_list.append(env_p[s.tensor].reshape(lhs_list[-1].shape))
    else:
        groups = {}
        for s in entry.shards:
            groups.setdefault(s.ranges, []).append(s)
        for ranges in sorted(groups):
            members = sorted(groups[ranges], key=lambda s: s.tensor)
            acc = None
            for s in members:
                v = env_p[s.tensor]
                acc = v if acc is None else m31.add(acc, v)
            lhs_list.append(_slice(tgt, ranges).reshape(-1, W))
            rhs_list.append(acc.reshape(-1, W))

    def as_field(x):
        if x.dtype == np.int64:
            return np.repeat((x % m31.PI).astype(np.uint64)[:, None], W, axis=1)
        return x

    n_obl = sum(x.shape[0] for x in lhs_list)
    if n_obl == 0:
        return OracleStageResult(stage.target, "proven", 0, valid=int(ctx.valid.sum()))
    lhs = np.concatenate([as_field(x) for x in lhs_list], axis=0)
    rhs = np.concatenate([as_field(x) for x in rhs_list], axis=0)
    bad = (lhs != rhs) & ctx.valid[None, :]
    bad_w = bad.any(axis=0)
    res = OracleStageResult(stage.target, "proven", n_obl, valid=int(ctx.valid.sum()),
                            bad=int(bad_w.sum()), bad_mask=bad)
    if bad_w.any():
        w = int(np.argmax(bad_w))
        o = int(np.argmax(bad[:, w]))
        res.status = "refuted"
        res.first_bad = (int(witnesses[w]), o)
        res.lhs, res.rhs = int(lhs[o, w]), int(rhs[o, w])
    elif res.valid == 0:
        res.status = "unknown"
    return res


def check_plan(plan, seed: int = 0, n_witness: int = 64, stages=None):
    """Oracle verdicts for every stage of a plan (no cancellation)."""
    from paper_2506_15961_b200.stages import build_stages, entry_order, shard_owner
    if stages is None:
        stages, _ = build_stages(plan)
    owner = shard_owner(plan, entry_order(plan))
    wit = np.arange(n_witness, dtype=np.uint64)
    return [check_stage(plan, st, owner, seed, wit) for st in stages]

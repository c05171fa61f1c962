"""Stages: construction (host) and discharge (sm_100a witness engine).

Stage construction is the reference's lineage-driven partition, kept
identical so both implementations check the same obligations
(pkg/src/planeq/stages.py:79-138): every produced checkpoint tensor is one
stage; its logical slice is the backward slice stopped at other checkpoints,
its parallel slice the backward slice from its shards stopped at shards of
strictly earlier checkpoints.

Discharge replaces the reference's symbolic execution + SMT query
(stages.py:267-389) with compiled witness evaluation: `lower_stage` turns a
stage into the engine's flat tensor-op program, interface construction
included -- full entries alias the logical element values, partial groups get
fresh variables for all members but the last, which is defined as the logical
value minus the others, integer checkpoints are pinned to the position
enumeration (the same assumption baking as stages.py:144-176) -- and
`discharge_stages` compiles all stages into one device image, evaluates every
obligation on a batch of random F_p witnesses in one launch, and turns the
per-stage outcome into the reference's StageResult shape.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field, fields
from fractions import Fraction
from typing import Any

import numpy as np

from . import field as F
from .errors import GraphError, ShapeError, UnsupportedOperator
from .graph import (Graph, LineageEntry, Node, backward_slice, range_extents, topo_sort,
                    unflatten, volume)
from .opshape import einsum_parse, reduce_axes
from .plan import Plan

IR_MAGIC = 0x50515701

# tensor-op opcodes (enum pqw_top in include/planeq_witness.h)
T_VARS, T_INTS, T_SLICE, T_RESID, T_CHECK, T_CHECKSUM, T_SIDE = 1, 2, 3, 4, 5, 6, 7
_KIND_CODES = ("add", "sub", "mul", "div", "dropout", "silu_grad", "identity", "scale", "shift",
               "pow", "rsqrt", "silu", "move", "softmax", "create_mask", "apply_mask", "view",
               "transpose", "expand", "sum", "mean", "matmul", "einsum", "full", "chunk",
               "embedding", "embedding_grad", "gnorm_sq", "all_reduce", "all_gather",
               "reduce_scatter", "all_to_all")
OPCODE = {k: 16 + i for i, k in enumerate(_KIND_CODES)}

VAR_STEP = 0xD1B54A32D192ED03


@dataclass
class Stage:
    target: str
    logical_nodes: list[Node]
    parallel_nodes: list[Node]
    l_inputs: list[str]
    p_inputs: list[str]
    assumed: list[str]
    owned_logical: list[str] = field(default_factory=list)
    owned_parallel: list[str] = field(default_factory=list)


@dataclass
class StageResult:
    target: str
    status: str  # proven | refuted | unknown
    obligations: int
    fastpath: int
    residual: int
    wall_s: float
    detail: dict[str, Any] | None = None
    note: str | None = None
    witnesses: int = 0
    valid_witnesses: int = 0
    failing_witnesses: int = 0
    degree_bound: int = 0
    false_equiv_log2: float | None = None

    def as_dict(self) -> dict[str, Any]:
        """dataclasses.asdict without its recursive deep copy (the detail dict
        is built fresh for each result): the report's per-stage record."""
        return {f: getattr(self, f) for f in _RESULT_FIELDS}


_RESULT_FIELDS = tuple(f.name for f in fields(StageResult))


def entry_order(plan: Plan, order: list[Node] | None = None) -> list[str]:
    """Checkpoints by producing-node position in logical topo order, inputs first."""
    pos = {n.id: i for i, n in enumerate(order if order is not None else topo_sort(plan.logical))}
    prod = plan.logical.producer_map()

    def key(tid: str) -> tuple[int, str]:
        n = prod.get(tid)
        return (pos[n.id] if n is not None else -1, tid)

    return sorted(plan.lineage, key=key)


def build_stages(plan: Plan) -> tuple[list[Stage], dict[str, list[str]]]:
    """One stage per produced checkpoint plus coverage bookkeeping (stages.py:91-138)."""
    logical, parallel, lineage = plan.logical, plan.parallel, plan.lineage
    lprod = logical.producer_map()
    pprod = parallel.producer_map()
    order = entry_order(plan)
    rank = {tid: i for i, tid in enumerate(order)}
    shards_of = {tid: [s.tensor for s in e.shards] for tid, e in lineage.items()}
    # earliest checkpoint claiming a shard tensor
    owner: dict[str, str] = {}
    for t in reversed(order):
        for st in shards_of[t]:
            owner[st] = t
    stages: list[Stage] = []
    claimed_l: set[str] = set()
    claimed_p: set[str] = set()
    all_ckpt = set(lineage)
    earlier_shards: set[str] = set()
    lmade, pmade = set(lprod), set(pprod)
    lpos = {n.id: i for i, n in enumerate(logical.nodes)}
    ppos = {n.id: i for i, n in enumerate(parallel.nodes)}
    for tid in order:
        if tid in lprod:
            lnodes, lbound = backward_slice(logical, [tid], all_ckpt - {tid}, lprod, lpos)
            lnodes = topo_sort(logical, lnodes, lmade)
            for b in sorted(lbound):
                if b not in lineage:
                    raise GraphError(f"stage {tid}: logical input {b!r} has no checkpoint entry")
            roots = [s.tensor for s in lineage[tid].shards]
            pnodes, pbound = backward_slice(parallel, roots, earlier_shards, pprod, ppos)
            pnodes = topo_sort(parallel, pnodes, pmade)
            for b in sorted(pbound):
                if b not in earlier_shards:
                    raise GraphError(f"stage {tid}: parallel input {b!r} is not a checkpoint shard")
            assumed = sorted(set(lbound) | {owner[b] for b in pbound}, key=rank.get)
            owned_l = sorted(n.id for n in lnodes if n.id not in claimed_l)
            claimed_l.update(owned_l)
            owned_p = sorted(n.id for n in pnodes if n.id not in claimed_p)
            claimed_p.update(owned_p)
            stages.append(Stage(tid, lnodes, pnodes, sorted(lbound), sorted(pbound), assumed,
                                owned_l, owned_p))
        earlier_shards.update(shards_of[tid])
    uncovered = {
        "logical": sorted(n.id for n in logical.nodes if n.id not in claimed_l),
        "parallel": sorted(n.id for n in parallel.nodes if n.id not in claimed_p),
    }
    return stages, uncovered


# -- lowering ------------------------------------------------------------------


def name_key(prefix: str) -> int:
    return F.fnv1a64("var:" + prefix)


def tensor_var_keys(seed: int, prefix: str, n: int) -> np.ndarray:
    """Keys of variables prefix.0 .. prefix.(n-1), vectorized (field.py convention)."""
    base = (seed ^ name_key(prefix)) & F.MASK64
    i = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(base) + i * np.uint64(VAR_STEP)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


@dataclass
class ObligationBlock:
    """A run of obligations: elements of `ranges` of the target, compared against shards."""
    first: int
    count: int
    label: str
    ranges: tuple[tuple[int, int], ...]


@dataclass
class LoweredStage:
    target: str
    ir: np.ndarray
    consts: np.ndarray
    var_keys: np.ndarray
    var_names: list[tuple[str, int]]   # (prefix, count) runs, in var-index order
    blocks: list[ObligationBlock]
    n_obligations: int
    early: StageResult | None = None   # decided during lowering (no program)

    def var_name(self, idx: int) -> str:
        for prefix, n in self.var_names:
            if idx < n:
                return f"{prefix}.{idx}"
            idx -= n
        raise IndexError(idx)

    def locate(self, obl: int) -> tuple[str, tuple[int, ...]]:
        for b in self.blocks:
            if b.first <= obl < b.first + b.count:
                ext = range_extents(b.ranges)
                loc = unflatten(obl - b.first, ext)
                return b.label, tuple(lo + i for (lo, _), i in zip(b.ranges, loc))
        raise IndexError(obl)


class _Lowerer:
    def __init__(self, seed: int):
        self.seed = seed
        self.tid: dict[str, int] = {}
        self.shapes: list[tuple[int, ...]] = []
        self.ops: list[int] = []
        self.n_ops = 0
        self.consts: list[tuple[int, int, int]] = []
        self.const_idx: dict[tuple, int] = {}
        self.var_keys: list[np.ndarray] = []
        self.var_names: list[tuple[str, int]] = []
        self.n_vars = 0

    def tensor(self, key: str, shape) -> int:
        idx = self.tid.get(key)
        if idx is None:
            idx = len(self.shapes)
            self.tid[key] = idx
            self.shapes.append(tuple(int(d) for d in shape))
        return idx

    def temp(self, shape) -> int:
        idx = len(self.shapes)
        self.shapes.append(tuple(int(d) for d in shape))
        return idx

    def const(self, q) -> int:
        q = Fraction(q)
        key = (q.numerator, q.denominator)
        got = self.const_idx.get(key)
        if got is None:
            got = len(self.consts)
            self.consts.append(F.const_triple(q))
            self.const_idx[key] = got
        return got

    def emit(self, op: int, ins, outs, attrs=()):
        self.ops.extend((op, len(ins), len(outs), len(attrs)))
        self.ops.extend(ins)
        self.ops.extend(outs)
        self.ops.extend(int(a) for a in attrs)
        self.n_ops += 1

    def vars_for(self, prefix: str, shape) -> int:
        n = volume(shape)
        out = self.temp(shape)
        self.emit(T_VARS, [], [out], [self.n_vars])
        self.var_keys.append(tensor_var_keys(self.seed, prefix, n))
        self.var_names.append((prefix, n))
        self.n_vars += n
        return out

    def ints_for(self, values: list[int], shape) -> int:
        out = self.temp(shape)
        base = len(self.consts)
        for v in values:
            self.consts.append(F.const_triple(v))
        self.emit(T_INTS, [], [out], [base])
        return out

    def program(self, n_obl: int) -> np.ndarray:
        head = [IR_MAGIC, len(self.shapes), self.n_ops, n_obl]
        for s in self.shapes:
            head.append(len(s))
            head.extend(s)
        return np.array(head + self.ops, dtype=np.int32)


def _node_attrs(low: _Lowerer, node: Node, in_shapes: list[tuple]) -> list[int]:
    k, a = node.kind, node.attrs
    if k in ("scale",):
        return [low.const(a["factor"])]
    if k == "shift":
        return [low.const(a["addend"])]
    if k == "full":
        return [low.const(a["value"])]
    if k == "pow":
        return [int(a["exponent"])]
    if k == "div":
        return [1 if a.get("den_positive") else 0]
    if k == "transpose":
        return [int(p) for p in a["perm"]]
    if k in ("sum", "mean"):
        return [1 if a.get("keepdims") else 0] + list(reduce_axes(a, len(in_shapes[0])))
    if k == "einsum":
        subs, rhs = einsum_parse(a["spec"], len(in_shapes), node.id)
        out = [len(subs)]
        for s in subs:
            out.append(len(s))
            out.extend(ord(c) for c in s)
        out.append(len(rhs))
        out.extend(ord(c) for c in rhs)
        return out
    if k == "chunk":
        return [int(a["axis"]) % len(in_shapes[0]), int(a["parts"]), int(a["index"])]
    if k in ("all_gather", "reduce_scatter"):
        return [int(a["axis"]) % len(in_shapes[0])]
    if k == "all_to_all":
        r = len(in_shapes[0])
        return [int(a["split_axis"]) % r, int(a["concat_axis"]) % r]
    return []


def lower_stage(plan: Plan, stage: Stage, owner: dict[str, str], seed: int) -> LoweredStage:
    """Stage -> engine program (interface, both sub-DFGs, obligations)."""
    logical, parallel, lineage = plan.logical, plan.parallel, plan.lineage
    low = _Lowerer(seed)
    boxes: dict[str, int] = {}

    def box_of(tid: str) -> int:
        got = boxes.get(tid)
        if got is not None:
            return got
        t = logical.tensors[tid]
        if t.dtype == "int":
            if t.meta.get("enum") != "position":
                raise UnsupportedOperator(f"integer checkpoint {tid!r} has no enumerated values")
            idx = low.ints_for(list(range(t.nelems())), t.shape)
        else:
            idx = low.vars_for(f"v.{tid}", t.shape)
        boxes[tid] = idx
        return idx

    produced_l = {o for n in stage.logical_nodes for o in n.outputs}
    for tid in stage.l_inputs:
        if tid not in produced_l:
            low.tid["L:" + tid] = box_of(tid)

    def run_nodes(nodes: list[Node], graph: Graph, pre: str, side: int):
        low.emit(T_SIDE, [], [], [side])
        for n in nodes:
            if n.kind not in OPCODE:
                from .errors import UnknownOperator
                raise UnknownOperator(n.kind)
            ins = []
            in_shapes = []
            for t in n.inputs:
                key = pre + t
                if key not in low.tid:
                    raise GraphError(f"stage {stage.target}: unbound input {t!r} of {n.id}")
                ins.append(low.tid[key])
                in_shapes.append(low.shapes[low.tid[key]])
            outs = [low.tensor(pre + t, graph.shape(t)) for t in n.outputs]
            low.emit(OPCODE[n.kind], ins, outs, _node_attrs(low, n, in_shapes))

    run_nodes(stage.logical_nodes, logical, "L:", 0)

    produced_p = {o for n in stage.parallel_nodes for o in n.outputs}
    done: set[str] = set()
    for st in stage.p_inputs:
        if st in produced_p:
            continue
        etid = owner[st]
        if etid in done:
            continue
        done.add(etid)
        entry = lineage[etid]
        tensor = logical.tensors[etid]
        box = box_of(etid)
        bshape = low.shapes[box]
        if entry.mode == "full":
            for s in entry.shards:
                out = low.tensor("P:" + s.tensor, range_extents(s.ranges))
                low.emit(T_SLICE, [box], [out], [lo for lo, _ in s.ranges])
            continue
        if tensor.dtype == "int":
            raise UnsupportedOperator(f"partial checkpoint over integer tensor {tensor.id!r}")
        for ranges, members in sorted(entry.groups().items()):
            members = sorted(members, key=lambda s: s.tensor)
            ext = range_extents(ranges)
            frees = []
            for s in members[:-1]:
                v = low.vars_for(f"ps.{s.tensor}", ext)
                low.tid["P:" + s.tensor] = v
                frees.append(v)
            sl = low.temp(ext)
            low.emit(T_SLICE, [box], [sl], [lo for lo, _ in ranges])
            if frees:
                last = low.tensor("P:" + members[-1].tensor, ext)
                low.emit(T_RESID, [sl] + frees, [last])
            else:
                low.tid["P:" + members[-1].tensor] = sl
        del bshape

    run_nodes(stage.parallel_nodes, parallel, "P:", 1)

    # obligations of the target (stages.py:316-340 order)
    entry = lineage[stage.target]
    tgt = low.tid["L:" + stage.target]
    blocks: list[ObligationBlock] = []
    n_obl = 0

    def shard_tensor(name: str) -> int:
        idx = low.tid.get("P:" + name)
        if idx is None:
            raise GraphError(f"stage {stage.target}: shard {name!r} was never computed")
        return idx

    if entry.mode == "full":
        for s in entry.shards:
            rhs = shard_tensor(s.tensor)
            ext = range_extents(s.ranges)
            lhs = low.temp(ext)
            low.emit(T_SLICE, [tgt], [lhs], [lo for lo, _ in s.ranges])
            cnt = volume(ext)
            low.emit(T_CHECK, [lhs, rhs], [], [n_obl])
            blocks.append(ObligationBlock(n_obl, cnt, s.tensor, s.ranges))
            n_obl += cnt
    else:
        for ranges, members in sorted(entry.groups().items()):
            members = sorted(members, key=lambda s: s.tensor)
            rhs = [shard_tensor(s.tensor) for s in members]
            ext = range_extents(ranges)
            lhs = low.temp(ext)
            low.emit(T_SLICE, [tgt], [lhs], [lo for lo, _ in ranges])
            cnt = volume(ext)
            low.emit(T_CHECKSUM, [lhs] + rhs, [], [n_obl])
            blocks.append(ObligationBlock(n_obl, cnt, "+".join(s.tensor for s in members), ranges))
            n_obl += cnt

    keys = np.concatenate(low.var_keys) if low.var_keys else np.zeros(0, dtype=np.uint64)
    consts = np.array(low.consts, dtype=np.int64).reshape(-1, 3) if low.consts else \
        np.zeros((0, 3), dtype=np.int64)
    return LoweredStage(stage.target, low.program(n_obl), consts, keys, low.var_names, blocks,
                        n_obl)


def shard_owner(plan: Plan, order: list[str] | None = None) -> dict[str, str]:
    order = order if order is not None else entry_order(plan)
    owner: dict[str, str] = {}
    for etid in reversed(order):
        for s in plan.lineage[etid].shards:
            owner[s.tensor] = etid
    return owner


def bound_log2(degree: int, valid: int) -> float | None:
    """log2 of the false-equivalence bound (deg/p)^valid, None if vacuous."""
    import math
    if valid <= 0 or degree <= 0:
        return None if valid <= 0 else float("-inf")
    per = math.log2(degree) - math.log2(F.P)
    if per >= 0:
        return None
    return per * valid

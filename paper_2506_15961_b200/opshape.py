"""Operator registry: shape rules of every supported operator kind.

The set of kinds and each kind's declared-shape rule follow the reference
registry (pkg/src/planeq/ops.py:100-909, REGISTRY at ops.py:902). Value
semantics are not here: they live in the witness compiler
(csrc/compiler.cpp, Compiler::run_op), which evaluates each kind on scalar
value ids. `validate_concrete` re-derives every node's output shapes, like the
reference's shapes.py:35-45.
"""

from __future__ import annotations

from .errors import ShapeError, UnknownOperator
from .graph import Graph, Node, Shape, topo_sort, volume

ELEMENTWISE2 = ("add", "sub", "mul", "div", "dropout", "silu_grad")
UNARY = ("identity", "scale", "shift", "pow", "rsqrt", "silu", "move")
COMM = ("all_reduce", "all_gather", "reduce_scatter", "all_to_all")
KINDS = frozenset(ELEMENTWISE2 + UNARY + COMM + (
    "softmax", "create_mask", "apply_mask", "view", "transpose", "expand", "sum", "mean",
    "matmul", "einsum", "full", "chunk", "embedding", "embedding_grad", "gnorm_sq"))
DIFF_INPUTS = {"add": (0, 1), "sub": (0, 1), "mul": (0, 1), "div": (0, 1), "dropout": (0,),
               "identity": (0,), "scale": (0,), "shift": (0,), "pow": (0,), "rsqrt": (0,),
               "silu": (0,), "softmax": (0,), "apply_mask": (0,), "view": (0,),
               "transpose": (0,), "expand": (0,), "sum": (0,), "mean": (0,), "matmul": (0, 1),
               "chunk": (0,), "embedding": (0,)}
IS_COMM = frozenset(COMM + ("move",))


def _s(shape) -> str:
    return "[" + ",".join(str(d) for d in shape) + "]"


def reduce_axes(attrs: dict, rank: int) -> tuple[int, ...]:
    axes = attrs.get("axes")
    if axes is None:
        return tuple(range(rank))
    return tuple(sorted(int(a) % rank for a in axes))


def einsum_parse(spec: str, n_in: int, node_id: str = "?") -> tuple[list[str], str]:
    spec = spec.replace(" ", "")
    lhs, rhs = spec.split("->")
    subs = lhs.split(",")
    if len(subs) != n_in:
        raise ShapeError(f"einsum {node_id}: spec arity mismatch")
    return subs, rhs


def infer_shapes(node: Node, ins: list[Shape]) -> list[Shape]:
    k = node.kind
    a = node.attrs

    def want(cond: bool, msg: str):
        if not cond:
            raise ShapeError(f"{k} {node.id}: {msg}")

    if k not in KINDS:
        raise UnknownOperator(k)
    if k in ELEMENTWISE2:
        want(len(ins) == 2, "expects 2 inputs")
        want(ins[1] == ins[0], f"operand shapes differ: {_s(ins[0])} vs {_s(ins[1])}")
        return [ins[0]]
    if k in UNARY:
        want(len(ins) == 1, "expects 1 input")
        if k == "pow":
            want(int(a.get("exponent", 0)) >= 1, "exponent must be >= 1")
        return [ins[0]]
    if k == "softmax":
        want(len(ins) == 1, "expects 1 input")
        ax = int(a.get("axis", -1))
        want(ax in (-1, len(ins[0]) - 1), "softmax supported on the last axis only")
        want(ins[0][-1] >= 2, "softmax axis must have extent >= 2")
        return [ins[0]]
    if k == "create_mask":
        want(len(ins) == 0, "expects no inputs")
        s = int(a["size"])
        want(s >= 2, "mask size must be >= 2")
        return [(s, s)]
    if k == "apply_mask":
        want(len(ins) == 2, "expects (x, mask)")
        x, m = ins
        want(len(m) == 2 and m[0] == m[1], "mask must be square")
        want(len(x) >= 2 and tuple(x[-2:]) == tuple(m),
             f"mask {_s(m)} must match trailing dims of {_s(x)}")
        return [x]
    if k == "view":
        want(len(ins) == 1, "expects 1 input")
        tgt = tuple(int(d) for d in a["shape"])
        want(volume(ins[0]) == volume(tgt), f"element count changes: {_s(ins[0])} -> {_s(tgt)}")
        return [tgt]
    if k == "transpose":
        perm = tuple(int(p) for p in a["perm"])
        want(len(ins) == 1 and sorted(perm) == list(range(len(ins[0]))),
             "perm must permute input axes")
        return [tuple(ins[0][p] for p in perm)]
    if k == "expand":
        tgt = tuple(int(d) for d in a["shape"])
        src = ins[0]
        want(len(tgt) == len(src), "expand cannot change rank")
        for s, t in zip(src, tgt):
            want(s == t or s == 1, f"cannot expand {_s(src)} to {_s(tgt)}")
        return [tgt]
    if k in ("sum", "mean"):
        want(len(ins) == 1, "expects 1 input")
        axes = reduce_axes(a, len(ins[0]))
        keep = bool(a.get("keepdims"))
        out = [1 if ax in axes else d for ax, d in enumerate(ins[0]) if keep or ax not in axes]
        return [tuple(out) if out else (1,)]
    if k == "matmul":
        want(len(ins) == 2, "expects 2 inputs")
        x, y = ins
        want(len(x) >= 2 and len(y) >= 2, "operands must be rank >= 2")
        want(len(y) == len(x) or len(y) == 2, "B must match A rank or be rank-2")
        if len(y) == len(x):
            want(x[:-2] == y[:-2], "leading (batch) dims must match")
        want(x[-1] == y[-2], f"contraction mismatch {_s(x)} @ {_s(y)}")
        return [tuple(x[:-1]) + (y[-1],)]
    if k == "einsum":
        subs, rhs = einsum_parse(a["spec"], len(ins), node.id)
        extent: dict[str, int] = {}
        for sub, shape in zip(subs, ins):
            want(len(sub) == len(shape), "subscript rank mismatch")
            for ch, d in zip(sub, shape):
                if ch in extent:
                    want(extent[ch] == d, f"index {ch} extent conflict")
                else:
                    extent[ch] = d
        contracted = [ch for ch in sorted(set("".join(subs))) if ch not in rhs]
        if contracted:
            want(volume(extent[ch] for ch in contracted) >= 2,
                 "contraction must fold at least 2 elements")
        return [tuple(extent[ch] for ch in rhs)]
    if k == "full":
        want(len(ins) == 0, "expects no inputs")
        return [tuple(int(d) for d in a["shape"])]
    if k == "chunk":
        ax, parts, idx = int(a["axis"]), int(a["parts"]), int(a["index"])
        d = ins[0][ax]
        want(parts >= 1 and 0 <= idx < parts, "bad parts/index")
        want(d % parts == 0, f"axis extent {d} not divisible by {parts}")
        out = list(ins[0])
        out[ax] = d // parts
        return [tuple(out)]
    if k == "embedding":
        want(len(ins) == 2, "expects (table, ids)")
        t, ids = ins
        want(len(t) == 2, "table must be rank-2")
        want(t[0] >= volume(ids), "vocab must cover enumerated token ids")
        return [tuple(ids) + (t[1],)]
    if k == "embedding_grad":
        g, ids = ins
        want(len(ins) == 2 and tuple(g[:-1]) == tuple(ids), "grad leading dims must match ids")
        v = int(a["vocab"])
        want(v >= volume(ids), "vocab must cover enumerated token ids")
        return [(v, g[-1])]
    if k == "gnorm_sq":
        want(len(ins) >= 1, "expects at least 1 input")
        return [(1,)]
    # communication: k inputs, k outputs, ordered like attrs["group"]
    n = len(a["group"])
    want(len(ins) == n, f"expects {n} inputs for group of {n}")
    if k == "all_reduce":
        for s in ins[1:]:
            want(s == ins[0], "all_reduce operands must share a shape")
        return [ins[0]] * n
    if k == "all_gather":
        ax = int(a["axis"])
        base = list(ins[0])
        total = 0
        for s in ins:
            want(list(s[:ax]) + list(s[ax + 1:]) == base[:ax] + base[ax + 1:],
                 "all_gather operands differ off-axis")
            total += s[ax]
        base[ax] = total
        return [tuple(base)] * n
    if k == "reduce_scatter":
        ax = int(a["axis"])
        for s in ins[1:]:
            want(s == ins[0], "reduce_scatter operands must share a shape")
        want(ins[0][ax] % n == 0, "scatter axis must divide evenly")
        out = list(ins[0])
        out[ax] //= n
        return [tuple(out)] * n
    # all_to_all
    sa, ca = int(a["split_axis"]), int(a["concat_axis"])
    for s in ins[1:]:
        want(s == ins[0], "all_to_all operands must share a shape")
    want(ins[0][sa] % n == 0, "split axis must divide evenly")
    out = list(ins[0])
    out[sa] //= n
    out[ca] = out[ca] * n
    return [tuple(out)] * n


def validate_concrete(graph: Graph) -> None:
    """Every node's declared output shapes equal its shape rule's result."""
    for node in topo_sort(graph):
        got = infer_shapes(node, [graph.shape(t) for t in node.inputs])
        for tid, shape in zip(node.outputs, got):
            want = graph.shape(tid)
            if tuple(shape) != tuple(want):
                raise ShapeError(f"{node.kind} {node.id}: declares {list(want)} for {tid} "
                                 f"but computes {list(shape)}")

"""TEST INFRASTRUCTURE ONLY. Operator semantics over F_p witness batches.

Restates the reference's concrete evaluator, pkg/src/planeq/oracle.py:81-357
(eval_node), one branch per operator kind, with two changes of domain:
values are F_p residues instead of Fractions, and every tensor carries a
trailing witness axis of length W. Uninterpreted functions (EXP, RSQRT,
SIGMOID) use the keyed hash of m31.uf -- any function-consistent
interpretation is admissible for the reference's uninterpreted semantics
(oracle.py:65-74 uses a sha256 stand-in the same way).

Integer (token) tensors stay concrete numpy int64 arrays without the witness
axis, like the reference keeps them as Python ints.

Definedness: every operand the reference guards with require_nonzero
(ops.py:149 div, :225 rsqrt, :265 softmax) is recorded; a witness where one of
them is 0 is invalid. A guarded operand that is 0 on every witness is treated
as the reference's constant-zero case and raises ZeroDivisionError.
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np

from . import m31

U64 = np.uint64


class Ctx:
    def __init__(self, seed: int, W: int):
        self.seed = seed
        self.W = W
        self.valid = np.ones(W, dtype=bool)

    def require(self, x: np.ndarray):
        x = x.reshape(-1, self.W)
        if x.size and np.all(x == 0, axis=1).any():
            raise ZeroDivisionError("guarded operand is zero on every witness")
        if x.size:
            self.valid &= np.all(x != 0, axis=0)

    def uf(self, fn: str, x):
        return m31.uf(self.seed, fn, x)


def _is_int(t) -> bool:
    return t.dtype == np.int64


def _norm_axes(attrs, rank):
    axes = attrs.get("axes")
    if axes is None:
        return tuple(range(rank))
    return tuple(sorted(int(a) % rank for a in axes))


def eval_node(node, ins: list[np.ndarray], out_shapes: list[tuple], ctx: Ctx) -> list[np.ndarray]:
    k = node.kind
    a = node.attrs
    W = ctx.W

    if k in ("add", "sub", "mul", "div", "dropout"):
        x, y = ins
        if k == "add":
            return [m31.add(x, y)]
        if k == "sub":
            return [m31.sub(x, y)]
        if k in ("mul", "dropout"):
            return [m31.mul(x, y)]
        ctx.require(y)
        return [m31.mul(x, m31.inv(y))]

    if k == "silu_grad":
        x, g = ins
        s = ctx.uf("SIGMOID", x)
        one = U64(1)
        inner = m31.add(s, m31.mul(m31.mul(x, s), m31.sub(np.full_like(s, one), s)))
        return [m31.mul(g, inner)]

    if k in ("identity", "move"):
        return [ins[0].copy()]

    if k == "scale":
        return [m31.mul(ins[0], m31.const(Fraction(a["factor"])))]

    if k == "shift":
        return [m31.add(ins[0], np.full_like(ins[0], m31.const(Fraction(a["addend"]))))]

    if k == "pow":
        e = int(a["exponent"])
        acc = ins[0]
        for _ in range(e - 1):
            acc = m31.mul(acc, ins[0])
        return [acc]

    if k == "rsqrt":
        ctx.require(ins[0])
        return [ctx.uf("RSQRT", ins[0])]

    if k == "silu":
        return [m31.mul(ins[0], ctx.uf("SIGMOID", ins[0]))]

    if k == "softmax":
        x = ins[0]
        es = ctx.uf("EXP", x)
        tot = m31.total(es, axis=-2)   # the last tensor axis sits before the witness axis
        ctx.require(tot)
        return [m31.mul(es, m31.inv(tot)[..., None, :])]

    if k == "create_mask":
        s = out_shapes[0]
        i = np.arange(s[0])[:, None]
        j = np.arange(s[1])[None, :]
        m = (j <= i).astype(np.uint64)
        return [np.repeat(m[..., None], W, axis=-1)]

    if k == "apply_mask":
        x, m = ins
        return [m31.mul(x, np.broadcast_to(m, x.shape))]

    if k == "view":
        x = ins[0]
        tail = () if _is_int(x) else (W,)
        return [x.reshape(tuple(out_shapes[0]) + tail)]

    if k == "transpose":
        perm = [int(p) for p in a["perm"]]
        x = ins[0]
        if not _is_int(x):
            perm = perm + [len(perm)]
        return [np.ascontiguousarray(np.transpose(x, perm))]

    if k == "expand":
        x = ins[0]
        tail = () if _is_int(x) else (W,)
        return [np.ascontiguousarray(np.broadcast_to(x, tuple(out_shapes[0]) + tail))]

    if k in ("sum", "mean"):
        x = ins[0]
        rank = x.ndim - 1
        axes = _norm_axes(a, rank)
        keep = bool(a.get("keepdims"))
        s = x.sum(axis=axes, keepdims=keep, dtype=np.uint64) % m31.P
        s = s.reshape(tuple(out_shapes[0]) + (W,))
        if k == "mean":
            count = 1
            for ax in axes:
                count *= x.shape[ax]
            s = m31.mul(s, m31.const(Fraction(1, count)))
        return [s]

    if k == "matmul":
        A, B = ins
        K = A.shape[-2]
        if B.ndim == A.ndim:
            # [..., M, K, W] x [..., K, N, W]
            acc = None
            for t in range(K):
                term = m31.mul(A[..., :, t:t + 1, :], B[..., t:t + 1, :, :])
                acc = term if acc is None else m31.add(acc, term)
        else:
            acc = None
            for t in range(K):
                term = m31.mul(A[..., :, t:t + 1, :], B[t:t + 1, :, :])
                acc = term if acc is None else m31.add(acc, term)
        return [acc.reshape(tuple(out_shapes[0]) + (W,))]

    if k == "einsum":
        spec = a["spec"].replace(" ", "")
        lhs, rhs = spec.split("->")
        subs = lhs.split(",")
        letters = sorted(set("".join(subs)))
        extent = {}
        for sub, t in zip(subs, ins):
            for ch, d in zip(sub, t.shape[:-1]):
                extent[ch] = d
        contracted = [ch for ch in letters if ch not in rhs]
        out = np.zeros(tuple(out_shapes[0]) + (W,), dtype=np.uint64)
        for oidx in np.ndindex(*out_shapes[0]):
            bind = dict(zip(rhs, oidx))
            acc = np.zeros(W, dtype=np.uint64)
            for combo in np.ndindex(*[extent[c] for c in contracted]):
                bind.update(zip(contracted, combo))
                prod = np.ones(W, dtype=np.uint64)
                for sub, t in zip(subs, ins):
                    prod = m31.mul(prod, t[tuple(bind[ch] for ch in sub)])
                acc = m31.add(acc, prod)
            out[oidx] = acc
        return [out]

    if k == "full":
        v = m31.const(Fraction(a["value"]))
        return [np.full(tuple(out_shapes[0]) + (W,), v, dtype=np.uint64)]

    if k == "chunk":
        ax = int(a["axis"])
        x = ins[0]
        ax = ax % (x.ndim if _is_int(x) else x.ndim - 1)
        width = out_shapes[0][ax]
        off = int(a["index"]) * width
        sl = [slice(None)] * x.ndim
        sl[ax] = slice(off, off + width)
        return [np.ascontiguousarray(x[tuple(sl)])]

    if k == "embedding":
        table, ids = ins
        if ids.min(initial=0) < 0 or ids.max(initial=0) >= table.shape[0]:
            raise IndexError("token id outside table")
        return [np.ascontiguousarray(table[ids])]

    if k == "embedding_grad":
        g, ids = ins
        v, h = out_shapes[0]
        out = np.zeros((v, h, W), dtype=np.uint64)
        flat_ids = ids.reshape(-1)
        gf = g.reshape(-1, h, W)
        for i, row in enumerate(flat_ids):
            out[row] = m31.add(out[row], gf[i])
        return [out]

    if k == "gnorm_sq":
        acc = np.zeros(W, dtype=np.uint64)
        for t in ins:
            sq = m31.mul(t, t).reshape(-1, W)
            acc = m31.add(acc, sq.sum(axis=0, dtype=np.uint64) % m31.P)
        return [acc.reshape(1, W)]

    if k == "all_reduce":
        tot = ins[0]
        for t in ins[1:]:
            tot = m31.add(tot, t)
        return [tot.copy() for _ in ins]

    if k == "all_gather":
        ax = int(a["axis"]) % (ins[0].ndim - 1)
        cat = np.concatenate(ins, axis=ax)
        return [cat.copy() for _ in ins]

    if k == "reduce_scatter":
        ax = int(a["axis"]) % (ins[0].ndim - 1)
        tot = ins[0]
        for t in ins[1:]:
            tot = m31.add(tot, t)
        outs = []
        for j in range(len(ins)):
            w = out_shapes[j][ax]
            sl = [slice(None)] * tot.ndim
            sl[ax] = slice(j * w, (j + 1) * w)
            outs.append(np.ascontiguousarray(tot[tuple(sl)]))
        return outs

    if k == "all_to_all":
        rank = ins[0].ndim - 1
        sa = int(a["split_axis"]) % rank
        ca = int(a["concat_axis"]) % rank
        parts = len(ins)
        q = ins[0].shape[sa] // parts
        outs = []
        for j in range(parts):
            pieces = []
            for src in range(parts):
                sl = [slice(None)] * (rank + 1)
                sl[sa] = slice(j * q, (j + 1) * q)
                pieces.append(ins[src][tuple(sl)])
            outs.append(np.ascontiguousarray(np.concatenate(pieces, axis=ca)))
        return outs

    raise ValueError(f"oracle has no rule for operator kind {k!r}")

"""Shape reduction: the smallest plan with the same verification verdict.

Re-implements the reference reducer (pkg/src/planeq/shapes.py:35-341, with
the per-operator rules of ops.py `reduce_dims` and the term language of
dims.py): every dimension is an integer unknown in [1, full]; both graphs are
walked emitting each operator's alignment/semantic constraints; lineage range
endpoints cut each checkpoint axis into shared piece variables; the system is
minimized for L1 (or "volume": max-dim first), then lexicographically pinned
in declaration order, so a plan always reduces to the same small plan. The
minimizer is z3 through its Python API (the reference drives the same solver
through SMT-LIB text); every model is re-checked by direct evaluation and the
rebuilt plan is revalidated concretely.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

from .errors import InfeasibleShapes, PlanEqError, ShapeError, SolverProtocolError, SolverUnavailable
from .graph import Graph, LineageEntry, entry_tiles_exactly, topo_sort
from .opshape import einsum_parse, reduce_axes, validate_concrete
from .plan import Plan, plan_from_dict, plan_to_dict

# -- integer term language: ("c", n) | ("v", name) | ("+", (..)) | ("*", (..)) ----------


def cint(n: int):
    return ("c", int(n))


def tsum(parts):
    flat, c = [], 0
    for p in parts:
        if p[0] == "c":
            c += p[1]
        elif p[0] == "+":
            flat.extend(p[1])
        else:
            flat.append(p)
    if c:
        flat.append(cint(c))
    if not flat:
        return cint(0)
    return flat[0] if len(flat) == 1 else ("+", tuple(flat))


def tprod(parts):
    flat, c = [], 1
    for p in parts:
        if p[0] == "c":
            c *= p[1]
        elif p[0] == "*":
            flat.extend(p[1])
        else:
            flat.append(p)
    if c == 0:
        return cint(0)
    if c != 1:
        flat.insert(0, cint(c))
    if not flat:
        return cint(1)
    return flat[0] if len(flat) == 1 else ("*", tuple(flat))


def eval_term(t, env) -> int:
    k = t[0]
    if k == "c":
        return t[1]
    if k == "v":
        return env[t[1]]
    if k == "+":
        return sum(eval_term(p, env) for p in t[1])
    v = 1
    for p in t[1]:
        v *= eval_term(p, env)
    return v


def holds(c, env) -> bool:
    op, a, b = c
    va, vb = eval_term(a, env), eval_term(b, env)
    return va == vb if op == "eq" else (va <= vb if op == "le" else va >= vb)


def render(c) -> str:
    def r(t):
        if t[0] == "c":
            return str(t[1])
        if t[0] == "v":
            return t[1]
        return "(" + (" + " if t[0] == "+" else "*").join(r(p) for p in t[1]) + ")"
    op, a, b = c
    return f"{r(a)} {dict(eq='==', le='<=', ge='>=')[op]} {r(b)}"


class Dims:
    """Variables (name -> full-scale bound, declaration order) and constraints."""

    def __init__(self):
        self.vars: dict[str, int] = {}
        self.order: list[str] = []
        self.cons: list[tuple] = []
        self.origin: list[str] = []
        self._fresh = 0

    def declare(self, name: str, full: int):
        if full == 1:
            return cint(1)
        if name in self.vars:
            self.vars[name] = max(self.vars[name], full)
        else:
            self.vars[name] = full
            self.order.append(name)
        return ("v", name)

    def fresh(self, base: str, full: int):
        if full == 1:
            return cint(1)
        self._fresh += 1
        return self.declare(f"f{self._fresh}.{base}", full)

    def add(self, c, origin: str):
        op, a, b = c
        if a[0] == "c" and b[0] == "c":
            if not holds(c, {}):
                self.cons.append(c)        # an impossible constant constraint is the witness
                self.origin.append(origin)
            return
        if op == "eq" and a == b:
            return
        if op == "ge" and b == ("c", 1):
            return
        self.cons.append(c)
        self.origin.append(origin)

    def eq(self, a, b, origin):
        self.add(("eq", a, b), origin)

    def ge(self, a, b, origin):
        self.add(("ge", a, b), origin)


def _eq_all(D: Dims, nid: str, xs, ys, what: str):
    for i, (x, y) in enumerate(zip(xs, ys)):
        D.eq(x, y, f"{nid}:{what}[{i}]")


def reduce_dims(node, ins: list[list], D: Dims, fins, fouts) -> list[list]:
    """Per-operator reduced-dimension rule (reference ops.py reduce_dims methods)."""
    k, a, nid = node.kind, node.attrs, node.id
    if k in ("add", "sub", "mul", "div", "dropout", "silu_grad"):
        for other in ins[1:]:
            _eq_all(D, nid, ins[0], other, "elemwise")
        return [list(ins[0])]
    if k in ("identity", "scale", "shift", "pow", "rsqrt", "silu", "move"):
        return [list(ins[0])]
    if k == "softmax":
        D.ge(ins[0][-1], cint(2), f"{nid}:softmax-axis")
        return [list(ins[0])]
    if k == "create_mask":
        d = D.fresh(f"{nid}.size", fouts[0][0])
        D.ge(d, cint(2), f"{nid}:mask-size")
        return [[d, d]]
    if k == "apply_mask":
        x, m = ins
        D.eq(m[0], m[1], f"{nid}:mask-square")
        _eq_all(D, nid, x[-2:], m, "mask-trailing")
        return [list(x)]
    if k in ("view", "expand"):
        tgt = fouts[0]
        base = a.get("view_key", nid)
        keys = a.get("factor_keys") or [None] * len(tgt)
        out = []
        for ax, d in enumerate(tgt):
            if k == "expand" and fins[0][ax] == d:
                out.append(ins[0][ax])
                continue
            key = keys[ax] if keys[ax] is not None else f"{base}.f{ax}"
            out.append(D.declare(f"k.{key}", d))
        if k == "view":
            D.eq(tprod(list(ins[0])), tprod(out), f"{nid}:view-volume")
        return [out]
    if k == "transpose":
        return [[ins[0][int(p)] for p in a["perm"]]]
    if k in ("sum", "mean"):
        axes = reduce_axes(a, len(ins[0]))
        keep = bool(a.get("keepdims"))
        fold = 1
        for ax in axes:
            fold *= fins[0][ax]
        if fold >= 2:
            red = [ins[0][ax] for ax in axes]
            D.ge(tsum(red), cint(len(red) + 1), f"{nid}:fold-size")
        out = [cint(1) if ax in axes else d for ax, d in enumerate(ins[0]) if keep or ax not in axes]
        return [out if out else [cint(1)]]
    if k == "matmul":
        x, y = ins
        D.eq(x[-1], y[-2], f"{nid}:contraction")
        if fins[0][-1] >= 2:
            D.ge(x[-1], cint(2), f"{nid}:contraction-size")
        if len(y) == len(x):
            _eq_all(D, nid, x[:-2], y[:-2], "batch")
        return [list(x[:-1]) + [y[-1]]]
    if k == "einsum":
        subs, rhs = einsum_parse(a["spec"], len(ins), nid)
        rep: dict = {}
        for sub, shape in zip(subs, ins):
            for ch, d in zip(sub, shape):
                if ch in rep:
                    D.eq(rep[ch], d, f"{nid}:einsum-{ch}")
                else:
                    rep[ch] = d
        contracted = [ch for ch in sorted(rep) if ch not in rhs]
        if contracted:
            D.ge(tsum([rep[ch] for ch in contracted]), cint(len(contracted) + 1),
                 f"{nid}:einsum-fold")
        return [[rep[ch] for ch in rhs]]
    if k == "full":
        return [[D.fresh(f"{nid}.d{ax}", int(d)) for ax, d in enumerate(fouts[0])]]
    if k == "chunk":
        ax, parts = int(a["axis"]), int(a["parts"])
        key = a.get("chunk_key")
        q = D.declare(f"k.{key}", fouts[0][ax]) if key else D.fresh(f"{nid}.q", fouts[0][ax])
        D.eq(ins[0][ax], tprod([cint(parts), q]), f"{nid}:chunk-even")
        out = list(ins[0])
        out[ax] = q
        return [out]
    if k == "embedding":
        t, ids = ins
        D.ge(t[0], tprod(list(ids)), f"{nid}:vocab-covers-ids")
        return [list(ids) + [t[1]]]
    if k == "embedding_grad":
        g, ids = ins
        _eq_all(D, nid, list(g[:-1]), list(ids), "grad-vs-ids")
        v = D.fresh(f"{nid}.v", fouts[0][0])
        D.ge(v, tprod(list(ids)), f"{nid}:vocab-covers-ids")
        return [[v, g[-1]]]
    if k == "gnorm_sq":
        if len(ins) == 1:
            D.ge(tsum(list(ins[0])), cint(len(ins[0]) + 1), f"{nid}:fold-size")
        return [[cint(1)]]
    if k == "all_reduce":
        for other in ins[1:]:
            _eq_all(D, nid, ins[0], other, "all_reduce")
        return [list(ins[0]) for _ in ins]
    if k == "all_gather":
        ax = int(a["axis"])
        for other in ins[1:]:
            _eq_all(D, nid, ins[0][:ax] + ins[0][ax + 1:], other[:ax] + other[ax + 1:],
                    "all_gather-offaxis")
        out = list(ins[0])
        out[ax] = tsum([s[ax] for s in ins])
        return [out for _ in ins]
    if k == "reduce_scatter":
        ax, n = int(a["axis"]), len(ins)
        for other in ins[1:]:
            _eq_all(D, nid, ins[0], other, "reduce_scatter")
        q = D.fresh(f"{nid}.q", fouts[0][ax])
        D.eq(ins[0][ax], tprod([cint(n), q]), f"{nid}:scatter-even")
        out = list(ins[0])
        out[ax] = q
        return [out for _ in ins]
    if k == "all_to_all":
        sa, ca, n = int(a["split_axis"]), int(a["concat_axis"]), len(ins)
        for other in ins[1:]:
            _eq_all(D, nid, ins[0], other, "all_to_all")
        q = D.fresh(f"{nid}.q", fouts[0][sa])
        D.eq(ins[0][sa], tprod([cint(n), q]), f"{nid}:split-even")
        out = list(ins[0])
        out[sa] = q
        out[ca] = tprod([cint(n), ins[0][ca]])
        return [out for _ in ins]
    raise PlanEqError(f"no reduction rule for operator kind {k!r}")


class _Grid:
    """Per-axis endpoint cuts of one lineage entry; each piece is a variable."""

    def __init__(self, tid: str, entry: LineageEntry, shape, D: Dims):
        self.points: list[list[int]] = []
        self.pieces: list[list] = []
        for ax, d in enumerate(shape):
            pts = {0, d}
            for rs in entry.groups():
                if len(rs) != len(shape):
                    raise ShapeError(f"lineage {tid}: shard rank != tensor rank")
                lo, hi = rs[ax]
                pts.add(max(0, min(lo, d)))
                pts.add(max(0, min(hi, d)))
            srt = sorted(pts)
            self.points.append(srt)
            self.pieces.append([D.declare(f"p.{tid}.{ax}.{i}", srt[i + 1] - srt[i])
                                for i in range(len(srt) - 1)])

    def dims(self):
        return [tsum(list(p)) for p in self.pieces]

    def span(self, ax: int, lo: int, hi: int):
        pts = self.points[ax]
        return tsum(self.pieces[ax][pts.index(lo):pts.index(hi)])

    def reduced_range(self, ax: int, lo: int, hi: int, env) -> tuple[int, int]:
        pts = self.points[ax]
        cum = [0]
        for p in self.pieces[ax]:
            cum.append(cum[-1] + eval_term(p, env))
        return cum[pts.index(lo)], cum[pts.index(hi)]


@dataclass
class Reduction:
    env: dict
    plan: Plan
    report: dict = field(default_factory=dict)


class _Reducer:
    def __init__(self, plan: Plan):
        if plan.parallel is None or plan.lineage is None:
            raise PlanEqError("reduction needs a parallel graph and lineage")
        self.plan = plan
        self.D = Dims()
        self.grids: dict[str, _Grid] = {}
        self.dims: dict[tuple[str, str], list] = {}
        self.misaligned: list[str] = []
        self.vocab_of_ids: dict[str, tuple] = {}

    def build(self):
        plan, D = self.plan, self.D
        for tid, entry in plan.lineage.items():
            shape = plan.logical.shape(tid)
            self.grids[tid] = _Grid(tid, entry, shape, D)
            if not entry_tiles_exactly(entry, shape):
                self.misaligned.append(tid)
        self._walk("L", plan.logical)
        self._walk("P", plan.parallel)
        for tid, entry in plan.lineage.items():
            grid = self.grids[tid]
            for s in entry.shards:
                terms = self.dims.get(("P", s.tensor))
                if terms is None:
                    continue
                if len(s.ranges) != len(terms):
                    raise ShapeError(f"lineage {tid}: shard {s.tensor} rank mismatch")
                for ax, (lo, hi) in enumerate(s.ranges):
                    D.eq(terms[ax], grid.span(ax, lo, hi), f"{tid}:shard-span:{s.tensor}")

    def _input_terms(self, tag, tid, src, shape):
        grid = self.grids.get(src)
        if grid is not None and tag == "L":
            return grid.dims()
        if grid is not None and tag == "P":
            for s in self.plan.lineage[src].shards:
                if s.tensor == tid:
                    return [grid.span(ax, lo, hi) for ax, (lo, hi) in enumerate(s.ranges)]
        return [self.D.declare(f"d.{tag}.{tid}.{ax}", d) for ax, d in enumerate(shape)]

    def _walk(self, tag: str, graph: Graph):
        D = self.D
        for tid in graph.inputs:
            t = graph.tensors[tid]
            src = t.meta.get("from", tid) if tag == "P" else tid
            self.dims[(tag, tid)] = self._input_terms(tag, tid, src, t.shape)
        inputs = set(graph.inputs)
        for node in topo_sort(graph):
            ins = [self.dims[(tag, t)] for t in node.inputs]
            outs = reduce_dims(node, ins, D, [graph.shape(t) for t in node.inputs],
                               [graph.shape(t) for t in node.outputs])
            if node.kind in ("embedding", "embedding_grad"):
                vterm = ins[0][0] if node.kind == "embedding" else outs[0][0]
                self.vocab_of_ids.setdefault(node.inputs[1], vterm)
            for tid, terms in zip(node.outputs, outs):
                self.dims[(tag, tid)] = terms
                if tag == "L" and tid in self.grids and tid not in inputs:
                    for ax, term in enumerate(terms):
                        D.eq(term, self.grids[tid].dims()[ax], f"{tid}:lineage-dim")

    # -- minimization ---------------------------------------------------------------

    def solve(self, objective: str, timeout_s: float) -> tuple[dict, dict]:
        D = self.D
        full = dict(D.vars)
        bad = [f"{render(c)}   [{o}]" for c, o in zip(D.cons, D.origin) if not holds(c, full)]
        if bad:
            raise InfeasibleShapes("shape constraints are unsatisfiable at full scale", witness=bad)
        names = list(D.order)
        if not names:
            return full, {"checks": 0, "solver_status": "trivial"}
        try:
            import z3
        except ImportError as e:  # pragma: no cover - the image ships z3
            raise SolverUnavailable(f"z3 python bindings unavailable: {e}") from e
        stats = {"checks": 0, "solver_status": "ok"}
        deadline = time.monotonic() + timeout_s
        V = {n: z3.Int(n) for n in names}

        def zt(t):
            k = t[0]
            if k == "c":
                return z3.IntVal(t[1])
            if k == "v":
                return V[t[1]]
            parts = [zt(p) for p in t[1]]
            if k == "+":
                return z3.Sum(parts)
            out = parts[0]
            for p in parts[1:]:
                out = out * p
            return out

        s = z3.Solver()
        for n in names:
            s.add(V[n] >= 1, V[n] <= D.vars[n])
        for op, a, b in D.cons:
            za, zb = zt(a), zt(b)
            s.add(za == zb if op == "eq" else (za <= zb if op == "le" else za >= zb))
        best = dict(full)

        def probe(extra) -> str:
            stats["checks"] += 1
            s.push()
            s.add(extra)
            s.set("timeout", max(500, int((deadline - time.monotonic()) * 1000)))
            r = s.check()
            if r == z3.sat:
                m = s.model()
                for n in names:
                    v = m.eval(V[n], model_completion=True)
                    best[n] = v.as_long()
            s.pop()
            if r == z3.unknown:
                stats["solver_status"] = "partial"
            return "sat" if r == z3.sat else ("unsat" if r == z3.unsat else "unknown")

        total = z3.Sum([V[n] for n in names])
        if objective == "volume":
            lo, hi = 1, max(best.values())
            while lo < hi and time.monotonic() < deadline:
                mid = (lo + hi) // 2
                r = probe(z3.And([V[n] <= mid for n in names]))
                if r == "sat":
                    hi = max(best.values())
                elif r == "unsat":
                    lo = mid + 1
                else:
                    break
            cap = max(best.values())
            s.add(z3.And([V[n] <= cap for n in names]))
        lo, hi = len(names), sum(best.values())
        while lo < hi and time.monotonic() < deadline:
            mid = (lo + hi) // 2
            r = probe(total <= mid)
            if r == "sat":
                hi = sum(best.values())
            elif r == "unsat":
                lo = mid + 1
            else:
                break
        s.add(total <= sum(best.values()))
        for n in names:
            if time.monotonic() > deadline:
                stats["solver_status"] = "partial"
                break
            if best[n] <= 1:
                continue
            lo, hi = 1, best[n]
            while lo < hi:
                mid = (lo + hi) // 2
                r = probe(V[n] <= mid)
                if r == "sat":
                    hi = best[n]
                elif r == "unsat":
                    lo = mid + 1
                else:
                    break
            s.add(V[n] == best[n])
        for c, o in zip(D.cons, D.origin):
            if not holds(c, best):
                raise SolverProtocolError(f"solver model violates {render(c)} [{o}]")
        return best, stats

    def rebuild(self, env) -> Plan:
        d = plan_to_dict(self.plan)
        for tag, gd in (("L", d["logical"]), ("P", d["parallel"])):
            shapes = {}
            for td in gd["tensors"]:
                shape = [eval_term(t, env) for t in self.dims[(tag, td["id"])]]
                shapes[td["id"]] = shape
                td["shape"] = shape
                if td["meta"].get("vocab") is not None:
                    vt = self.vocab_of_ids.get(td["id"])
                    if vt is not None:
                        td["meta"] = dict(td["meta"], vocab=eval_term(vt, env))
            for nd in gd["nodes"]:
                kind, attrs = nd["kind"], nd["attrs"]
                if kind in ("view", "expand", "full"):
                    attrs["shape"] = list(shapes[nd["outputs"][0]])
                elif kind == "create_mask":
                    attrs["size"] = shapes[nd["outputs"][0]][0]
                elif kind == "embedding_grad":
                    attrs["vocab"] = shapes[nd["outputs"][0]][0]
        for ed in d["lineage"]:
            grid = self.grids[ed["logical"]]
            for sd in ed["shards"]:
                sd["ranges"] = [list(grid.reduced_range(ax, lo, hi, env))
                                for ax, (lo, hi) in enumerate(sd["ranges"])]
        d["provenance"] = dict(d.get("provenance") or {})
        d["provenance"]["reduced_from"] = {tid: list(self.plan.logical.shape(tid))
                                           for tid in self.plan.lineage}
        return plan_from_dict(d)


def reduce_plan(plan: Plan, objective: str = "l1", solver_argv: list[str] | None = None,
                timeout_s: float = 120.0) -> Reduction:
    """Shrink a plan to its minimal shape assignment (verdict-preserving)."""
    t0 = time.monotonic()
    validate_concrete(plan.logical)
    validate_concrete(plan.parallel)
    red = _Reducer(plan)
    red.build()
    env, stats = red.solve(objective, timeout_s)
    small = red.rebuild(env)
    validate_concrete(small.logical)
    validate_concrete(small.parallel)
    report = {"objective": objective, "vars": len(red.D.order), "constraints": len(red.D.cons),
              "misaligned": sorted(red.misaligned), "orig_total": sum(red.D.vars.values()),
              "reduced_total": sum(env.get(n, 1) for n in red.D.order),
              "wall_s": round(time.monotonic() - t0, 3), **stats}
    return Reduction(env=env, plan=small, report=report)

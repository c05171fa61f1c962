"""TEST INFRASTRUCTURE ONLY: regenerate tests/golden/* from the reference.

Runs in the build container only (needs the reference package under
/root/reference/pkg/src and its dependencies: sympy, z3 on PATH). The GPU box
never runs this; it only reads the committed fixtures.

Produces
  tests/golden/ops.json          per-operator vectors: integer inputs, and the
                                 reference's exact-rational eval_node output
                                 (pkg/src/planeq/oracle.py:81) mapped into F_p,
                                 with EXP/RSQRT/SIGMOID interpreted by the
                                 keyed hash (rational -> residue -> hash).
  tests/golden/plans/<name>.json.gz   work plans (reduced by the reference's
                                 own reduce_plan when it succeeds, else full
                                 scale) of the toy decoder under several
                                 parallel configs, faulted mutants of them, and
                                 the reference's random soundness corpus.
  tests/golden/verdicts.json     the reference's verify_plan outcome on each
                                 plan (no_reduce=True on the stored work plan,
                                 no_cancel=True): overall verdict, per-stage
                                 status list, stage targets, or the exception
                                 class it raised; plus build_stages structure.

Usage: python -m oracle.gen_golden [--quick]
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from fractions import Fraction

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLDEN = os.path.join(ROOT, "tests", "golden")
P = (1 << 31) - 1
SEED = 1234


def _ref():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import planeq  # noqa: F401
    return planeq


def _residue(q) -> int:
    q = Fraction(q)
    return (q.numerator % P) * pow(q.denominator % P, P - 2, P) % P


def _hash_uf(seed: int):
    sys.path.insert(0, ROOT)
    from paper_2506_15961_b200 import field as F
    keys = {fn: F.fn_key(seed, fn) for fn in F.FN_NAMES}

    def uf(fn, x):
        return Fraction(F.uf_apply(keys[fn], _residue(x)))
    return uf


# -- operator vectors -----------------------------------------------------------


def gen_ops(seed: int = SEED, trials: int = 3) -> dict:
    _ref()
    from planeq.oracle import RT, _PROBE_INSTANCES, _probe_node, eval_node
    uf = _hash_uf(seed)
    rng = random.Random(seed)
    out = {"seed": seed, "p": P, "cases": []}
    for kind in sorted(_PROBE_INSTANCES):
        node, in_shapes, out_shapes = _probe_node(kind)
        for t in range(trials):
            ins, ins_json = [], []
            for j, s in enumerate(in_shapes):
                n = 1
                for d in s:
                    n *= d
                if kind in ("embedding", "embedding_grad") and j == 1:
                    vocab = in_shapes[0][0] if kind == "embedding" else int(node.attrs["vocab"])
                    vals = [rng.randrange(vocab) for _ in range(n)]
                    ins.append(RT(s, vals))
                    ins_json.append({"shape": list(s), "int": True, "data": vals})
                else:
                    vals = [rng.randrange(1, P) for _ in range(n)]
                    ins.append(RT(s, [Fraction(v) for v in vals]))
                    ins_json.append({"shape": list(s), "int": False, "data": vals})
            try:
                got = eval_node(node, ins, out_shapes, "exact", uf)
            except ZeroDivisionError:
                continue
            attrs = {k: (str(v) if isinstance(v, Fraction) else v) for k, v in node.attrs.items()}
            out["cases"].append({
                "kind": kind, "attrs": attrs, "inputs": ins_json,
                "out_shapes": [list(s) for s in out_shapes],
                "outputs": [[_residue(v) for v in rt.data] for rt in got],
            })
    return out


# -- plan corpus -----------------------------------------------------------------


def _toy_plans(quick: bool):
    _ref()
    from planeq.completion import LossSpec, complete
    from planeq.parallelize import ParallelConfig, parallelize
    from planeq.toy import ToyConfig, toy_forward, toy_interiors
    fw = toy_forward(ToyConfig())
    g = complete(fw, LossSpec(kind="mean"))
    cfgs = [("tp2", ParallelConfig(tp=2)), ("pp2nm2", ParallelConfig(pp=2, nm=2)),
            ("dp2tp2pp2nm2", ParallelConfig(dp=2, tp=2, pp=2, nm=2)),
            ("tp2pp2", ParallelConfig(tp=2, pp=2)), ("dp2tp2nm2", ParallelConfig(dp=2, tp=2, nm=2))]
    if quick:
        cfgs = cfgs[:1]
    out = {}
    for name, cfg in cfgs:
        out[name] = parallelize(g, cfg, lineage_interiors=toy_interiors(g))
    return out


def _work_plan(plan):
    """The plan verify would discharge: reduced when the reference can reduce it."""
    from planeq.shapes import reduce_plan
    try:
        return reduce_plan(plan).plan, "reduced"
    except Exception as e:  # noqa: BLE001 - the reference's own failure is recorded
        return plan, f"full ({type(e).__name__})"


def _fault_mutants(base_name, plan, per_category: int, rng: random.Random):
    from planeq.faults import CATEGORIES, inject, list_sites
    out = []
    for cat in list(CATEGORIES) + ["extra_op"]:
        sites = list_sites(plan, cat)
        rng.shuffle(sites)
        for spec in sites[:per_category]:
            out.append((f"{base_name}.{cat}.{len(out)}", inject(plan, spec), spec.to_dict()))
    return out


def _verify_job(args):
    """Reference outcome on one plan: verify_plan with default options (shape
    reduction on) and no_cancel, plus the reduced work plan when reduction
    succeeds (that is the plan the GPU parity tests discharge)."""
    name, blob, full_too = args
    _ref()
    from planeq.plan import dumps, loads
    from planeq.shapes import reduce_plan
    from planeq.stages import build_stages
    from planeq.verify import VerifyOptions, verify_plan
    plan = loads(blob)
    rec = {"name": name}
    work_blob = None

    def outcome(p, no_reduce):
        t0 = time.time()
        out = {}
        try:
            rep = verify_plan(p, VerifyOptions(jobs=1, no_reduce=no_reduce, no_cancel=True,
                                               timeout_s=120.0))
            out["verdict"] = rep["verdict"]
            out["refuted_by"] = rep.get("refuted_by")
            out["stage_status"] = [(s["target"], s["status"]) for s in rep["stages"]]
            out["stage_reason"] = {s["target"]: (s.get("detail") or {}).get("reason")
                                   for s in rep["stages"] if s["status"] != "proven"}
            out["obligations"] = [(s["target"], s["obligations"]) for s in rep["stages"]]
        except Exception as e:  # noqa: BLE001
            out["error"] = type(e).__name__
            out["message"] = str(e)[:300]
        out["ref_wall_s"] = round(time.time() - t0, 3)
        return out

    rec["default"] = outcome(plan, False)
    try:
        work = reduce_plan(plan).plan
        work_blob = dumps(work)
        stages, _ = build_stages(work)
        rec["work_stages"] = [{"target": s.target, "logical": [n.id for n in s.logical_nodes],
                               "parallel": [n.id for n in s.parallel_nodes],
                               "l_inputs": s.l_inputs, "p_inputs": s.p_inputs} for s in stages]
    except Exception as e:  # noqa: BLE001
        rec["reduce_error"] = type(e).__name__
    if full_too:
        rec["no_reduce"] = outcome(plan, True)
    return rec, work_blob


def gen_plans(quick: bool = False, jobs: int = 8):
    _ref()
    from planeq.oracle import random_plan
    from planeq.plan import dumps
    rng = random.Random(SEED)
    corpus = []   # (name, plan, meta, full_too)
    for name, plan in _toy_plans(quick).items():
        corpus.append((name, plan, {"source": "toy"}, False))
        if name == "dp2tp2pp2nm2" or quick:
            for mname, mutant, spec in _fault_mutants(name, plan, 1 if quick else 2, rng):
                corpus.append((mname, mutant, {"source": "fault", "fault": spec}, False))
    for i in range(8 if quick else 40):
        fault = i % 2 == 1
        try:
            plan = random_plan(SEED * 100003 + i, fault)
        except Exception:  # noqa: BLE001
            continue
        corpus.append((f"rnd{i}", plan, {"source": "random_plan", "fault": fault}, True))
    pdir = os.path.join(GOLDEN, "plans")
    os.makedirs(pdir, exist_ok=True)
    for f in os.listdir(pdir):
        os.remove(os.path.join(pdir, f))
    args = [(name, dumps(plan), full) for name, plan, _, full in corpus]
    with ProcessPoolExecutor(max_workers=jobs) as ex:
        outs = list(ex.map(_verify_job, args))
    recs = []
    for (name, plan, meta, full), (rec, work_blob) in zip(corpus, outs):
        rec["meta"] = meta
        # store the plan itself (host-side tests) and the reduced work plan
        with gzip.open(os.path.join(pdir, f"{name}.json.gz"), "wt") as f:
            f.write(dumps(plan))
        if work_blob is not None:
            with gzip.open(os.path.join(pdir, f"{name}.work.json.gz"), "wt") as f:
                f.write(work_blob)
            rec["work_plan"] = f"plans/{name}.work.json.gz"
        rec["plan"] = f"plans/{name}.json.gz"
        recs.append(rec)
    return recs


def main(argv=None):
    argv = argv if argv is not None else sys.argv[1:]
    quick = "--quick" in argv
    os.makedirs(GOLDEN, exist_ok=True)
    t0 = time.time()
    ops = gen_ops()
    with open(os.path.join(GOLDEN, "ops.json"), "w") as f:
        json.dump(ops, f, sort_keys=True)
    print(f"ops: {len(ops['cases'])} cases ({time.time() - t0:.1f}s)", flush=True)
    if "--ops-only" in argv:
        return 0
    recs = gen_plans(quick=quick)
    with open(os.path.join(GOLDEN, "verdicts.json"), "w") as f:
        json.dump({"generator": "oracle/gen_golden.py", "reference": REF_SRC,
                   "plans": recs}, f, sort_keys=True, indent=1)
    print(f"plans: {len(recs)} ({time.time() - t0:.1f}s)")
    for r in recs:
        d = r["default"]
        print(r["name"], d.get("verdict", d.get("error")), d["ref_wall_s"],
              "work" if "work_plan" in r else r.get("reduce_error"))
    return 0


if __name__ == "__main__":
    sys.exit(main())

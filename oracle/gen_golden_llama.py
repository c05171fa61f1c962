"""TEST INFRASTRUCTURE ONLY: reference verdicts on the Llama-family plans.

The reference ships no Llama/DeepSeek builder, so the plans come from this
repo's generator (paper_2506_15961_b200.workloads, shape-reduced by
construction); the *verdicts* come from the reference implementation itself
(pkg/src/planeq/verify.py:62 verify_plan, no_reduce=True, no_cancel=True,
with its bundled decision engine `python -m planeq.smtsolver` so every stage
is decided instead of timing out in z3). Covers BASELINE configs[0] (2-layer
TP2xDP2), a small member of configs[1]'s family (TP, PP, DP, microbatches,
sequence parallelism) and configs[2]'s bug-injected variants (wrong
all-reduce scaling, misordered concat, dropped partial sum, DP averaging).

Writes tests/golden/plans/llama.*.json.gz and tests/golden/verdicts_llama.json.
Usage (build container only): python -m oracle.gen_golden_llama
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys
import time
from concurrent.futures import ProcessPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLDEN = os.path.join(ROOT, "tests", "golden")
REF_SRC = "/root/reference/pkg/src"
SEED = 77


def _plans():
    sys.path.insert(0, ROOT)
    from paper_2506_15961_b200.faults import inject, list_sites
    from paper_2506_15961_b200.workloads import LlamaPlanSpec, llama_plan
    base = {
        "llama.2l-tp2dp2": LlamaPlanSpec(2, tp=2, pp=1, dp=2, nm=1, sp=False, desc="configs[0]"),
        "llama.2l-tp2pp2dp2nm2-sp": LlamaPlanSpec(2, tp=2, pp=2, dp=2, nm=2, sp=True,
                                                 desc="configs[1] family, small"),
    }
    out = []
    rng = random.Random(SEED)
    for name, spec in base.items():
        plan = llama_plan(spec)
        out.append((name, plan, {"source": "llama", "spec": spec.desc}))
        if name.endswith("-sp"):
            for cat in ("wrong_allreduce_scaling", "misordered_concat", "dropped_partial_sum",
                        "wrong_scaling"):
                sites = list_sites(plan, cat)
                if cat == "wrong_scaling":
                    sites = [s for s in sites if s.detail.get("variant") == "avg"]
                rng.shuffle(sites)
                for spec_ in sites[:2]:
                    out.append((f"{name}.{cat}.{len(out)}", inject(plan, spec_),
                                {"source": "llama-fault", "fault": spec_.to_dict()}))
    return out


def _job(args):
    name, blob = args
    os.environ["PLANEQ_SOLVER"] = sys.executable + " -m planeq.smtsolver"
    os.environ["PYTHONPATH"] = REF_SRC
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    from planeq.plan import loads
    from planeq.stages import build_stages
    from planeq.verify import VerifyOptions, verify_plan
    plan = loads(blob)
    rec = {"name": name}
    t0 = time.time()
    try:
        stages, _ = build_stages(plan)
        rec["stages"] = [{"target": s.target, "logical": [n.id for n in s.logical_nodes],
                          "parallel": [n.id for n in s.parallel_nodes]} for s in stages]
        rep = verify_plan(plan, VerifyOptions(jobs=1, no_reduce=True, no_cancel=True,
                                              timeout_s=300.0))
        rec["verdict"] = rep["verdict"]
        rec["refuted_by"] = rep.get("refuted_by")
        rec["stage_status"] = [(s["target"], s["status"]) for s in rep["stages"]]
        rec["stage_reason"] = {s["target"]: (s.get("detail") or {}).get("reason")
                               for s in rep["stages"] if s["status"] == "unknown"}
    except Exception as e:  # noqa: BLE001 - recorded as the reference's outcome
        rec["error"] = type(e).__name__
        rec["message"] = str(e)[:300]
    rec["ref_wall_s"] = round(time.time() - t0, 2)
    return rec


def main():
    sys.path.insert(0, ROOT)
    from paper_2506_15961_b200.plan import dumps
    plans = _plans()
    pdir = os.path.join(GOLDEN, "plans")
    os.makedirs(pdir, exist_ok=True)
    args = []
    for name, plan, _meta in plans:
        blob = dumps(plan)
        with gzip.open(os.path.join(pdir, f"{name}.json.gz"), "wt") as f:
            f.write(blob)
        args.append((name, blob))
    with ProcessPoolExecutor(max_workers=6) as ex:
        recs = list(ex.map(_job, args))
    for rec, (name, _plan, meta) in zip(recs, plans):
        rec["meta"] = meta
        rec["plan"] = f"plans/{name}.json.gz"
    with open(os.path.join(GOLDEN, "verdicts_llama.json"), "w") as f:
        json.dump({"generator": "oracle/gen_golden_llama.py", "solver": "reference bundled engine",
                   "plans": recs}, f, indent=1, sort_keys=True)
    for r in recs:
        print(r["name"], r.get("verdict", r.get("error")), r["ref_wall_s"])


if __name__ == "__main__":
    main()

"""TEST INFRASTRUCTURE ONLY: reference verdicts on DeepSeek-V3-family plans.

BASELINE configs[4]: MLA attention + MoE with expert parallelism (expert
weights split over the tensor group, token dispatch by all_to_all from the
sequence-parallel region). The plans come from this repo's generator
(paper_2506_15961_b200.workloads / builder.deepseek_forward, shape-reduced by
construction); the verdicts come from the reference implementation itself
(pkg/src/planeq/verify.py:62 verify_plan with its bundled decision engine),
exactly as oracle/gen_golden_llama.py does for the Llama family. Fault
variants misorder an all_to_all's inputs and drop a partial sum.

Writes tests/golden/plans/deepseek.*.json.gz and tests/golden/verdicts_deepseek.json.
Usage (build container only): python -m oracle.gen_golden_deepseek
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys
from concurrent.futures import ProcessPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLDEN = os.path.join(ROOT, "tests", "golden")
SEED = 91


def _plans():
    sys.path.insert(0, ROOT)
    from paper_2506_15961_b200.faults import inject, list_sites
    from paper_2506_15961_b200.workloads import GENERATED, deepseek_plan
    out = []
    rng = random.Random(SEED)
    name = "deepseek.2l-tp2dp2-sp"
    plan = deepseek_plan(GENERATED["deepseek-2l-tp2dp2-sp"])
    out.append((name, plan, {"source": "deepseek", "spec": "configs[4] family, small"}))
    for cat in ("misordered_concat", "dropped_partial_sum"):
        sites = list_sites(plan, cat)
        a2a = [s for s in sites if s.site.startswith("a2a.")]
        rng.shuffle(sites)
        pick = (a2a[:1] + [s for s in sites if s not in a2a][:1]) if a2a else sites[:2]
        for spec_ in pick:
            out.append((f"{name}.{cat}.{len(out)}", inject(plan, spec_),
                        {"source": "deepseek-fault", "fault": spec_.to_dict()}))
    return out


def main():
    sys.path.insert(0, ROOT)
    from oracle.gen_golden_llama import _job
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
    with open(os.path.join(GOLDEN, "verdicts_deepseek.json"), "w") as f:
        json.dump({"generator": "oracle/gen_golden_deepseek.py",
                   "solver": "reference bundled engine", "plans": recs}, f, indent=1,
                  sort_keys=True)
    for r in recs:
        print(r["name"], r.get("verdict", r.get("error")), r["ref_wall_s"])


if __name__ == "__main__":
    main()

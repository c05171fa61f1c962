"""TEST INFRASTRUCTURE ONLY: the reference's own per-stage verdicts on a large workload.

Same record as oracle/gen_golden_full.py (tests/golden/verdicts_full_<name>.json,
plan digest + per-stage (target, status)), produced by the reference's own code
on the reference's own Plan object:

  * plan: this repo's deterministic generator output (workloads.get_workload,
    fault-injected variants "<workload>~<category>" included), serialised with
    this repo's dumps and parsed back by the reference's planeq.plan.loads;
  * stages: the reference's planeq.stages.build_stages, run once in the parent;
  * verdicts: the reference's planeq.stages.run_stage on every stage (the loop
    body of verify.py:62 verify_plan with no_reduce and no_cancel, its bundled
    decision engine), in forked worker processes that inherit the plan and
    the stage list copy-on-write.

verify_plan's own worker pool re-parses the plan text and re-runs
build_stages in every worker, and pickles the plan text into every task
(verify.py:48-58, :104-107); on the 0.5 GB Llama3-405B plan text that alone
is hours, so the fan-out here is done once by fork instead. Stage verdicts
are the same function of (plan, stage) either way.

Progress is appended to .work/sweep_<name>.jsonl so an interrupted sweep
resumes where it stopped.

With --budget-s T the sweep stops after T seconds of wall time and writes a
partial record instead (tests/golden/verdicts_partial_<name>.json: the stages
done so far with their indices, merged with an earlier partial record of the
same plan digest); --shuffle SEED takes the remaining stages in a seeded
random order, so a bounded run samples the whole plan instead of its prefix.

Usage (build container only):
  python -m oracle.gen_golden_sweep <workload> [jobs] [--mem-gb G] [--shuffle SEED] [--budget-s T]
"""

from __future__ import annotations

import gc
import hashlib
import json
import os
import resource
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLDEN = os.path.join(ROOT, "tests", "golden")
WORK = os.path.join(ROOT, ".work")
REF_SRC = "/root/reference/pkg/src"

_S: dict = {}


def _one(i: int) -> dict:
    from planeq.stages import run_stage
    st = _S["stages"][i]
    t0 = time.time()
    try:
        r = run_stage(_S["plan"], st, None, 300.0)
        rec = {"i": i, "target": r.target, "status": r.status,
               "reason": (r.detail or {}).get("reason") or r.note}
    except MemoryError:
        rec = {"i": i, "target": st.target, "status": "error", "reason": "MemoryError"}
    except Exception as e:  # noqa: BLE001 - the reference's own outcome
        rec = {"i": i, "target": st.target, "status": "error",
               "reason": f"{type(e).__name__}: {str(e)[:200]}"}
    rec["wall_s"] = round(time.time() - t0, 2)
    return rec


def _init(mem_gb: float):
    if mem_gb > 0:
        lim = int(mem_gb * (1 << 30))
        resource.setrlimit(resource.RLIMIT_AS, (lim, lim))


def main():
    def opt(flag, cast, default):
        return cast(sys.argv[sys.argv.index(flag) + 1]) if flag in sys.argv else default
    mem_gb = opt("--mem-gb", float, 0.0)
    shuffle = opt("--shuffle", int, None)
    budget_s = opt("--budget-s", float, 0.0)
    args = [a for k, a in enumerate(sys.argv[1:], 1)
            if not a.startswith("--") and not sys.argv[k - 1].startswith("--")]
    name = args[0]
    jobs = int(args[1]) if len(args) > 1 else max(1, (os.cpu_count() or 2) - 2)
    sys.path.insert(0, ROOT)
    os.makedirs(WORK, exist_ok=True)
    t_start = time.time()
    from paper_2506_15961_b200.plan import dumps
    from paper_2506_15961_b200.workloads import get_workload
    _desc, plan = get_workload(name)
    blob = dumps(plan)
    del plan
    digest = hashlib.sha256(blob.encode()).hexdigest()
    os.environ["PLANEQ_SOLVER"] = sys.executable + " -m planeq.smtsolver"
    os.environ["PYTHONPATH"] = REF_SRC
    sys.path.insert(0, REF_SRC)
    from planeq.plan import loads
    from planeq.stages import build_stages
    rplan = loads(blob)
    del blob
    t0 = time.time()
    stages, _uncovered = build_stages(rplan)
    t_build = time.time() - t0
    print(f"{name}: {len(stages)} stages, reference build_stages {t_build:.1f}s", flush=True)
    prog = os.path.join(WORK, f"sweep_{name}.jsonl")
    done: dict[int, dict] = {}
    if os.path.exists(prog):
        with open(prog) as f:
            for line in f:
                d = json.loads(line)
                if d.get("digest") == digest:
                    done[d["i"]] = d
    part_path = os.path.join(GOLDEN, f"verdicts_partial_{name}.json")
    prior = json.load(open(part_path)) if os.path.exists(part_path) else None
    if prior and prior.get("plan_sha256") == digest:
        idx = prior.get("stage_index") or list(range(len(prior["stage_status"])))
        for i, (tgt, st) in zip(idx, prior["stage_status"]):
            done.setdefault(i, {"i": i, "target": tgt, "status": st,
                                "reason": prior.get("stage_reason", {}).get(tgt), "wall_s": 0.0})
    todo = [i for i in range(len(stages)) if i not in done]
    if shuffle is not None:
        import random
        random.Random(shuffle).shuffle(todo)
    _S.update(plan=rplan, stages=stages)
    gc.collect()
    gc.freeze()
    import multiprocessing as mp
    with open(prog, "a") as out, mp.get_context("fork").Pool(jobs, _init, (mem_gb,)) as pool:
        for k, rec in enumerate(pool.imap_unordered(_one, todo, chunksize=1)):
            rec["digest"] = digest
            out.write(json.dumps(rec) + "\n")
            out.flush()
            done[rec["i"]] = rec
            if k % 50 == 0:
                print(f"  {len(done)}/{len(stages)} ({time.time() - t_start:.0f}s)", flush=True)
            if budget_s and time.time() - t_start > budget_s:
                _write_partial(part_path, name, digest, jobs, done, len(stages), t_build, prior)
                pool.terminate()
                return
    recs = [done[i] for i in range(len(stages))]
    statuses = {r["status"] for r in recs}
    verdict = ("refuted" if "refuted" in statuses else
               "unknown" if statuses - {"proven"} else "proven")
    rec = {
        "name": name, "plan_sha256": digest, "generator": "oracle/gen_golden_sweep.py",
        "solver": "reference bundled engine", "jobs": jobs,
        "verdict": verdict,
        "stage_status": [(r["target"], r["status"]) for r in recs],
        "stage_reason": {r["target"]: r["reason"] for r in recs if r["status"] != "proven"
                         and r.get("reason")},
        "ref_build_stages_s": round(t_build, 1),
        "ref_stage_cpu_s": round(sum(r["wall_s"] for r in recs), 1),
        "ref_wall_s": round(time.time() - t_start, 1),
    }
    with open(os.path.join(GOLDEN, f"verdicts_full_{name}.json"), "w") as f:
        json.dump(rec, f, indent=1)
    print(name, rec["verdict"], rec["ref_wall_s"], "s",
          {k: sum(1 for _, st in rec["stage_status"] if st == k)
           for k in ("proven", "refuted", "unknown", "error")}, flush=True)


def _write_partial(path, name, digest, jobs, done, n_total, t_build, prior):
    idx = sorted(done)
    rec = {
        "name": name, "plan_sha256": digest,
        "generator": "oracle/gen_golden_sweep.py (bounded: --budget-s; remaining stages in seeded random order)",
        "solver": "reference bundled engine", "jobs": jobs, "partial": True,
        "stages_checked": len(idx), "stages_total": n_total,
        "stage_index": idx,
        "stage_status": [(done[i]["target"], done[i]["status"]) for i in idx],
        "stage_reason": {done[i]["target"]: done[i]["reason"] for i in idx
                         if done[i]["status"] != "proven" and done[i].get("reason")},
        "ref_build_stages_s": round(t_build, 1),
        "ref_stage_cpu_s": round(sum(done[i].get("wall_s", 0.0) for i in idx)
                                 + (prior or {}).get("ref_stage_cpu_s", 0.0), 1),
        "note": (prior or {}).get("note", ""),
    }
    with open(path, "w") as f:
        json.dump(rec, f, indent=1)
    print(name, "partial", len(idx), "/", n_total, flush=True)


if __name__ == "__main__":
    main()

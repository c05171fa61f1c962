"""Top-level verdict pipeline (drop-in for pkg/src/planeq/verify.py:62 verify_plan).

Same order of business as the reference: concrete shape validation, lineage
validation (tiling violations refute structurally), shape reduction, stage
construction, stage discharge, one aggregated verdict. Discharge runs on the
sm_100a witness engine: every stage of the plan is compiled into one device
image and evaluated in one launch (no worker pool, no solver processes).

Verdicts: "proven" -- every stage closed; "refuted" -- some stage has a
confirmed counterexample (an integer witness assignment plus the keyed-hash
interpretation of EXP/RSQRT/SIGMOID, replayable with exact rationals);
"unknown" -- some stage had no valid witness (all denominators vanished).
"""

from __future__ import annotations

import hashlib
import time
from dataclasses import dataclass
from typing import Any

import numpy as np

from . import field as F
from .engine import (STAGE_BAD_INDEX, STAGE_LOG_DIV0, STAGE_LOSSY, STAGE_OK, STAGE_PAR_DIV0,
                     STAGE_PROVEN, STAGE_REFUTED_CONST, Engine)
from .errors import EngineError, GraphError, PlanEqError, UncoveredNode
from .graph import validate_lineage
from .opshape import validate_concrete
from .plan import Plan
from .stages import (LoweredStage, Stage, StageResult, bound_log2, build_stages, entry_order,
                     lower_stage, shard_owner)

DEFAULT_WITNESSES = 512


@dataclass
class VerifyOptions:
    jobs: int = 1
    no_reduce: bool = False
    objective: str = "l1"
    solver_argv: list[str] | None = None
    timeout_s: float = 60.0
    no_cancel: bool = False
    strict: bool = False
    # witness engine
    witnesses: int = DEFAULT_WITNESSES
    seed: int = 0
    device: int | None = None  # None: LOCAL_RANK under torchrun, else 0
    shard: bool = True  # under torch.distributed (world > 1): split stages over the ranks


def _aggregate(results: list[StageResult], cancelled: int) -> str:
    statuses = {r.status for r in results}
    if "refuted" in statuses:
        return "refuted"
    if "unknown" in statuses or cancelled or not results:
        return "unknown"
    return "proven"


def _const_detail(lw: LoweredStage, comp) -> dict[str, Any]:
    label, idx = lw.locate(comp.info)
    both_int = comp.exact_lhs is not None and comp.exact_rhs is not None
    lv = comp.exact_lhs if comp.exact_lhs is not None else comp.const_lhs
    rv = comp.exact_rhs if comp.exact_rhs is not None else comp.const_rhs
    d = {"shard": label, "index": list(idx), "lhs_value": str(lv), "rhs_value": str(rv)}
    if both_int:
        d["reason"] = "token index mismatch"
    else:
        d["assignment"] = {}
    return d


REPLAY_TOL = 1e-6   # reference stages.py:52
REPLAY_ENVS = 8     # reference stages.py:247 (seeded candidate environments)
# after the reference's own environments: a seeded search at decreasing
# magnitudes, standing in for the reference's first candidate, the solver's
# model (stages.py:246), which a witness engine does not have
SEARCH_SCALES = (2.0, 1.0, 0.5, 0.25, 0.125)
SEARCH_PER_SCALE = 32


def replay_envs(tag: str, names: list[str], n_env: int = REPLAY_ENVS) -> np.ndarray:
    """The reference's seeded replay environments (stages.py:247-252): value of
    variable n in environment k = (sha256("tag:k:n")[:4] mod 1600 - 800) / 256."""
    out = np.empty((n_env, len(names)), dtype=np.float64)
    for k in range(n_env):
        for j, n in enumerate(names):
            h = hashlib.sha256(f"{tag}:{k}:{n}".encode()).digest()
            out[k, j] = (int.from_bytes(h[:4], "big") % 1600 - 800) / 256.0
    return out


def search_envs(tag: str, n_vars: int) -> np.ndarray:
    """Further candidate environments: uniform in [-s, s] for each search scale,
    from a generator seeded by the stage target."""
    seed = int.from_bytes(hashlib.sha256(f"{tag}:search".encode()).digest()[:8], "big")
    rng = np.random.default_rng(seed)
    return np.concatenate([rng.uniform(-s, s, size=(SEARCH_PER_SCALE, n_vars))
                           for s in SEARCH_SCALES])


def host_confirm(eng: Engine, index: int, target: str, names: list[str], witness: int):
    """pqw_confirm over the reference's environments, then the search ones.
    Returns (environments, (exact obligation, env index, replay obligation,
    lhs, rhs, obligations with an uninterpreted function))."""
    envs = np.concatenate([replay_envs(target, names), search_envs(target, len(names))])
    return envs, eng.confirm(index, witness, envs, REPLAY_TOL)


def _confirm(eng: Engine, ref, comp, first_bad: int, seed: int, source=None):
    """A field witness broke an obligation; decide what the reference reports
    (stages.py:221-264): an obligation free of uninterpreted functions that
    fails at the witness is an exact rational counterexample ("refuted",
    confirmation "exact"); otherwise the obligations with EXP/RSQRT/SIGMOID in
    their cone are replayed with the genuine functions in the reference's
    seeded environments -- a difference beyond REPLAY_TOL refutes
    (confirmation "real"), none leaves the stage "unknown" with the
    reference's reason. Returns (status, detail, note)."""
    w, obl = first_bad >> 32, first_bad & 0xFFFFFFFF
    lw = ref.lowered()
    names = [lw.var_name(j) for j in range(comp.n_vars)]
    envs, (exact, k, o2, lv, rv, n_uf) = host_confirm(eng, comp.index, ref.target, names, w)
    if exact >= 0:
        d = _witness_detail(eng, lw, comp, (w << 32) | exact, seed, source)
        d["confirmation"] = "exact"
        return "refuted", d, None
    field = {"witness": w, "obligation": obl, "field": f"F_p, p={F.P}", "seed": seed,
             "uf": "keyed-hash (field.py uf_apply)"}
    if o2 >= 0:
        label, idx = lw.locate(o2)
        support = eng.support(comp.index, o2)
        env = envs[k]
        assign = sorted((names[j], float(env[j])) for j in support)
        return "refuted", {"shard": label, "index": list(idx), "lhs_value": str(lv),
                           "rhs_value": str(rv), "assignment": {n: str(v) for n, v in assign[:16]},
                           "confirmation": "real",
                           "replay_env": (f"reference seeded environment {k}" if k < REPLAY_ENVS
                                          else f"search environment {k - REPLAY_ENVS}"),
                           "obligation": o2, "field_witness": field}, None
    return "unknown", {"reason": "countermodel failed replay confirmation",
                       "uf_obligations": n_uf, "field_witness": field}, \
        ("F_p witness differs only under the keyed-hash interpretation of "
         "EXP/RSQRT/SIGMOID; the real-valued replay did not confirm it")


def _witness_detail(engine: Engine, lw: LoweredStage, comp, first_bad: int,
                    seed: int, source=None) -> dict[str, Any]:
    w, obl = int(first_bad) >> 32, int(first_bad) & 0xFFFFFFFF
    lhs, rhs, vals = (source or EngineWitnesses(engine)).probe(comp, w, obl)
    label, idx = lw.locate(obl)
    support = engine.support(comp.index, obl)
    names = sorted((lw.var_name(i), int(vals[i])) for i in support)
    return {
        "shard": label,
        "index": list(idx),
        "lhs_value": str(lhs),
        "rhs_value": str(rhs),
        "assignment": {n: str(v) for n, v in names[:16]},
        "witness": w,
        "obligation": obl,
        "field": f"F_p, p={F.P}",
        "seed": seed,
        "uf": "keyed-hash (field.py uf_apply)",
    }


class _StageRef:
    """One stage of a discharge: its target, how to lower it on the host (for
    counterexample reports and to raise deferred lowering errors), and its
    engine compile handle (None when the host lowering raises)."""

    __slots__ = ("target", "lower", "comp", "lw", "stage")

    def __init__(self, target: str, lower, comp, lw=None, stage: int = -1):
        self.target, self.lower, self.comp, self.lw = target, lower, comp, lw
        self.stage = stage  # index in the plan's stage list

    def lowered(self) -> LoweredStage:
        if self.lw is None:
            self.lw = self.lower()
        return self.lw


class EngineWitnesses:
    """Where witness outcomes come from: the engine's device image (upload,
    one launch, results; probe re-evaluates one witness on the GPU). The one
    implementation the product uses; tests may substitute a CPU source with
    the same two methods to drive the host logic without a device."""

    def __init__(self, eng: Engine):
        self.eng = eng

    def run(self, refs, opts) -> tuple:
        t0 = time.perf_counter()
        self.eng.upload()
        t1 = time.perf_counter()
        self.eng.launch(opts.witnesses)
        fb, nv, nb = self.eng.results()
        self.times = {"upload_s": t1 - t0, "launch_results_s": time.perf_counter() - t1}
        return fb, nv, nb, self.eng.last_launch_ms()

    def probe(self, comp, w: int, obl: int):
        return self.eng.probe(comp.index, w, obl, comp.n_vars)


def _run(refs: list[_StageRef], eng: Engine, opts: VerifyOptions, host_s: float,
         stats: dict, errors: str = "raise", source=None) -> tuple[list, int, dict]:
    """Compile (pending front/back ends), launch once, and turn the engine's
    per-stage outcome into StageResults in stage order with the reference's
    cancellation (verify.py:119-122). errors="collect": a stage whose
    discharge raises yields a distributed.StageFailure in its place."""
    t0 = time.perf_counter()
    comps = [r.comp for r in refs]
    needs_gpu = any(c is not None and c.status == STAGE_OK for c in comps)
    t_front = time.perf_counter() - t0
    gpu_ms = 0.0
    fb = nv = nb = None
    source = source or EngineWitnesses(eng)
    if needs_gpu:
        fb, nv, nb, gpu_ms = source.run(refs, opts)
    t_dev = time.perf_counter() - t0
    stats["phases"] = {"front_s": round(t_front, 6), **{k: round(v, 6) for k, v in
                                                         getattr(source, "times", {}).items()}}
    n_gpu = sum(1 for c in comps if c is not None and c.status == STAGE_OK)
    per_stage = (host_s + t_dev) / max(len(refs), 1)
    results: list[StageResult] = []
    cancelled = 0
    for ref in refs:
        try:
            r = _one(ref, eng, opts, fb, nv, nb, per_stage, source)
        except PlanEqError as e:
            if errors != "collect":
                raise
            from .distributed import StageFailure
            results.append(StageFailure(e))
            continue
        results.append(r)
        if r.status == "refuted" and not opts.no_cancel:
            cancelled = len(refs) - len(results)
            break
    stats["phases"]["report_s"] = round(time.perf_counter() - t0 - t_dev, 6)
    stats.update({"gpu_ms": round(gpu_ms, 4), "gpu_stages": n_gpu, "witnesses": opts.witnesses,
                  "device_s": round(t_dev, 6)})
    if needs_gpu and isinstance(source, EngineWitnesses):
        stats.update(eng.image_stats())
    return results, cancelled, stats


def _device(opts: VerifyOptions) -> int:
    if opts.device is not None:
        return opts.device
    from .distributed import local_device
    return local_device()


def _one(ref: _StageRef, eng: Engine, opts: VerifyOptions, fb, nv, nb,
         per_stage: float, source=None) -> StageResult:
    comp = ref.comp
    if comp is None:
        ref.lowered()  # the host lowering raises the reference's exception
        raise EngineError(f"stage {ref.target}: the native lowering declined a stage "
                          "the host lowers")
    r = StageResult(ref.target, "proven", comp.obligations, comp.fast, comp.residual,
                    per_stage, degree_bound=comp.degree)
    if comp.status == STAGE_PROVEN:
        r.note = "closed by value numbering"
    elif comp.status == STAGE_REFUTED_CONST:
        r.status = "refuted"
        r.detail = _const_detail(ref.lowered(), comp)
    elif comp.status == STAGE_PAR_DIV0:
        r = StageResult(ref.target, "refuted", 0, 0, 0, per_stage,
                        {"reason": "parallel side divides by zero: "
                                   "constant denominator violates side condition"})
    elif comp.status == STAGE_LOG_DIV0:
        raise GraphError(f"stage {ref.target}: logical side divides by zero: "
                         "constant denominator violates side condition")
    elif comp.status == STAGE_BAD_INDEX:
        raise GraphError(f"stage {ref.target}: token id outside its embedding table")
    elif comp.status == STAGE_LOSSY:
        r.status = "unknown"
        r.note = ("a constant is a nonzero multiple of the field prime: evaluation in F_p "
                  "cannot decide this stage")
    else:
        i = comp.index
        r.witnesses = opts.witnesses
        r.valid_witnesses = int(nv[i])
        r.failing_witnesses = int(nb[i])
        r.false_equiv_log2 = bound_log2(comp.degree, int(nv[i]))
        if int(fb[i]) != 0xFFFFFFFFFFFFFFFF:
            r.status, r.detail, r.note = _confirm(eng, ref, comp, int(fb[i]), opts.seed, source)
        elif int(nv[i]) == 0:
            r.status = "unknown"
            r.note = "no witness kept every denominator nonzero"
    return r


def discharge(plan: Plan, stages: list[Stage], opts: VerifyOptions,
              engine: Engine | None = None, errors: str = "raise") -> tuple[list, int, dict]:
    """Run every stage (host Stage records, lowered by stages.lower_stage)
    through the witness engine; returns (results, cancelled, stats)."""
    own = engine is None
    eng = engine or Engine(_device(opts), opts.seed, F.fn_keys(opts.seed))
    try:
        t0 = time.perf_counter()
        owner = shard_owner(plan, entry_order(plan))
        refs = []
        for st in stages:
            try:
                lw = lower_stage(plan, st, owner, opts.seed)
            except PlanEqError as e:
                refs.append(_StageRef(st.target, _raiser(e), None))
                continue
            refs.append(_StageRef(st.target, None, eng.add_stage(lw.ir, lw.consts, lw.var_keys), lw))
        t_compile = time.perf_counter() - t0
        stats = {"host_path": "python", "compile_s": round(t_compile, 6)}
        return _run(refs, eng, opts, t_compile, stats, errors)
    finally:
        if own:
            eng.close()


def _raiser(exc: BaseException):
    def f():
        raise exc
    return f


def discharge_native(nplan, opts: VerifyOptions, engine: Engine | None = None,
                     which: list[int] | None = None, indices=None,
                     errors: str = "raise", source=None) -> tuple[list, int, dict]:
    """Run the stages of a NativePlan (all, or the listed indices) through the
    witness engine: lowering and compilation in C++ on host threads.
    `indices`: engine indices of every plan stage already queued into
    `engine` (NativePlan.add_stages), so nothing is lowered twice."""
    plan = nplan.plan
    own = engine is None
    eng = engine or Engine(_device(opts), opts.seed, F.fn_keys(opts.seed))
    try:
        t0 = time.perf_counter()
        sel = list(range(nplan.n_stages)) if which is None else list(which)
        if indices is None:
            idx = nplan.add_stages(eng, opts.seed, which)
        else:
            idx = np.asarray([indices[i] for i in sel], dtype=np.int32)
        targets = nplan.targets()
        owner = None
        refs = []
        for k, i in zip(idx.tolist(), sel):
            def lower(i=i):
                nonlocal owner
                if owner is None:
                    owner = shard_owner(plan, entry_order(plan))
                return lower_stage(plan, nplan.stage(i), owner, opts.seed)
            refs.append(_StageRef(targets[i], lower, eng.stage_lazy(k) if k >= 0 else None,
                                  stage=i))
        t_add = time.perf_counter() - t0
        stats = {"host_path": "native", "lower_s": round(t_add, 6)}
        return _run(refs, eng, opts, t_add, stats, errors, source)
    finally:
        if own:
            eng.close()


def _native(plan: Plan):
    """NativePlan of `plan`, or None when the native core declines it."""
    from .native import NativePlan, PlanDeclined
    try:
        return NativePlan(plan)
    except PlanDeclined:
        return None


def verify_plan(plan: Plan, opts: VerifyOptions | None = None) -> dict[str, Any]:
    """The reference's verify_plan (verify.py:62-145): validation, optional
    shape reduction, stage construction, discharge, one verdict. Stage
    construction and lowering run in the native core; the host's own checks
    run only when it declines a plan (they raise the reference's errors).

    Python's cyclic garbage collector is paused for the call: a large plan is
    millions of objects, and a full collection triggered by the report's
    allocations would traverse all of them (measured: 1-2 s outliers on
    Llama3-405B); nothing here creates reference cycles."""
    import gc
    paused = gc.isenabled()
    gc.disable()
    try:
        return _verify_plan(plan, opts)
    finally:
        if paused:
            gc.enable()


def _verify_plan(plan: Plan, opts: VerifyOptions | None) -> dict[str, Any]:
    opts = opts or VerifyOptions()
    t0 = time.perf_counter()
    times: dict[str, float] = {}
    report: dict[str, Any] = {"verdict": "unknown", "stages": [], "jobs": opts.jobs}
    if plan.parallel is None or plan.lineage is None:
        raise GraphError("plan has no parallel graph or no lineage")
    nat = _native(plan)
    times["pack_s"] = time.perf_counter() - t0
    t = time.perf_counter()
    if nat is None or not nat.validate():
        validate_concrete(plan.logical)
        validate_concrete(plan.parallel)
        nat = None  # well formed after all: the host path takes it from here
    problems = [] if nat is not None and nat.lineage_clean() else \
        validate_lineage(plan.logical, plan.parallel, plan.lineage)
    times["validate_s"] = time.perf_counter() - t
    tiling = [p for p in problems if "do not tile" in p]
    hard = [p for p in problems if "do not tile" not in p]
    if hard:
        raise GraphError("; ".join(hard))
    if tiling:
        report.update(verdict="refuted", refuted_by="structure", structure=tiling)
        report["wall_s"] = round(time.perf_counter() - t0, 6)
        return report

    work = plan
    if not opts.no_reduce:
        from .shapes import reduce_plan
        red = reduce_plan(plan, objective=opts.objective, solver_argv=opts.solver_argv,
                          timeout_s=opts.timeout_s)
        work = red.plan
        report["reduction"] = red.report
        if work is not plan:
            nat = _native(work)

    t = time.perf_counter()
    if nat is not None and nat.build_stages():
        stages = None
        uncovered = nat.uncovered()
    else:
        nat = None
        stages, uncovered = build_stages(work)
    times["build_stages_s"] = time.perf_counter() - t
    report["uncovered"] = uncovered
    loose = uncovered["parallel"] + uncovered["logical"]
    if loose:
        if opts.strict:
            raise UncoveredNode(loose)
        report["warning"] = (f"{len(loose)} node(s) feed no checkpoint and are "
                             f"not checked: {loose[:8]}")

    from .distributed import discharge_sharded, world_info
    t = time.perf_counter()
    if opts.shard and world_info()[1] > 1:
        results, cancelled, stats = discharge_sharded(work, stages, opts, nplan=nat)
    elif nat is not None:
        results, cancelled, stats = discharge_native(nat, opts)
    else:
        results, cancelled, stats = discharge(work, stages, opts)
    times["discharge_s"] = time.perf_counter() - t
    n_stages = nat.n_stages if nat is not None else len(stages)
    if nat is not None:
        nat.close()
    verdict = _aggregate(results, cancelled)
    total_ob = sum(r.obligations for r in results)
    total_fast = sum(r.fastpath for r in results)
    stats["times"] = {k: round(v, 6) for k, v in times.items()}
    report.update(
        verdict=verdict,
        stages=[r.as_dict() for r in results],
        cancelled=cancelled,
        obligations=total_ob,
        fastpath_rate=round(total_fast / total_ob, 6) if total_ob else None,
        engine=stats,
        wall_s=round(time.perf_counter() - t0, 6),
    )
    if not n_stages:
        report["note"] = "lineage has no produced checkpoints; nothing was proven"
    for r in results:
        if r.status == "refuted":
            report["counterexample"] = {"target": r.target, **(r.detail or {})}
            break
    return report

"""Binding an installed reference package (`planeq`) to this engine.

INTEGRATION.md's reference-side stub, as a module: `install(planeq.verify)`
replaces, inside the reference's own `verify_plan` (pkg/src/planeq/verify.py:62),
the per-stage `run_stage` loop (verify.py:115-126) by one discharge of the
whole plan through the native plan core and the sm_100a engine. The first
`run_stage` call for a plan discharges every stage of it (one launch) and
caches the results; each call then returns the reference's own StageResult
type for its stage. Everything else -- validation, reduction, build_stages,
the report, the verdict aggregation -- stays the reference's code.

The reference's Plan objects are packed directly (the packer reads the same
field names from any object). `source` substitutes where witness outcomes come
from (default: the engine's device image; tests pass a CPU stand-in).
"""

from __future__ import annotations

from typing import Callable


def discharge_plan(plan, opts=None, source=None) -> dict:
    """target -> this engine's StageResult for every stage of `plan`."""
    from .native import NativePlan
    from .verify import VerifyOptions, discharge_native
    opts = opts or VerifyOptions(no_cancel=True)
    nat = NativePlan(plan)
    if not nat.build_stages():
        raise ValueError(f"native plan core declined the plan: {getattr(nat, 'declined', '?')}")
    try:
        results, _cancelled, _stats = discharge_native(nat, opts, source=source)
    finally:
        nat.close()
    return {r.target: r for r in results}


def install(verify_module, opts=None, source=None) -> Callable[[], None]:
    """Serve `verify_module.run_stage` (the reference's planeq.verify) from this
    engine. Returns a function restoring the original."""
    original = verify_module.run_stage
    result_cls = verify_module.StageResult
    cache: dict = {}

    def run_stage(plan, stage, solver_argv=None, timeout_s=60.0):
        if cache.get("plan") is not plan:
            cache.clear()
            cache["plan"] = plan
            cache["results"] = discharge_plan(plan, opts, source)
        r = cache["results"][stage.target]
        return result_cls(r.target, r.status, r.obligations, r.fastpath, r.residual, r.wall_s,
                          r.detail, r.note)

    verify_module.run_stage = run_stage

    def restore():
        verify_module.run_stage = original
    return restore

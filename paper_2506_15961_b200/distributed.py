"""Multi-GPU discharge: stages are independent, so they shard across the GPUs of
one box (one process per GPU, torch.distributed) by a cost-balanced static
partition; the only collective is the gather of per-stage verdicts (and their
counterexamples) at the end -- there is no data-path exchange.

Mirrors what the reference does with its worker pool (pkg/src/planeq/verify.py:
99-126: stages fanned out to `jobs` processes, results collected in stage
order, first refutation cancels the rest): here every rank discharges its
share in one launch with cancellation off, the results are gathered, and the
reference's in-order cancellation is applied to the merged list, so the
report is identical to a single-GPU run -- including which error is raised:
a stage whose discharge raises is sent through the gather as an error record
and re-raised only if the single-GPU loop would have reached it.

Partition (native path): every rank lowers every stage and runs the compiler
front ends (cheap, identical programs compiled once), which tells the device
cost of each stage -- scheduling units of its residual cones, 0 for stages
the front end decides -- then an LPT partition of those costs; each rank
schedules, uploads and launches only its share (pqw_stage_select).
"""

from __future__ import annotations

import os
from dataclasses import replace
from typing import Callable

from . import errors as _errors
from .stages import Stage, StageResult


def stage_cost(st: Stage) -> int:
    """Static cost proxy of a host Stage record (node count of both slices);
    used only when the native core is not in play."""
    return len(st.parallel_nodes) + len(st.logical_nodes)


def partition(costs: list[int], n: int) -> list[list[int]]:
    """LPT static partition of item indices into n cost-balanced parts
    (zero-cost items are spread round-robin so every part keeps its share of
    host-side work)."""
    parts: list[list[int]] = [[] for _ in range(n)]
    load = [0] * n
    count = [0] * n
    for i in sorted(range(len(costs)), key=lambda i: (-costs[i], i)):
        k = min(range(n), key=lambda j: (load[j], count[j], j))
        parts[k].append(i)
        load[k] += costs[i]
        count[k] += 1
    return [sorted(p) for p in parts]


def world_info(group=None) -> tuple[int, int]:
    try:
        import torch.distributed as dist
    except ImportError:
        return 0, 1
    if not (dist.is_available() and dist.is_initialized()):
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def local_device() -> int:
    """The GPU a rank drives: LOCAL_RANK (torchrun) modulo the visible devices."""
    local = int(os.environ.get("LOCAL_RANK", "0"))
    try:
        from .engine import device_count
        n = device_count()
    except Exception:
        n = 0
    return local % n if n > 0 else local


def share_host_threads() -> None:
    """Ranks of one box share its host cores: unless PQW_THREADS is set, each
    rank's native plan core and compiler use cores / local world size."""
    if "PQW_THREADS" in os.environ:
        return
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
    if local_world > 1:
        try:
            cores = len(os.sched_getaffinity(0))
        except (AttributeError, OSError):
            cores = os.cpu_count() or 1
        os.environ["PQW_THREADS"] = str(max(1, cores // local_world))


class StageFailure:
    """A stage whose discharge raised, as sent through the gather."""

    def __init__(self, exc: BaseException):
        self.cls = type(exc).__name__
        self.module = type(exc).__module__
        self.msg = str(exc)

    def exception(self) -> BaseException:
        cls = getattr(_errors, self.cls, None) if self.module == _errors.__name__ else None
        if cls is None or not (isinstance(cls, type) and issubclass(cls, BaseException)):
            return RuntimeError(f"{self.cls}: {self.msg}")
        exc = cls.__new__(cls)
        Exception.__init__(exc, self.msg)
        return exc

    def __repr__(self):
        return f"StageFailure({self.cls}: {self.msg})"


def merge_results(per_rank: list[list[tuple[int, dict]]], n_stages: int,
                  no_cancel: bool) -> tuple[list[StageResult], int]:
    """Stage-ordered results from the ranks' (stage index, result) lists; the
    first refuted stage cancels the rest unless no_cancel (reference
    verify.py:111-122). A failure record re-raises its exception when the
    single-GPU loop would have reached that stage."""
    slots: list = [None] * n_stages
    for payload in per_rank:
        for i, d in payload:
            slots[i] = d if isinstance(d, StageFailure) else StageResult(**d)
    if any(s is None for s in slots):
        raise RuntimeError("a stage is missing from the gathered results")
    results: list[StageResult] = []
    for r in slots:
        if isinstance(r, StageFailure):
            raise r.exception()
        results.append(r)
        if r.status == "refuted" and not no_cancel:
            return results, n_stages - len(results)
    return results, 0


def _native_share(nplan, opts, rank: int, world: int):
    """Cost every stage (front ends), take this rank's LPT share, discharge it.
    Returns ([(stage index, result | StageFailure)], stats, parts)."""
    from . import field as F
    from .engine import Engine
    from .verify import discharge_native
    eng = Engine(opts.device, opts.seed, F.fn_keys(opts.seed))
    try:
        idx = nplan.add_stages(eng, opts.seed)
        costs = [eng.cost(int(k)) if k >= 0 else 0 for k in idx]
        parts = partition(costs, world)
        mine = parts[rank]
        flags = [0] * len(idx)
        for i in mine:
            if idx[i] >= 0:
                flags[int(idx[i])] = 1
        eng.select(flags[: eng.n_stages])
        local, _, stats = discharge_native(nplan, replace(opts, no_cancel=True), engine=eng,
                                           which=mine, indices=idx, errors="collect")
    finally:
        eng.close()
    stats["stage_costs_local"] = sum(costs[i] for i in mine)
    return list(zip(mine, local)), stats, parts


def discharge_sharded(plan, stages: list[Stage] | None, opts, group=None,
                      discharge_fn: Callable | None = None, nplan=None):
    """This rank's share of the stages, then an all_gather of the results.
    Returns (results, cancelled, stats) like verify.discharge, identical on
    every rank. With `nplan` (a NativePlan) the share is chosen by front-end
    device cost; otherwise by the host Stage records' node counts and
    discharged by `discharge_fn` (default: the GPU engine's host path)."""
    import torch.distributed as dist
    rank, world = world_info(group)
    if opts.device is None:
        opts = replace(opts, device=local_device())
    share_host_threads()
    if nplan is not None:
        pairs, stats, parts = _native_share(nplan, opts, rank, world)
        n_stages = nplan.n_stages
    else:
        if discharge_fn is None:
            from functools import partial
            from .verify import discharge
            discharge_fn = partial(discharge, errors="collect")
        parts = partition([stage_cost(s) for s in stages], world)
        mine = parts[rank]
        try:
            local, _, stats = discharge_fn(plan, [stages[i] for i in mine],
                                           replace(opts, no_cancel=True))
            pairs = list(zip(mine, local))
        except Exception as e:  # noqa: BLE001 - re-raised in stage order after the gather
            fail = StageFailure(e)
            pairs = [(i, fail) for i in mine]
            stats = {"error": repr(fail)}
        n_stages = len(stages)
    payload = [(i, r if isinstance(r, StageFailure) else r.as_dict()) for i, r in pairs]
    if dist.get_backend(group) == "nccl":
        # all_gather_object stages the pickles on the current CUDA device
        import torch
        torch.cuda.set_device(opts.device)
    gathered: list = [None] * world
    dist.all_gather_object(gathered, (payload, stats), group=group)
    results, cancelled = merge_results([g[0] for g in gathered], n_stages, opts.no_cancel)
    rank_stats = [g[1] for g in gathered]
    merged = {"ranks": world, "gpu_ms_max": max(s.get("gpu_ms", 0.0) for s in rank_stats),
              "gpu_stages": sum(s.get("gpu_stages", 0) for s in rank_stats),
              "stages_per_rank": [len(p) for p in parts], "per_rank": rank_stats,
              "host_path": rank_stats[0].get("host_path")}
    return results, cancelled, merged

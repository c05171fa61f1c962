"""Multi-GPU discharge: stages are independent, so they shard across the GPUs of
one box (one process per GPU, torch.distributed) by a cost-balanced static
partition; the only collective is the gather of per-stage verdicts (and their
counterexamples) at the end -- there is no data-path exchange.

Mirrors what the reference does with its worker pool (pkg/src/planeq/verify.py:
99-126: stages fanned out to `jobs` processes, results collected in stage
order, first refutation cancels the rest): here every rank discharges its
share in one launch with cancellation off, the results are gathered, and the
reference's in-order cancellation is applied to the merged list, so the
report is identical to a single-GPU run.
"""

from __future__ import annotations

from dataclasses import asdict, replace
from typing import Callable

from .stages import Stage, StageResult


def stage_cost(st: Stage) -> int:
    """Static cost proxy of a stage: nodes on both sides (the bytecode length
    is known only after compilation; node counts track it closely)."""
    return len(st.parallel_nodes) + len(st.logical_nodes)


def partition(costs: list[int], n: int) -> list[list[int]]:
    """LPT static partition of item indices into n cost-balanced parts."""
    parts: list[list[int]] = [[] for _ in range(n)]
    load = [0] * n
    for i in sorted(range(len(costs)), key=lambda i: (-costs[i], i)):
        k = min(range(n), key=lambda j: (load[j], j))
        parts[k].append(i)
        load[k] += costs[i]
    return [sorted(p) for p in parts]


def world_info(group=None) -> tuple[int, int]:
    try:
        import torch.distributed as dist
    except ImportError:
        return 0, 1
    if not (dist.is_available() and dist.is_initialized()):
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def merge_results(per_rank: list[list[tuple[int, dict]]], n_stages: int,
                  no_cancel: bool) -> tuple[list[StageResult], int]:
    """Stage-ordered results from the ranks' (stage index, result) lists; the
    first refuted stage cancels the rest unless no_cancel (reference
    verify.py:111-122)."""
    slots: list[StageResult | None] = [None] * n_stages
    for payload in per_rank:
        for i, d in payload:
            slots[i] = StageResult(**d)
    if any(s is None for s in slots):
        raise RuntimeError("a stage is missing from the gathered results")
    results: list[StageResult] = []
    for r in slots:
        results.append(r)
        if r.status == "refuted" and not no_cancel:
            return results, n_stages - len(results)
    return results, 0


def discharge_sharded(plan, stages: list[Stage], opts, group=None,
                      discharge_fn: Callable | None = None):
    """This rank's share of `stages` through `discharge_fn` (default: the GPU
    engine), then an all_gather of the results. Returns (results, cancelled,
    stats) like verify.discharge, identical on every rank."""
    import torch.distributed as dist
    if discharge_fn is None:
        from .verify import discharge as discharge_fn
    rank, world = world_info(group)
    parts = partition([stage_cost(s) for s in stages], world)
    mine = parts[rank]
    local, _, stats = discharge_fn(plan, [stages[i] for i in mine], replace(opts, no_cancel=True))
    payload = [(i, asdict(r)) for i, r in zip(mine, local)]
    gathered: list = [None] * world
    dist.all_gather_object(gathered, (payload, stats), group=group)
    results, cancelled = merge_results([g[0] for g in gathered], len(stages), opts.no_cancel)
    rank_stats = [g[1] for g in gathered]
    merged = {"ranks": world, "gpu_ms_max": max(s.get("gpu_ms", 0.0) for s in rank_stats),
              "gpu_stages": sum(s.get("gpu_stages", 0) for s in rank_stats),
              "stages_per_rank": [len(p) for p in parts], "per_rank": rank_stats}
    return results, cancelled, merged

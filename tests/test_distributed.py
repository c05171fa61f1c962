"""Multi-rank discharge on CPU (gloo, world_size 2): the cost-balanced stage
partition plus the verdict gather reproduce the single-process report exactly,
including the reference's in-order cancellation. The per-rank discharge is
the CPU oracle here (test infrastructure); on GPUs it is the engine."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from golden_io import load_plan, verdicts
from paper_2506_15961_b200.distributed import merge_results, partition, stage_cost
from paper_2506_15961_b200.stages import StageResult, build_stages, entry_order, shard_owner


def oracle_discharge(plan, stages, opts):
    """Test-only stand-in for verify.discharge: oracle verdicts per stage."""
    from oracle.stage_check import check_stage
    owner = shard_owner(plan, entry_order(plan))
    wit = np.arange(16, dtype=np.uint64)
    out = []
    for st in stages:
        o = check_stage(plan, st, owner, 3, wit)
        out.append(StageResult(st.target, o.status, 0, 0, 0, 0.0,
                               detail={"first_bad": list(o.first_bad)} if o.first_bad else None))
    return out, 0, {"gpu_ms": float(len(stages)), "gpu_stages": len(stages)}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, plan_name, no_cancel, q):
    import torch.distributed as dist
    from paper_2506_15961_b200.distributed import discharge_sharded
    from paper_2506_15961_b200.verify import VerifyOptions
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = load_plan(plan_name)
        stages, _ = build_stages(plan)
        res, cancelled, stats = discharge_sharded(plan, stages, VerifyOptions(no_cancel=no_cancel),
                                                  discharge_fn=oracle_discharge)
        q.put((rank, [(r.target, r.status, r.detail) for r in res], cancelled,
               stats["stages_per_rank"]))
    finally:
        dist.destroy_process_group()


def test_partition_is_balanced_and_complete():
    costs = [50, 7, 7, 30, 1, 22, 22, 9, 3, 40]
    parts = partition(costs, 3)
    assert sorted(i for p in parts for i in p) == list(range(len(costs)))
    loads = [sum(costs[i] for i in p) for p in parts]
    assert max(loads) - min(loads) <= max(costs)
    assert partition(costs, 1) == [list(range(len(costs)))]


def test_merge_applies_in_order_cancellation():
    mk = lambda t, s: {"target": t, "status": s, "obligations": 0, "fastpath": 0,  # noqa: E731
                       "residual": 0, "wall_s": 0.0}
    per_rank = [[(0, mk("a", "proven")), (3, mk("d", "refuted"))],
                [(1, mk("b", "refuted")), (2, mk("c", "proven"))]]
    res, cancelled = merge_results(per_rank, 4, no_cancel=False)
    assert [r.target for r in res] == ["a", "b"] and cancelled == 2
    res, cancelled = merge_results(per_rank, 4, no_cancel=True)
    assert [r.status for r in res] == ["proven", "refuted", "proven", "refuted"] and cancelled == 0


PICK = [r for r in verdicts() if r["name"] in ("tp2", "dp2tp2pp2nm2.wrong_scaling.8")]


@pytest.mark.parametrize("no_cancel", [True, False])
@pytest.mark.parametrize("rec", PICK, ids=[r["name"] for r in PICK])
def test_two_rank_gloo_discharge_matches_single_process(rec, no_cancel):
    plan = load_plan(rec["work_plan"])
    stages, _ = build_stages(plan)
    single, _, _ = oracle_discharge(plan, stages, None)
    want, want_cancelled = merge_results([[(i, r.__dict__) for i, r in enumerate(single)]],
                                         len(stages), no_cancel)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, rec["work_plan"], no_cancel, q))
             for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, res, cancelled, per_rank in got:
        assert res == [(r.target, r.status, r.detail) for r in want], rank
        assert cancelled == want_cancelled
        assert sum(per_rank) == len(stages) and min(per_rank) > 0
    assert stage_cost(stages[0]) > 0


def _native_worker(rank, world, port, plan_name, q):
    """One rank of the product's native partition (distributed._native_share up
    to the discharge): lower every stage, cost it with the compiler front end,
    LPT-partition the costs, select this rank's share."""
    import torch.distributed as dist
    from paper_2506_15961_b200 import field as F
    from paper_2506_15961_b200.engine import STAGE_OK, Engine
    from paper_2506_15961_b200.native import NativePlan
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = load_plan(plan_name)
        nat = NativePlan(plan)
        assert nat.validate() and nat.build_stages()
        eng = Engine(0, 3, F.fn_keys(3))
        idx = nat.add_stages(eng, 3)
        costs = [eng.cost(int(k)) for k in idx]
        ok = [eng.stage_status(int(k)).status == STAGE_OK for k in idx]
        parts = partition(costs, world)
        flags = [0] * eng.n_stages
        for i in parts[rank]:
            flags[int(idx[i])] = 1
        eng.select(flags)
        st = eng.image_stats()  # back ends of the selected share only
        gathered = [None] * world
        dist.all_gather_object(gathered, parts)
        q.put((rank, parts, gathered, costs, ok, st["gpu_stages"]))
        eng.close()
    finally:
        dist.destroy_process_group()


def test_two_rank_native_partition_is_consistent():
    """gloo, world size 2: every rank derives the same partition of the native
    plan's stages from front-end device costs (decided stages cost 0), the
    shares are disjoint and complete, and each rank schedules only the
    GPU stages of its own share."""
    rec = next(r for r in verdicts() if r["name"] == "dp2tp2pp2nm2")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_native_worker, args=(r, 2, port, rec["work_plan"], q))
             for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    out.sort()
    (_, p0, g0, c0, ok0, n0), (_, p1, g1, c1, ok1, n1) = out
    assert g0 == g1 == [p0, p1]
    assert sorted(p0[0] + p0[1]) == list(range(len(c0)))
    assert c0 == c1 and ok0 == ok1
    assert all((c > 0) == o for c, o in zip(c0, ok0))
    assert n0 == sum(1 for i in p0[0] if ok0[i]) and n1 == sum(1 for i in p0[1] if ok0[i])


def test_merge_raises_failures_in_stage_order():
    """A stage whose discharge raised on some rank re-raises after the gather
    only when the single-GPU loop would have reached it (reference
    verify.py:115-126: the first refutation stops the loop unless no_cancel)."""
    from paper_2506_15961_b200.distributed import StageFailure
    from paper_2506_15961_b200.errors import GraphError

    def res(t, status):
        return StageResult(t, status, 1, 0, 1, 0.0).as_dict()

    fail = StageFailure(GraphError("stage s2: logical side divides by zero"))
    # rank 0 owns stages 0 and 2, rank 1 owns 1 and 3
    late = [[(0, res("s0", "proven")), (2, fail)], [(1, res("s1", "refuted")), (3, res("s3", "proven"))]]
    results, cancelled = merge_results(late, 4, no_cancel=False)
    assert [r.status for r in results] == ["proven", "refuted"] and cancelled == 2
    with pytest.raises(GraphError, match="divides by zero"):
        merge_results(late, 4, no_cancel=True)
    early = [[(0, fail), (2, res("s2", "proven"))], [(1, res("s1", "refuted")), (3, res("s3", "proven"))]]
    with pytest.raises(GraphError):
        merge_results(early, 4, no_cancel=False)

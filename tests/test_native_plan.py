"""The native plan core (csrc/plan.cpp behind pqw_plan_*) against the host code it
replaces on the verify path: opshape.validate_concrete, stages.build_stages and
stages.lower_stage (which restate the reference's shapes.py:35-45,
stages.py:79-176 and :267-340).

On every golden plan (the reference's toy/fault/random corpus, the Llama and
DeepSeek families): the same stages (targets, slices in topological order,
boundaries, assumed checkpoints, owned nodes, uncovered nodes) and, word for
word, the same tensor-op program, constant table and variable keys per stage.
On malformed plans: the native core declines, and verify_plan raises the
reference's exception (the host checks run on the declined plan).
"""

import copy
import dataclasses
import json
import os

import numpy as np
import pytest

from golden_io import GOLDEN, load_plan, verdicts
from paper_2506_15961_b200.errors import (CycleError, DanglingTensorError, GraphError,
                                          PlanFormatError, ShapeError, UnknownOperator)
from paper_2506_15961_b200.graph import Node, Tensor
from paper_2506_15961_b200.native import NativePlan
from paper_2506_15961_b200.opshape import validate_concrete
from paper_2506_15961_b200.stages import build_stages, entry_order, lower_stage, shard_owner
from paper_2506_15961_b200.verify import VerifyOptions, verify_plan


def _golden_plans():
    out = [(r["name"], r["work_plan"]) for r in verdicts() if r.get("work_plan")]
    for fname in ("verdicts_llama.json", "verdicts_deepseek.json"):
        p = os.path.join(GOLDEN, fname)
        if os.path.exists(p):
            out += [(r["name"], r["plan"]) for r in json.load(open(p))["plans"]]
    return out


PLANS = _golden_plans()


def _python_ok(fn, *a):
    try:
        return True, fn(*a)
    except Exception as e:  # noqa: BLE001
        return False, e


@pytest.mark.parametrize("name,rel", PLANS, ids=[n for n, _ in PLANS])
def test_native_stages_and_programs_match_host(lib, name, rel):
    _check_against_host(load_plan(rel), name)


@pytest.mark.parametrize("name,rel", PLANS[:6], ids=[n for n, _ in PLANS[:6]])
def test_native_core_on_back_to_front_node_order(lib, name, rel):
    """Both graphs' node lists reversed (still acyclic, but producers now follow
    their consumers): the validation and slice-order fast paths for
    front-to-back graphs do not apply, and the stages and programs still equal
    the host's."""
    plan = load_plan(rel)
    plan.logical.nodes.reverse()
    plan.parallel.nodes.reverse()
    _check_against_host(plan, name)


def _check_against_host(plan, name):
    nat = NativePlan(plan)
    ok_py = all(_python_ok(validate_concrete, g)[0] for g in (plan.logical, plan.parallel))
    assert nat.validate() == ok_py, name
    from paper_2506_15961_b200.graph import validate_lineage
    assert nat.lineage_clean() == (validate_lineage(plan.logical, plan.parallel,
                                                    plan.lineage) == []), name
    ok, got = _python_ok(build_stages, plan)
    assert nat.build_stages() == ok, (name, got)
    if not ok:
        return
    stages, unc = got
    nst = nat.stages()
    assert [s.target for s in nst] == [s.target for s in stages]
    for a, b in zip(stages, nst):
        assert [n.id for n in a.logical_nodes] == [n.id for n in b.logical_nodes], a.target
        assert [n.id for n in a.parallel_nodes] == [n.id for n in b.parallel_nodes], a.target
        assert (a.l_inputs, a.p_inputs, a.assumed) == (b.l_inputs, b.p_inputs, b.assumed)
        assert (a.owned_logical, a.owned_parallel) == (b.owned_logical, b.owned_parallel)
    assert nat.uncovered() == unc
    owner = shard_owner(plan, entry_order(plan))
    for i, st in enumerate(stages):
        seed = 11 + i
        ok, lw = _python_ok(lower_stage, plan, st, owner, seed)
        if not ok:
            with pytest.raises(Exception):
                nat.stage_program(i, seed)
            continue
        ir, cs, vk = nat.stage_program(i, seed)
        assert np.array_equal(ir, lw.ir), st.target
        assert np.array_equal(cs, lw.consts.reshape(-1, 3)), st.target
        assert np.array_equal(vk, lw.var_keys), st.target
    nat.close()


def _base():
    rec = next(r for r in verdicts() if r["name"] == "tp2")
    return load_plan(rec["work_plan"])


def _first(g, kind):
    return next(i for i, n in enumerate(g.nodes) if n.kind == kind)


def _mutations():
    def shape(plan):
        g = plan.parallel
        n = g.nodes[_first(g, "matmul")]
        t = g.tensors[n.outputs[0]]
        g.tensors[t.id] = Tensor(t.id, tuple(t.shape[:-1]) + (t.shape[-1] + 1,), t.role, t.dtype,
                                 t.device, t.microbatch, dict(t.meta))
        return ShapeError

    def unknown(plan):
        g = plan.logical
        i = _first(g, "add")
        g.nodes[i] = copy.replace(g.nodes[i], kind="frobnicate") if hasattr(copy, "replace") \
            else Node(g.nodes[i].id, "frobnicate", g.nodes[i].inputs, g.nodes[i].outputs,
                      dict(g.nodes[i].attrs), g.nodes[i].device, g.nodes[i].seq)
        return UnknownOperator

    def dangling(plan):
        g = plan.parallel
        i = _first(g, "mul")
        n = g.nodes[i]
        g.tensors["ghost"] = Tensor("ghost", g.tensors[n.inputs[0]].shape)
        g.nodes[i] = Node(n.id, n.kind, ("ghost",) + tuple(n.inputs[1:]), n.outputs,
                          dict(n.attrs), n.device, n.seq)
        return DanglingTensorError

    def cycle(plan):
        g = plan.logical
        i = _first(g, "add")
        n = g.nodes[i]
        later = next(m for m in g.nodes[i + 1:] if m.kind in ("add", "mul")
                     and g.tensors[m.outputs[0]].shape == g.tensors[n.inputs[0]].shape)
        g.nodes[i] = Node(n.id, n.kind, (later.outputs[0],) + tuple(n.inputs[1:]), n.outputs,
                          dict(n.attrs), n.device, n.seq)
        return (CycleError, GraphError)

    def twice(plan):
        g = plan.parallel
        a = g.nodes[_first(g, "mul")]
        b = next(m for m in g.nodes if m.kind == "add")
        i = g.nodes.index(b)
        g.nodes[i] = Node(b.id, b.kind, b.inputs, a.outputs, dict(b.attrs), b.device, b.seq)
        return (PlanFormatError, GraphError, ShapeError)

    return {"shape": shape, "unknown": unknown, "dangling": dangling, "cycle": cycle,
            "twice": twice}


@pytest.mark.parametrize("kind", sorted(_mutations()))
def test_malformed_plans_are_declined_and_raise_the_host_error(lib, kind):
    plan = _base()
    want = _mutations()[kind](plan)
    nat = NativePlan(plan)
    declined = not nat.validate() or not nat.build_stages()
    assert declined, kind
    with pytest.raises(want):
        verify_plan(plan, VerifyOptions(no_reduce=True))


def test_verify_plan_reports_stage_errors_of_the_host(lib):
    """A graph input without a checkpoint entry: the native build declines and
    the host's build_stages raises its GraphError."""
    plan = _base()
    victim = next(t for t in plan.logical.inputs if t in plan.lineage)
    del plan.lineage[victim]
    nat = NativePlan(plan)
    assert nat.validate()
    assert not nat.build_stages()
    with pytest.raises(GraphError):
        build_stages(plan)


@pytest.mark.parametrize("name,rel", PLANS[:8] + PLANS[-4:], ids=[n for n, _ in PLANS[:8] + PLANS[-4:]])
def test_cpp_packer_matches_python_packer(lib, name, rel):
    """csrc/pack.cpp (the _pqw_pack extension) emits the columns of native.py's
    Python packer, byte for byte, for both graphs."""
    from paper_2506_15961_b200 import native as N
    ext = N._ext()
    assert ext is not None, "the _pqw_pack extension is not built"
    plan = load_plan(rel)
    for g in (plan.logical, plan.parallel):
        c1, c2 = N._Consts(), N._Consts()
        got, cnt = N._pack_columns(g, c1)
        try:
            N._ext = lambda: None
            want, cnt2 = N._pack_columns(g, c2)
        finally:
            N._ext = lambda: ext
        assert cnt == cnt2
        assert c1.triples == c2.triples
        for k in want:
            if k == "consts":
                continue
            a, b = got[k], want[k]
            if isinstance(b, bytes):
                assert a == b, (name, k)
            else:
                assert np.array_equal(np.asarray(a), np.asarray(b)), (name, k)
    got = N._lineage_columns(plan.lineage)
    try:
        N._ext = lambda: None
        want = N._lineage_columns(plan.lineage)
    finally:
        N._ext = lambda: ext
    if not plan.lineage:  # the Python columns pad empty arrays to one element
        want = tuple(w[:0] if isinstance(w, np.ndarray) else w for w in want)
    for a, b in zip(got[:4], want[:4]):
        assert np.array_equal(a, b), name
    assert got[4] == want[4], name


def test_parallel_packer_matches_serial_packer(lib):
    """The threaded fast path of csrc/pack.cpp (large graphs) emits exactly the
    serial path's columns and constant numbering."""
    from paper_2506_15961_b200 import native as N
    from paper_2506_15961_b200.stages import OPCODE
    from paper_2506_15961_b200.workloads import get_workload
    ext = N._ext()
    _d, plan = get_workload("llama3-8b-tp4pp2dp2-sp")
    assert len(plan.parallel.nodes) + len(plan.parallel.tensors) > 50000  # threads engage
    for g in (plan.logical, plan.parallel):
        c1, c2 = N._Consts(), N._Consts()
        fast = ext.pack_graph(g, OPCODE, c1)
        os.environ["PQW_PACK_SERIAL"] = "1"
        try:
            serial = ext.pack_graph(g, OPCODE, c2)
        finally:
            del os.environ["PQW_PACK_SERIAL"]
        assert fast == serial
        assert c1.triples == c2.triples


def _lineage_mutations():
    from paper_2506_15961_b200.graph import LineageEntry, Shard

    def first_split(plan):
        return next(t for t, e in plan.lineage.items()
                    if len({s.ranges for s in e.shards}) > 1)

    def overlap(plan):
        t = first_split(plan)
        e = plan.lineage[t]
        r0 = e.shards[0].ranges
        shards = (Shard(e.shards[0].tensor, r0),) + tuple(Shard(s.tensor, r0) for s in e.shards[1:])
        plan.lineage[t] = LineageEntry(e.logical, e.mode, shards)

    def unknown_shard(plan):
        t = first_split(plan)
        e = plan.lineage[t]
        plan.lineage[t] = LineageEntry(e.logical, e.mode,
                                       (Shard("no-such-tensor", e.shards[0].ranges),) + e.shards[1:])

    def bad_mode(plan):
        t = first_split(plan)
        e = plan.lineage[t]
        plan.lineage[t] = LineageEntry(e.logical, "mirrored", e.shards)

    def out_of_bounds(plan):
        t = first_split(plan)
        e = plan.lineage[t]
        (lo, hi), rest = e.shards[0].ranges[0], e.shards[0].ranges[1:]
        shards = (Shard(e.shards[0].tensor, ((lo + 100, hi + 100),) + rest),) + e.shards[1:]
        plan.lineage[t] = LineageEntry(e.logical, e.mode, shards)
    return {"overlap": overlap, "unknown_shard": unknown_shard, "bad_mode": bad_mode,
            "out_of_bounds": out_of_bounds}


@pytest.mark.parametrize("kind", sorted(_lineage_mutations()))
def test_lineage_check_matches_host(lib, kind):
    """pqw_plan_check_lineage flags exactly the plans validate_lineage flags."""
    from paper_2506_15961_b200.graph import validate_lineage
    plan = _base()
    _lineage_mutations()[kind](plan)
    nat = NativePlan(plan)
    assert validate_lineage(plan.logical, plan.parallel, plan.lineage)
    assert not nat.lineage_clean()


def test_batched_queue_dedups_like_per_stage_add(lib):
    """pqw_plan_add_stages groups equal programs itself (hashing and comparing
    on host threads, then handing the engine the verified duplicate); the
    engine must end up as if every stage had gone through pqw_stage_add one by
    one -- same statuses, same number of distinct programs -- also when a
    second batch lands on programs the engine already holds."""
    from paper_2506_15961_b200 import field as F
    from paper_2506_15961_b200.engine import Engine
    from paper_2506_15961_b200.workloads import get_workload
    _, plan = get_workload("llama3-8b-tp4pp2dp2-sp")
    nat = NativePlan(plan)
    assert nat.validate() and nat.build_stages()
    n, seed = nat.n_stages, 5
    one = Engine(0, 0, F.fn_keys(0))
    for i in range(n):
        ir, cs, vk = nat.stage_program(i, seed)
        one.add_stage(ir, cs, vk)
    batch = Engine(0, 0, F.fn_keys(0))
    ia = nat.add_stages(batch, seed)
    split = Engine(0, 0, F.fn_keys(0))
    ib = np.concatenate([nat.add_stages(split, seed, list(range(0, n, 2))),
                         nat.add_stages(split, seed, list(range(1, n, 2)))])
    order = list(range(0, n, 2)) + list(range(1, n, 2))
    assert list(ia) == list(range(n)) and sorted(ib) == list(range(n))
    def st(e, i):
        return dataclasses.replace(e.stage_status(i), index=0)
    want = [st(one, i) for i in range(n)]
    assert [st(batch, i) for i in range(n)] == want
    assert [st(split, int(ib[k])) for k in np.argsort(order)] == want
    s1, s2, s3 = one.image_stats(), batch.image_stats(), split.image_stats()
    assert s1["cache_hits"] == s2["cache_hits"] == s3["cache_hits"] > n // 2
    for e in (one, batch, split):
        e.close()
    nat.close()


def test_native_core_in_a_forked_child(lib, monkeypatch):
    """The library's host thread pool does not survive fork(); a child process
    (e.g. a fork-based worker pool around verify_plan) gets a pool of its own
    instead of waiting on the parent's workers forever."""
    import signal
    import time
    monkeypatch.setenv("PQW_THREADS", "4")
    plan = _base()

    def run():
        nat = NativePlan(plan)
        ok = nat.validate() and nat.build_stages()
        n = nat.n_stages
        nat.close()
        return ok, n

    want = run()  # the parent's pool now has parked workers
    pid = os.fork()
    if pid == 0:  # child: must finish, with the same stages
        signal.alarm(60)
        try:
            os._exit(0 if run() == want else 1)
        except BaseException:  # noqa: BLE001
            os._exit(2)
    deadline = time.time() + 90
    while True:
        done, status = os.waitpid(pid, os.WNOHANG)
        if done:
            break
        if time.time() > deadline:
            os.kill(pid, signal.SIGKILL)
            os.waitpid(pid, 0)
            raise AssertionError("native core hung in a forked child")
        time.sleep(0.05)
    assert os.WIFEXITED(status) and os.WEXITSTATUS(status) == 0, status

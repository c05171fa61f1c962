"""CPU check of the host compiler: compiled bytecode, emulated in numpy
(tests/bytecode_emu.py), must reproduce the oracle's per-witness outcome on
every stage of the golden work plans. Runs without a GPU."""

import os

import numpy as np
import pytest

import bytecode_emu
from golden_io import GOLDEN, load_plan, verdicts
from oracle.stage_check import check_stage
from paper_2506_15961_b200 import field as F
from paper_2506_15961_b200.engine import STAGE_OK, STAGE_PROVEN, STAGE_REFUTED_CONST, Engine
from paper_2506_15961_b200.stages import build_stages, entry_order, lower_stage, shard_owner

RECS = [r for r in verdicts() if "work_plan" in r] if os.path.exists(
    os.path.join(GOLDEN, "verdicts.json")) else []
PICK = [r for r in RECS if r["meta"]["source"] != "random_plan"][:10] + \
    [r for r in RECS if r["meta"]["source"] == "random_plan"][:10]


@pytest.mark.parametrize("rec", PICK, ids=[r["name"] for r in PICK])
def test_bytecode_matches_oracle(lib, rec):
    seed, W = 5, 8
    plan = load_plan(rec["work_plan"])
    stages, _ = build_stages(plan)
    owner = shard_owner(plan, entry_order(plan))
    eng = Engine(0, seed, F.fn_keys(seed))
    wit = np.arange(W, dtype=np.uint64)
    base = 0
    for st in stages:
        lw = lower_stage(plan, st, owner, seed)
        c = eng.add_stage(lw.ir, lw.consts, lw.var_keys)
        o = check_stage(plan, st, owner, seed, wit)
        if c.status == STAGE_OK:
            code, ns = eng.bytecode(c.index)
            policy = ("random", "ahead", "behind")[c.index % 3]
            valid, bad = bytecode_emu.run(code, ns, lw.var_keys, base, seed, wit,
                                          n_warps=16, policy=policy, rng_seed=c.index)
            assert int(valid.sum()) == o.valid, st.target
            emu_bad = (bad >= 0) & valid
            want = o.bad_mask.any(axis=0) if o.bad_mask is not None else np.zeros(W, bool)
            assert np.array_equal(emu_bad, want), st.target
            if o.first_bad is not None:
                w = int(np.argmax(emu_bad))
                assert (w, int(bad[w])) == o.first_bad
        elif c.status == STAGE_PROVEN:
            assert o.status == "proven", st.target
        elif c.status == STAGE_REFUTED_CONST:
            assert o.status == "refuted", st.target
        base += lw.var_keys.size
    eng.close()


SPILL_PICK = [r for r in RECS if r["meta"]["source"] != "random_plan"][:4]


@pytest.mark.parametrize("warps,slots", [(8, 48), (16, 64)])
@pytest.mark.parametrize("rec", SPILL_PICK, ids=[r["name"] for r in SPILL_PICK])
def test_small_value_file_spills_correctly(lib, rec, warps, slots, monkeypatch):
    """A tiny shared value file forces the allocator to keep values in global
    memory (FILL/SPILL) and the warps to synchronise on spill slots too."""
    monkeypatch.setenv("PQW_FAST_SLOTS", str(slots))
    monkeypatch.setenv("PQW_WARPS", str(warps))
    seed, W = 7, 4
    plan = load_plan(rec["work_plan"])
    stages, _ = build_stages(plan)
    owner = shard_owner(plan, entry_order(plan))
    eng = Engine(0, seed, F.fn_keys(seed))
    wit = np.arange(W, dtype=np.uint64)
    spilled = 0
    for st in stages:
        lw = lower_stage(plan, st, owner, seed)
        c = eng.add_stage(lw.ir, lw.consts, lw.var_keys)
        if c.status != STAGE_OK:
            continue
        o = check_stage(plan, st, owner, seed, wit)
        code, ns = eng.bytecode(c.index)
        assert ns <= slots
        spilled += any(ins[0] == "FILL" for stream in bytecode_emu.decode(code, warps)
                       for ins in stream)
        for policy in ("ahead", "behind", "random"):
            valid, bad = bytecode_emu.run(code, ns, lw.var_keys, 0, seed, wit, n_warps=warps,
                                          policy=policy, rng_seed=c.index)
            assert int(valid.sum()) == o.valid, (st.target, policy)
            emu_bad = (bad >= 0) & valid
            want = o.bad_mask.any(axis=0) if o.bad_mask is not None else np.zeros(W, bool)
            assert np.array_equal(emu_bad, want), (st.target, policy)
    assert spilled, "expected at least one stage to spill"
    eng.close()

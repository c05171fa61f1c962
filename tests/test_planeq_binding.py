"""The drop-in proven against the real `planeq` (build container only).

The INTEGRATION.md binding (paper_2506_15961_b200/planeq_binding.py) is
installed into the reference package's own `verify_plan`
(pkg/src/planeq/verify.py:62), replacing its run_stage loop; the reference's
Plan objects go straight into the native plan core. The report the reference
then produces must agree per stage with the reference's own golden verdicts
wherever the reference decides, and equal this package's verify_plan on the
same plan stage for stage.

There is no GPU in the build container, so the witness outcomes come from a
CPU stand-in for the engine's device image (the oracle: test infrastructure,
proven bit-identical to the GPU by tests/test_gpu_parity.py and
test_workload_parity.py); everything else -- packing, validation, stage
construction, lowering, compilation, confirmation, the verdict mapping -- is
the product path.
"""

import gzip
import os
import sys

import numpy as np
import pytest

from golden_io import GOLDEN, load_plan, verdicts

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources not present")

NAMES = ("tp2", "dp2tp2pp2nm2", "dp2tp2pp2nm2.wrong_scaling.8", "dp2tp2pp2nm2.bad_partition.6",
         "dp2tp2pp2nm2.shuffled_microbatch.10", "dp2tp2pp2nm2.extra_op.16", "tp2pp2", "rnd3",
         "rnd7")


class OracleWitnesses:
    """CPU stand-in for verify.EngineWitnesses (test infrastructure)."""

    def __init__(self, plan, seed: int, n_witness: int):
        from oracle.stage_check import check_stage
        from paper_2506_15961_b200.stages import build_stages, entry_order, shard_owner
        self.check = check_stage
        self.plan = plan
        self.stages, _ = build_stages(plan)
        self.owner = shard_owner(plan, entry_order(plan))
        self.seed, self.W = seed, n_witness

    def run(self, refs, opts):
        n = max(r.comp.index for r in refs if r.comp is not None) + 1
        fb = np.full(n, 0xFFFFFFFFFFFFFFFF, dtype=np.uint64)
        nv = np.zeros(n, dtype=np.uint32)
        nb = np.zeros(n, dtype=np.uint32)
        wit = np.arange(self.W, dtype=np.uint64)
        for r in refs:
            if r.comp is None or r.comp.status != 0:
                continue
            o = self.check(self.plan, self.stages[r.stage], self.owner, self.seed, wit)
            i = r.comp.index
            nv[i], nb[i] = o.valid, o.bad
            if o.first_bad is not None:
                fb[i] = (o.first_bad[0] << 32) | o.first_bad[1]
        return fb, nv, nb, 0.0

    def probe(self, comp, w, obl):
        return 0, 1, np.zeros(max(comp.n_vars, 1), dtype=np.uint32)


def _reference():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    os.environ.setdefault("PLANEQ_SOLVER", sys.executable + " -m planeq.smtsolver")
    from planeq import plan as rplan
    from planeq import verify as rverify
    return rplan, rverify


@pytest.mark.parametrize("name", NAMES)
def test_reference_verify_plan_runs_on_the_engine(lib, name):
    from paper_2506_15961_b200.planeq_binding import install
    from paper_2506_15961_b200.verify import VerifyOptions, verify_plan
    rplan, rverify = _reference()
    rec = next(r for r in verdicts() if r["name"] == name)
    with gzip.open(os.path.join(GOLDEN, rec["work_plan"]), "rt") as f:
        text = f.read()
    ours = VerifyOptions(no_cancel=True, witnesses=64, seed=3)
    restore = install(rverify, ours,
                      source=OracleWitnesses(load_plan(rec["work_plan"]), 3, 64))
    try:
        rep = rverify.verify_plan(rplan.loads(text),
                                  rverify.VerifyOptions(no_reduce=True, no_cancel=True))
    finally:
        restore()
    got = [(s["target"], s["status"]) for s in rep["stages"]]
    want = [tuple(x) for x in rec["default"]["stage_status"]]
    assert [t for t, _ in got] == [t for t, _ in want]
    for (t, g), (_, w) in zip(got, want):
        if w in ("proven", "refuted"):
            assert g == w, (name, t)
    # this package's own verify_plan on the same plan, same witness source
    import paper_2506_15961_b200.verify as V
    src = OracleWitnesses(load_plan(rec["work_plan"]), 3, 64)
    orig = V.discharge_native

    def with_source(*a, **k):
        k["source"] = src
        return orig(*a, **k)
    V.discharge_native = with_source
    try:
        mine = verify_plan(load_plan(rec["work_plan"]), ours)
    finally:
        V.discharge_native = orig
    assert [(s["target"], s["status"]) for s in mine["stages"]] == got
    assert mine["verdict"] == rep["verdict"]

"""Host callers either side of the path reproduce the reference byte for byte:
toy builder + completion + parallelizer (the plan), fault injector (the
mutant), shape reducer (the work plan). Golden files come from the reference
itself (oracle/gen_golden.py)."""

import gzip
import os

import pytest

from golden_io import GOLDEN, verdicts
from paper_2506_15961_b200 import builder, completion
from paper_2506_15961_b200.faults import FaultSpec, inject, list_sites
from paper_2506_15961_b200.parallelize import ParallelConfig, parallelize
from paper_2506_15961_b200.plan import dumps, loads

RECS = verdicts() if os.path.exists(os.path.join(GOLDEN, "verdicts.json")) else []
TOY = {r["name"]: r for r in RECS if r["meta"]["source"] == "toy"}
FAULTS = [r for r in RECS if r["meta"]["source"] == "fault"]
CFGS = {"tp2": ParallelConfig(tp=2), "pp2nm2": ParallelConfig(pp=2, nm=2),
        "dp2tp2pp2nm2": ParallelConfig(dp=2, tp=2, pp=2, nm=2),
        "tp2pp2": ParallelConfig(tp=2, pp=2), "dp2tp2nm2": ParallelConfig(dp=2, tp=2, nm=2)}


def _text(rel):
    with gzip.open(os.path.join(GOLDEN, rel), "rt") as f:
        return f.read()


def _toy_plan(cfg):
    g = completion.complete(builder.toy_forward(builder.ToyConfig()), completion.LossSpec("mean"))
    return parallelize(g, cfg, lineage_interiors=builder.toy_interiors(g))


@pytest.mark.parametrize("name", sorted(TOY))
def test_toy_plan_byte_identical(name):
    assert dumps(_toy_plan(CFGS[name])) == _text(TOY[name]["plan"])


@pytest.mark.parametrize("name", sorted(TOY))
def test_reduced_plan_byte_identical(name):
    from paper_2506_15961_b200.errors import PlanEqError
    from paper_2506_15961_b200.shapes import reduce_plan
    rec = TOY[name]
    plan = loads(_text(rec["plan"]))
    if "work_plan" not in rec:
        with pytest.raises(PlanEqError):
            reduce_plan(plan)
        return
    assert dumps(reduce_plan(plan).plan) == _text(rec["work_plan"])


@pytest.mark.parametrize("rec", FAULTS, ids=[r["name"] for r in FAULTS])
def test_fault_mutant_byte_identical(rec):
    base_name = rec["name"].split(".")[0]
    base = loads(_text(TOY[base_name]["plan"]))
    spec = rec["meta"]["fault"]
    fs = FaultSpec(spec["category"], spec["site"], spec["detail"])
    assert fs in list_sites(base, fs.category)
    assert dumps(inject(base, fs)) == _text(rec["plan"])


def test_config_errors():
    from paper_2506_15961_b200.errors import ConfigError, UnsupportedOperator
    with pytest.raises(ConfigError):
        builder.ToyConfig(layers=0)
    g = completion.complete(builder.toy_forward(builder.ToyConfig()), completion.LossSpec("mean"))
    with pytest.raises(UnsupportedOperator):
        parallelize(g, ParallelConfig(dp=3))

"""Host-side API parity: plan format, graph utilities, stage construction.

The stage partition must be exactly the reference's (same targets, same
logical/parallel node lists, same interface tensors) for verdict parity to be
meaningful; tests/golden/verdicts.json records the reference's build_stages
output on every golden work plan.
"""

import gzip
import os

import pytest

from golden_io import GOLDEN, load_plan, verdicts
from paper_2506_15961_b200 import errors
from paper_2506_15961_b200.graph import (Graph, LineageEntry, Node, Shard, Tensor, iter_box,
                                         topo_sort, validate_lineage)
from paper_2506_15961_b200.opshape import validate_concrete
from paper_2506_15961_b200.plan import dumps, loads
from paper_2506_15961_b200.stages import build_stages

RECS = verdicts() if os.path.exists(os.path.join(GOLDEN, "verdicts.json")) else []
WORK = [r for r in RECS if "work_plan" in r]


def _g(nodes, inputs, tensors):
    g = Graph()
    for tid, shape in tensors.items():
        g.add_tensor(Tensor(tid, shape))
    g.inputs = list(inputs)
    for n in nodes:
        g.add_node(n)
    return g


def test_topo_sort_empty_and_chain():
    assert topo_sort(Graph()) == []
    g = _g([Node("c", "identity", ("b",), ("c",)), Node("b", "identity", ("a",), ("b",))],
           ["a"], {"a": (1,), "b": (1,), "c": (1,)})
    assert [n.id for n in topo_sort(g)] == ["b", "c"]


def test_topo_sort_cycle_and_dangling():
    g = _g([Node("n1", "add", ("a", "y"), ("x",)), Node("n2", "identity", ("x",), ("y",))],
           ["a"], {"a": (1,), "x": (1,), "y": (1,)})
    with pytest.raises(errors.CycleError):
        topo_sort(g)
    g2 = _g([Node("n1", "identity", ("ghost",), ("x",))], [], {"x": (1,)})
    with pytest.raises(errors.DanglingTensorError):
        topo_sort(g2)


def test_validate_lineage_examples():
    lg = Graph()
    lg.add_tensor(Tensor("t", (4, 4)))
    pg = Graph()
    for n, s in (("a", (2, 4)), ("b", (2, 4)), ("p", (2, 4))):
        pg.add_tensor(Tensor(n, s))
    ok = {"t": LineageEntry("t", "full", (Shard("a", ((0, 2), (0, 4))), Shard("b", ((2, 4), (0, 4)))))}
    assert validate_lineage(lg, pg, ok) == []
    bad = {"t": LineageEntry("t", "full", (Shard("a", ((0, 2), (0, 4))), Shard("b", ((0, 2), (0, 4)))))}
    assert any("do not tile" in p for p in validate_lineage(lg, pg, bad))
    part = {"t": LineageEntry("t", "partial", (Shard("p", ((0, 2), (0, 4))),))}
    assert validate_lineage(lg, pg, part)


def test_iter_box_row_major():
    assert list(iter_box(((0, 2), (1, 3)))) == [(0, 1), (0, 2), (1, 1), (1, 2)]
    assert list(iter_box(())) == [()]


def test_plan_errors():
    with pytest.raises(errors.PlanFormatError):
        loads("{}")
    with pytest.raises(errors.SchemaVersionError):
        loads('{"version": 2, "logical": {}}')
    with pytest.raises(errors.PlanFormatError):
        loads("not json")


@pytest.mark.parametrize("rec", RECS[:6], ids=[r["name"] for r in RECS[:6]])
def test_reference_plan_files_round_trip_byte_identical(rec):
    with gzip.open(os.path.join(GOLDEN, rec["plan"]), "rt") as f:
        text = f.read()
    assert dumps(loads(text)) == text


@pytest.mark.parametrize("rec", WORK, ids=[r["name"] for r in WORK])
def test_build_stages_matches_reference(rec):
    plan = load_plan(rec["work_plan"])
    validate_concrete(plan.logical)
    validate_concrete(plan.parallel)
    stages, _ = build_stages(plan)
    got = [{"target": s.target, "logical": [n.id for n in s.logical_nodes],
            "parallel": [n.id for n in s.parallel_nodes], "l_inputs": s.l_inputs,
            "p_inputs": s.p_inputs} for s in stages]
    assert got == rec["work_stages"]

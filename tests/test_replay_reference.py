"""Counterexamples are reproducible by the reference's own evaluator.

For every refuted stage of the golden fault plans, the first failing witness
(the oracle's, which the GPU tests prove bit-identical to the GPU's) is
replayed through the reference implementation itself: the stage's obligation
expressions are rebuilt with the reference's symbolic engine
(pkg/src/planeq/stages.py:144-176 interface, ops.py:923 sym_execute), then
evaluated exactly (sym.py:322 eval_expr) at the integer witness assignment
with EXP/RSQRT/SIGMOID interpreted as the keyed hash of the argument's residue.
The two sides must differ as rationals, and their residues must equal the
values the witness engine reports.

Runs only where /root/reference is present (the build container).
"""

import os
import sys
from fractions import Fraction

import numpy as np
import pytest

from golden_io import load_plan, verdicts
from oracle.stage_check import check_stage
from paper_2506_15961_b200 import field as F
from paper_2506_15961_b200.stages import build_stages, entry_order, shard_owner

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources not present")

RECS = [r for r in verdicts() if "work_plan" in r and r["meta"]["source"] in ("fault", "random_plan")
        and r["default"].get("verdict") in ("refuted", "unknown")]


def _ref_modules():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from planeq import plan as rplan
    from planeq import stages as rstages
    from planeq import ops as rops
    from planeq import sym as rsym
    from planeq.graph import iter_box, range_extents
    return rplan, rstages, rops, rsym, iter_box, range_extents


_REF_CACHE: dict = {}


def _ref_obligations(rplan, rstages, rops, rsym, iter_box, plan_text, target):
    """The reference's (lhs, rhs) expression list for one stage, in obligation order."""
    key = hash(plan_text)
    if key not in _REF_CACHE:
        plan = rplan.loads(plan_text)
        _REF_CACHE.clear()
        _REF_CACHE[key] = (plan, rstages.build_stages(plan)[0])
    plan, stages = _REF_CACHE[key]
    stage = next(s for s in stages if s.target == target)
    alg = rsym.Algebra()
    ctx = rsym.ExecContext(alg)
    lshapes = {t.id: t.shape for t in plan.logical.tensors.values()}
    pshapes = {t.id: t.shape for t in plan.parallel.tensors.values()}
    boxes = {}

    def box_of(tid):
        if tid not in boxes:
            boxes[tid] = rstages._logical_box(plan.logical.tensors[tid], alg)
        return boxes[tid]

    env_l = {}
    produced_l = {o for n in stage.logical_nodes for o in n.outputs}
    for tid in stage.l_inputs:
        if tid not in produced_l:
            env_l[tid] = box_of(tid)
    rops.sym_execute(plan.logical, stage.logical_nodes, env_l, lshapes, ctx)
    owner = {}
    for etid in reversed(rstages.entry_order(plan)):
        for s in plan.lineage[etid].shards:
            owner[s.tensor] = etid
    env_p, done = {}, set()
    produced_p = {o for n in stage.parallel_nodes for o in n.outputs}
    for st in stage.p_inputs:
        if st in produced_p or owner[st] in done:
            continue
        done.add(owner[st])
        rstages._materialize_entry(plan.lineage[owner[st]], plan.logical.tensors[owner[st]],
                                   box_of(owner[st]), alg, env_p)
    rops.sym_execute(plan.parallel, stage.parallel_nodes, env_p, pshapes, ctx)
    entry = plan.lineage[target]
    box = env_l[target]
    out = []
    if entry.mode == "full":
        for s in entry.shards:
            vt = env_p[s.tensor]
            for li, g in enumerate(iter_box(s.ranges)):
                out.append((box.at(g), vt.data[li]))
    else:
        for ranges, members in sorted(entry.groups().items()):
            members = sorted(members, key=lambda s: s.tensor)
            vts = [env_p[s.tensor] for s in members]
            for li, g in enumerate(iter_box(ranges)):
                out.append((box.at(g), alg.addn([vt.data[li] for vt in vts])))
    _ref_obligations.last_conds = ctx.conds
    return out, alg


def _ref_obligations_ctx(rplan, rstages, rops, rsym, iter_box, plan_text, target):
    """(obligation expression pairs, definedness conditions) of one stage."""
    pairs, _alg = _ref_obligations(rplan, rstages, rops, rsym, iter_box, plan_text, target)
    return pairs, _ref_obligations.last_conds


@pytest.mark.parametrize("rec", RECS, ids=[r["name"] for r in RECS])
def test_counterexample_replays_in_reference_evaluator(rec):
    import gzip
    from golden_io import GOLDEN
    rplan, rstages, rops, rsym, iter_box, _ = _ref_modules()
    seed, W = 21, 16
    plan = load_plan(rec["work_plan"])
    with gzip.open(os.path.join(GOLDEN, rec["work_plan"]), "rt") as f:
        text = f.read()
    stages, _ = build_stages(plan)
    owner = shard_owner(plan, entry_order(plan))
    keys = {fn: F.fn_key(seed, fn) for fn in F.FN_NAMES}

    def uf(fn, x):
        return Fraction(F.uf_apply(keys[fn], F.residue(x)))

    refuted = 0
    for st in stages:
        if refuted == 3:  # the reference's symbolic execution is slow: 3 per plan
            break
        o = check_stage(plan, st, owner, seed, np.arange(W, dtype=np.uint64))
        if o.status != "refuted":
            continue
        refuted += 1
        w, obl = o.first_bad
        pairs, _alg = _ref_obligations(rplan, rstages, rops, rsym, iter_box, text, st.target)
        lhs, rhs = pairs[obl]
        # the witness assignment: every interface variable at witness w
        env = {}
        for name in rsym.collect_vars([lhs, rhs]):
            prefix, i = name.rsplit(".", 1)
            env[name] = Fraction(F.witness_value(F.var_key(seed, prefix, int(i)), w))
        lv = lhs if isinstance(lhs, int) else rsym.eval_expr(lhs, env, uf)
        rv = rhs if isinstance(rhs, int) else rsym.eval_expr(rhs, env, uf)
        assert lv != rv, st.target
        assert F.residue(lv) == o.lhs and F.residue(rv) == o.rhs, st.target
    if rec["default"].get("verdict") == "refuted" and rec["default"].get("refuted_by") != "structure":
        assert refuted > 0


def _ds_recs():
    import json
    from golden_io import GOLDEN
    p = os.path.join(GOLDEN, "verdicts_deepseek.json")
    if not os.path.exists(p):
        return []
    return [r for r in json.load(open(p))["plans"] if r.get("stage_reason")]


DS_RECS = _ds_recs()


@pytest.mark.parametrize("rec", DS_RECS, ids=[r["name"] for r in DS_RECS])
def test_unconfirmed_reference_countermodels_are_real(rec):
    """Where the reference reports "unknown" (its solver returned unknown, or its
    countermodel failed exact replay), the witness engine's counterexample
    replays: the two sides of the failing obligation differ as rationals in the
    reference's own evaluator."""
    import gzip
    from golden_io import GOLDEN
    rplan, rstages, rops, rsym, iter_box, _ = _ref_modules()
    seed, W = 21, 16
    plan = load_plan(rec["plan"])
    with gzip.open(os.path.join(GOLDEN, rec["plan"]), "rt") as f:
        text = f.read()
    stages, _ = build_stages(plan)
    owner = shard_owner(plan, entry_order(plan))
    keys = {fn: F.fn_key(seed, fn) for fn in F.FN_NAMES}

    def uf(fn, x):
        return Fraction(F.uf_apply(keys[fn], F.residue(x)))

    targets = sorted(rec["stage_reason"])[:2]
    for st in stages:
        if st.target not in targets:
            continue
        o = check_stage(plan, st, owner, seed, np.arange(W, dtype=np.uint64))
        assert o.status == "refuted", st.target
        w, obl = o.first_bad
        pairs, _alg = _ref_obligations(rplan, rstages, rops, rsym, iter_box, text, st.target)
        lhs, rhs = pairs[obl]
        env = {}
        for name in rsym.collect_vars([lhs, rhs]):
            prefix, i = name.rsplit(".", 1)
            env[name] = Fraction(F.witness_value(F.var_key(seed, prefix, int(i)), w))
        lv = lhs if isinstance(lhs, int) else rsym.eval_expr(lhs, env, uf)
        rv = rhs if isinstance(rhs, int) else rsym.eval_expr(rhs, env, uf)
        assert lv != rv, st.target
        assert F.residue(lv) == o.lhs and F.residue(rv) == o.rhs, st.target

#!/usr/bin/env python
"""Kernel time per distinct stage program of a workload (all stages sharing
that program launched together), next to its op count and spills: shows
which programs the interpreter runs least efficiently. GPU only."""
import sys
import time
from collections import defaultdict

import numpy as np

sys.path.insert(0, ".")
from paper_2506_15961_b200 import field as F  # noqa: E402
from paper_2506_15961_b200.engine import STAGE_OK, Engine  # noqa: E402
from paper_2506_15961_b200.stages import build_stages, entry_order, lower_stage, shard_owner  # noqa: E402
from paper_2506_15961_b200.workloads import get_workload  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "llama3-8b-tp4pp2dp2-sp"
W = 512
_d, plan = get_workload(name)
stages, _ = build_stages(plan)
owner = shard_owner(plan, entry_order(plan))
groups = defaultdict(list)
for st in stages:
    lw = lower_stage(plan, st, owner, 0)
    groups[(lw.ir.size, lw.ir.tobytes().__hash__(), lw.consts.size)].append(lw)
rows = []
for key, lws in groups.items():
    eng = Engine(0, 0, F.fn_keys(0))
    cs = [eng.add_stage(l.ir, l.consts, l.var_keys) for l in lws]
    if cs[0].status != STAGE_OK:
        eng.close()
        continue
    eng.upload()
    for _ in range(3):
        eng.launch(W)
        eng.results()
    ts = []
    for _ in range(5):
        eng.launch(W)
        eng.results()
        ts.append(eng.last_launch_ms())
    s = eng.image_stats()
    fo = sum(s["field_ops"].values())
    h = s["op_hist"]
    ms = float(np.median(ts))
    rows.append((ms, len(lws), s["instructions"] // len(lws), fo // len(lws), h["FILL"] // len(lws),
                 s["bundles"] // len(lws), s["waits"] // len(lws), s["max_slots"]))
    eng.close()
tot = sum(r[0] for r in rows)
print(f"{'ms':>8} {'share':>6} {'stages':>6} {'records':>8} {'fieldops':>9} {'fills':>7} "
      f"{'bundles':>7} {'waits':>7} {'slots':>5} {'ns/fieldop/witness':>10}")
for r in sorted(rows, reverse=True):
    ms, n, rec, fo, fi, b, wt, sl = r
    print(f"{ms:8.3f} {100 * ms / tot:5.1f}% {n:6d} {rec:8d} {fo:9d} {fi:7d} {b:7d} {wt:7d} {sl:5d} "
          f"{ms * 1e6 / (fo * n * W / 148):10.3f}")
print("sum of per-program launches", round(tot, 3), "ms")

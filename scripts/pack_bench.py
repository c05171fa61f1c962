"""Host-side timing of the native plan core on a workload (no GPU needed):
packing (C++ packer; PQW_PACK_SERIAL=1 for the serial path), validation,
stage construction, lowering + queueing, compiler front and back ends."""
import os
import sys
import time

sys.path.insert(0, ".")
from paper_2506_15961_b200 import field as F  # noqa: E402
from paper_2506_15961_b200 import native as N  # noqa: E402
from paper_2506_15961_b200.engine import Engine  # noqa: E402
from paper_2506_15961_b200.workloads import get_workload  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "llama3-405b-tp8pp16dp2"
desc, plan = get_workload(name)
for mode in ("threaded", "serial", "threaded"):
    if mode == "serial":
        os.environ["PQW_PACK_SERIAL"] = "1"
    else:
        os.environ.pop("PQW_PACK_SERIAL", None)
    t = [time.perf_counter()]
    nat = N.NativePlan(plan)
    t.append(time.perf_counter())
    nat.validate()
    t.append(time.perf_counter())
    nat.build_stages()
    t.append(time.perf_counter())
    eng = Engine(0, 0, F.fn_keys(0))
    idx = nat.add_stages(eng, 0)
    t.append(time.perf_counter())
    [eng.stage_lazy(int(k)).status for k in idx[:1]]
    t.append(time.perf_counter())
    eng.image_stats()
    t.append(time.perf_counter())
    d = [round(b - a, 3) for a, b in zip(t, t[1:])]
    print(f"{name} packer={mode}: pack+create {d[0]}s validate {d[1]}s build_stages {d[2]}s "
          f"lower+queue {d[3]}s front {d[4]}s back {d[5]}s", flush=True)
    eng.close()
    nat.close()

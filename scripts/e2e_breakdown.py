"""Where verify_plan's wall time goes on a workload (GPU): repeated runs, the
engine-side steps timed separately."""
import sys
import time

sys.path.insert(0, ".")
from paper_2506_15961_b200 import field as F  # noqa: E402
from paper_2506_15961_b200.engine import Engine  # noqa: E402
from paper_2506_15961_b200.native import NativePlan  # noqa: E402
from paper_2506_15961_b200.verify import VerifyOptions, verify_plan  # noqa: E402
from paper_2506_15961_b200.workloads import get_workload  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "llama-2l-tp2dp2"
_d, plan = get_workload(name)
for i in range(8):
    t0 = time.perf_counter()
    rep = verify_plan(plan, VerifyOptions(no_reduce=True, witnesses=512, device=0))
    t1 = time.perf_counter()
    print(f"verify_plan {t1 - t0:.4f}s", rep["engine"].get("times"), rep["engine"].get("phases"),
          "lower_s", rep["engine"].get("lower_s"), flush=True)
for i in range(3):
    t = [time.perf_counter()]
    nat = NativePlan(plan); nat.validate(); nat.build_stages(); t.append(time.perf_counter())
    eng = Engine(0, 0, F.fn_keys(0)); t.append(time.perf_counter())
    idx = nat.add_stages(eng, 0); t.append(time.perf_counter())
    eng.image_stats(); t.append(time.perf_counter())
    eng.upload(); t.append(time.perf_counter())
    eng.launch(512); eng.results(); t.append(time.perf_counter())
    eng.close(); nat.close(); t.append(time.perf_counter())
    names = ("plan", "engine_create", "add_stages", "compile", "upload", "launch+results", "close")
    print(" ".join(f"{n} {b - a:.4f}" for n, a, b in zip(names, t, t[1:])), flush=True)

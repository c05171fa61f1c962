"""Host-side phase times of the native plan path on the 405B workload (no GPU
work): the C++ packer per graph (prefetch on/off), pqw_plan_create's load
phases (PQW_TIMING), validate and build_stages. Prints one line per repeat."""
import gc
import os
import sys
import time

sys.path.insert(0, ".")
from paper_2506_15961_b200 import native as N  # noqa: E402
from paper_2506_15961_b200.workloads import get_workload  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "llama3-405b-tp8pp16dp2"
_, plan = get_workload(name)
gc.disable()
ext = N._ext()
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)), flush=True)
for variant in ("default", "nopf", "default"):
    if variant == "nopf":
        os.environ["PQW_PACK_NOPF"] = "1"
    else:
        os.environ.pop("PQW_PACK_NOPF", None)
    for r in range(3):
        c = N._Consts()
        t0 = time.perf_counter()
        ext.pack_graph(plan.parallel, N.OPCODE, c)
        t1 = time.perf_counter()
        nat = N.NativePlan(plan)
        t2 = time.perf_counter()
        nat.validate()
        t3 = time.perf_counter()
        nat.build_stages()
        t4 = time.perf_counter()
        nat.close()
        print(f"{variant}: pack(parallel graph) {1e3*(t1-t0):.1f} ms  NativePlan {1e3*(t2-t1):.1f} ms  "
              f"validate {1e3*(t3-t2):.1f} ms  build_stages {1e3*(t4-t3):.1f} ms", flush=True)

"""Host-side timing of the native plan core's stages on a workload (no GPU needed):
plan packing with 1..16 packer processes, validation, stage construction."""
import sys
import time

sys.path.insert(0, ".")
from paper_2506_15961_b200 import native as N  # noqa: E402
from paper_2506_15961_b200.workloads import get_workload  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "llama3-405b-tp8pp16dp2"
desc, plan = get_workload(name)
for k in (1, 4, 8, 16):
    N._workers = lambda k=k: k
    t = time.perf_counter()
    nat = N.NativePlan(plan)
    t1 = time.perf_counter()
    nat.validate()
    t2 = time.perf_counter()
    nat.build_stages()
    t3 = time.perf_counter()
    print(f"{name} packers={k}: pack+create {t1 - t:.3f}s validate {t2 - t1:.3f}s "
          f"build_stages {t3 - t2:.3f}s", flush=True)
    nat.close()

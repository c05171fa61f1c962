"""Named verification workloads for bench.py and the tests.

A workload is a work plan (the plan the discharge step runs on). Round 1
ships the reference's own reduced toy-decoder plans (committed fixtures under
tests/golden/plans, produced by the reference's parallelizer and shape
reducer); generated Llama-style plans are added by plangen.
"""

from __future__ import annotations

import gzip
import os

from .plan import Plan, loads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN_PLANS = os.path.join(ROOT, "tests", "golden", "plans")

FIXTURES = {
    "toy-dp2tp2pp2nm2": ("dp2tp2pp2nm2.work.json.gz",
                         "reference toy decoder (2 layers), dp2 tp2 pp2 nm2, reduced by the reference"),
    "toy-tp2": ("tp2.work.json.gz", "reference toy decoder (2 layers), tp2, reduced by the reference"),
}
DEFAULT = "toy-dp2tp2pp2nm2"


def _fixture(fname: str) -> Plan:
    with gzip.open(os.path.join(GOLDEN_PLANS, fname), "rt") as f:
        return loads(f.read())


def get_workload(name: str = "default") -> tuple[str, Plan]:
    if name == "default":
        name = DEFAULT
    if name in FIXTURES:
        fname, desc = FIXTURES[name]
        return f"{name}: {desc}", _fixture(fname)
    raise KeyError(f"unknown workload {name!r}; known: {sorted(FIXTURES)}")

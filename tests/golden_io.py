"""Helpers to read the committed golden fixtures (tests/golden)."""

import gzip
import json
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def verdicts():
    with open(os.path.join(GOLDEN, "verdicts.json")) as f:
        return json.load(f)["plans"]


def load_plan(rel):
    from paper_2506_15961_b200.plan import loads
    with gzip.open(os.path.join(GOLDEN, rel), "rt") as f:
        return loads(f.read())


def ops_cases():
    with open(os.path.join(GOLDEN, "ops.json")) as f:
        return json.load(f)

"""Build a variant of the engine library into variants/<name>.so with extra nvcc flags
(for A/B runs: PQW_LIB=variants/<name>.so). Usage: python scripts/build_variant.py NAME [FLAGS...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_15961_b200 import build as B  # noqa: E402

name = sys.argv[1]
os.environ["PQW_NVCC_FLAGS"] = " ".join(sys.argv[2:])
os.makedirs(os.path.join(os.path.dirname(B.HERE), "variants"), exist_ok=True)
B.OUT = os.path.join(os.path.dirname(B.HERE), "variants", name + ".so")
print(B.build(force=True))

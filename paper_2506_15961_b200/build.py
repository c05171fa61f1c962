"""Build libplaneq_witness.so in-tree for sm_100a (nvcc, no GPU needed)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libplaneq_witness.so")
SOURCES = ["compiler.cpp", "schedule.cpp", "plan.cpp", "witness_kernel.cu"]
HEADERS = ["compiler.hpp", "field.hpp", "isa.hpp", "pool.hpp", "schedule.hpp", "interp.cuh"]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "planeq_witness.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def _ext_path() -> str:
    import sysconfig
    return os.path.join(HERE, "_pqw_pack" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_pack(force: bool = False) -> str:
    """The CPython host packer (csrc/pack.cpp -> _pqw_pack extension, g++)."""
    import sysconfig
    out = _ext_path()
    src = os.path.join(CSRC, "pack.cpp")
    if not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(src):
        return out
    cxx = os.environ.get("CXX", "g++")
    cmd = [cxx, "-O2", "-std=c++17", "-shared", "-fPIC", "-I", sysconfig.get_paths()["include"],
           src, "-o", out + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("g++ failed building the _pqw_pack extension")
    os.replace(out + ".tmp", out)
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    build_pack(force)
    if not force and not _stale():
        return OUT
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
           "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v",
           "-diag-suppress", "128", "-o", OUT + ".tmp"] + os.environ.get("PQW_NVCC_FLAGS", "").split() + \
        [os.path.join(CSRC, s) for s in SOURCES]
    r = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libplaneq_witness.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))

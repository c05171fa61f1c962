"""ctypes binding of the sm_100a witness engine (include/planeq_witness.h).

The library is built in-tree (``paper_2506_15961_b200/libplaneq_witness.so``,
see build.py). There is deliberately no CPU evaluation path: if the library
or a CUDA device is missing, the calls that need them raise
``EngineUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from .errors import EngineError, EngineUnavailable

LIB_NAME = "libplaneq_witness.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)
ABI_VERSION = 5

# PQW_STAGE_* codes
STAGE_OK = 0
STAGE_PROVEN = 1
STAGE_REFUTED_CONST = 2
STAGE_PAR_DIV0 = 3
STAGE_LOG_DIV0 = 4
STAGE_BAD_INDEX = 5
STAGE_PENDING = 6
STAGE_LOSSY = 7

# bytecode opcodes (pqw_bop)
BOP_NAMES = ("END", "DOT", "SUM", "SUB", "NEG", "HASH", "INV", "VAR", "CONST", "CHK", "DEN",
             "FILL", "SPILL", "WAIT", "SIGNAL")
N_BOPS = len(BOP_NAMES)
IMAGE_STATS_LEN = 16 + N_BOPS
FIELD_CLASSES = ("mul", "add", "hash", "inv", "cmp")

EXPORTS = ("pqw_abi_version", "pqw_last_error", "pqw_device_count", "pqw_engine_create",
           "pqw_engine_destroy", "pqw_stage_add", "pqw_stage_status", "pqw_reset", "pqw_stage_bytecode",
           "pqw_obligation_support", "pqw_upload", "pqw_launch", "pqw_results", "pqw_probe",
           "pqw_last_launch_ms", "pqw_image_stats", "pqw_peak_fieldops", "pqw_stage_select",
           "pqw_stage_cost", "pqw_confirm",
           # native plan core (native.py)
           "pqw_plan_create", "pqw_plan_destroy", "pqw_plan_validate", "pqw_plan_check_lineage",
           "pqw_plan_build_stages",
           "pqw_plan_stage_target", "pqw_plan_stage_nodes", "pqw_plan_uncovered",
           "pqw_plan_add_stages", "pqw_plan_stage_program")


class _Ins(C.Structure):
    _fields_ = [("op", C.c_uint32), ("dst", C.c_uint32), ("a", C.c_uint32), ("b", C.c_uint32)]


_lib = None


def load_library(path: str | None = None):
    """Load (once) and type the C-ABI library; raise EngineUnavailable if absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or os.environ.get("PQW_LIB") or LIB_PATH
    if not os.path.exists(p):
        raise EngineUnavailable(
            f"{LIB_NAME} not built (expected at {p}); run __graft_entry__.build()")
    try:
        lib = C.CDLL(p)
    except OSError as e:
        raise EngineUnavailable(f"cannot load {p}: {e}") from e
    u64p = C.POINTER(C.c_uint64)
    u32p = C.POINTER(C.c_uint32)
    i64p = C.POINTER(C.c_int64)
    i32p = C.POINTER(C.c_int32)
    lib.pqw_abi_version.restype = C.c_int
    lib.pqw_last_error.restype = C.c_char_p
    lib.pqw_device_count.restype = C.c_int
    lib.pqw_engine_create.argtypes = [C.c_int, C.c_uint64, u64p, C.POINTER(C.c_void_p)]
    lib.pqw_engine_create.restype = C.c_int
    lib.pqw_engine_destroy.argtypes = [C.c_void_p]
    lib.pqw_engine_destroy.restype = None
    lib.pqw_stage_add.argtypes = [C.c_void_p, i32p, C.c_size_t, i64p, C.c_size_t, u64p,
                                  C.c_size_t, i64p]
    lib.pqw_stage_add.restype = C.c_int
    lib.pqw_stage_status.argtypes = [C.c_void_p, C.c_int, i64p]
    lib.pqw_stage_status.restype = C.c_int
    lib.pqw_reset.argtypes = [C.c_void_p]
    lib.pqw_reset.restype = C.c_int
    lib.pqw_stage_bytecode.argtypes = [C.c_void_p, C.c_int, C.POINTER(_Ins), C.c_size_t, u32p]
    lib.pqw_stage_bytecode.restype = C.c_long
    lib.pqw_obligation_support.argtypes = [C.c_void_p, C.c_int, C.c_uint32, u32p, C.c_size_t]
    lib.pqw_obligation_support.restype = C.c_long
    lib.pqw_upload.argtypes = [C.c_void_p]
    lib.pqw_upload.restype = C.c_int
    lib.pqw_launch.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p]
    lib.pqw_launch.restype = C.c_int
    lib.pqw_results.argtypes = [C.c_void_p, u64p, u32p, u32p, C.c_size_t]
    lib.pqw_results.restype = C.c_int
    lib.pqw_probe.argtypes = [C.c_void_p, C.c_int, C.c_uint32, C.c_uint32, u32p, u32p, u32p,
                              C.c_size_t]
    lib.pqw_probe.restype = C.c_int
    lib.pqw_last_launch_ms.argtypes = [C.c_void_p, C.POINTER(C.c_float)]
    lib.pqw_last_launch_ms.restype = C.c_int
    lib.pqw_image_stats.argtypes = [C.c_void_p, u64p, C.c_size_t]
    lib.pqw_image_stats.restype = C.c_int
    lib.pqw_stage_select.argtypes = [C.c_void_p, C.POINTER(C.c_uint8), C.c_size_t]
    lib.pqw_stage_select.restype = C.c_int
    lib.pqw_stage_cost.argtypes = [C.c_void_p, C.c_int]
    lib.pqw_stage_cost.restype = C.c_int64
    lib.pqw_confirm.argtypes = [C.c_void_p, C.c_int, C.c_uint32, C.POINTER(C.c_double),
                                C.c_size_t, C.c_double, i64p, C.POINTER(C.c_double)]
    lib.pqw_confirm.restype = C.c_int
    lib.pqw_peak_fieldops.argtypes = [C.c_int, C.POINTER(C.c_double)]
    lib.pqw_peak_fieldops.restype = C.c_int
    if lib.pqw_abi_version() != ABI_VERSION:
        raise EngineUnavailable(f"{p} has ABI {lib.pqw_abi_version()}, expected {ABI_VERSION}")
    if path is None:
        _lib = lib
    return lib


def device_count() -> int:
    return int(load_library().pqw_device_count())


def peak_fieldops(device: int = 0) -> dict:
    """Measured register-resident F_p op rates of the device (ops/s)."""
    lib = load_library()
    out = (C.c_double * 4)()
    rc = lib.pqw_peak_fieldops(device, out)
    if rc < 0:
        msg = lib.pqw_last_error().decode(errors="replace")
        raise (EngineUnavailable if rc == -2 else EngineError)(msg)
    return {"mul": out[0], "add": out[1], "hash": out[2], "inv": out[3]}


_I64_MIN = -(1 << 63)


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


@dataclass
class StageCompile:
    """What the compiler reports for one stage (out_status of pqw_stage_add)."""
    index: int
    status: int
    info: int
    obligations: int
    fast: int
    residual: int
    code_len: int
    slots: int
    degree: int
    const_lhs: int
    const_rhs: int
    exact_lhs: int | None
    exact_rhs: int | None
    field_ops: int
    n_vars: int
    spill_slots: int = 0
    bundles: int = 0


class _LazyStage:
    """StageCompile of a queued stage, fetched (compiling every pending stage
    of the engine at once) on first attribute access."""

    __slots__ = ("_eng", "index", "_sc")

    def __init__(self, eng: "Engine", index: int):
        self._eng = eng
        self.index = index
        self._sc = None

    def __getattr__(self, name):
        if self._sc is None:
            self._sc = self._eng.stage_status(self.index)
        return getattr(self._sc, name)


class Engine:
    """One engine = one compiled device image of many stages on one GPU."""

    def __init__(self, device: int = 0, seed: int = 0, fn_keys: tuple[int, int, int] = (0, 0, 0)):
        self.lib = load_library()
        self.device = device
        self.seed = seed
        keys = (C.c_uint64 * 3)(*[k & ((1 << 64) - 1) for k in fn_keys])
        h = C.c_void_p()
        self._check(self.lib.pqw_engine_create(device, seed & ((1 << 64) - 1), keys, C.byref(h)))
        self._h = h
        self.n_stages = 0

    def _check(self, rc: int):
        if rc < 0:
            msg = self.lib.pqw_last_error().decode(errors="replace")
            if rc == -2:
                raise EngineUnavailable(msg)
            raise EngineError(f"witness engine error {rc}: {msg}")
        return rc

    def close(self):
        if getattr(self, "_h", None):
            self.lib.pqw_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- compile ---------------------------------------------------------------
    def add_stage(self, ir: np.ndarray, consts: np.ndarray, var_keys: np.ndarray) -> "StageCompile":
        """Queue one stage; compilation is deferred (all distinct programs are
        compiled together on host threads). The returned object resolves its
        fields through pqw_stage_status on first access."""
        ir = np.ascontiguousarray(ir, dtype=np.int32)
        consts = np.ascontiguousarray(consts, dtype=np.int64).reshape(-1)
        var_keys = np.ascontiguousarray(var_keys, dtype=np.uint64)
        st = np.zeros(16, dtype=np.int64)
        idx = self._check(self.lib.pqw_stage_add(
            self._h, _ptr(ir, C.c_int32), ir.size, _ptr(consts, C.c_int64), consts.size // 3,
            _ptr(var_keys, C.c_uint64), var_keys.size, _ptr(st, C.c_int64)))
        self.n_stages += 1
        return _LazyStage(self, idx)

    def stage_lazy(self, idx: int) -> "StageCompile":
        """Compile handle of an already queued stage (resolved on first use)."""
        return _LazyStage(self, idx)

    def stage_status(self, idx: int) -> StageCompile:
        st = (C.c_int64 * 16)()  # a ctypes buffer: no numpy round trip per stage
        self._check(self.lib.pqw_stage_status(self._h, idx, st))
        s = st[:]
        return StageCompile(index=idx, status=s[0], info=s[1], obligations=s[2], fast=s[3],
                            residual=s[4], code_len=s[5], slots=s[6], degree=s[7],
                            const_lhs=s[8], const_rhs=s[9],
                            exact_lhs=None if s[10] == _I64_MIN else s[10],
                            exact_rhs=None if s[11] == _I64_MIN else s[11],
                            field_ops=s[12], n_vars=s[13], spill_slots=s[14], bundles=s[15])

    def select(self, active) -> None:
        """Schedule and upload only the stages whose flag is set."""
        a = np.ascontiguousarray(np.asarray(active, dtype=np.uint8))
        self._check(self.lib.pqw_stage_select(self._h, _ptr(a, C.c_uint8), a.size))

    def cost(self, idx: int) -> int:
        """Front-end device cost of a queued stage (0: decided at compile time)."""
        return int(self._check(self.lib.pqw_stage_cost(self._h, idx)))

    def reset(self):
        self._check(self.lib.pqw_reset(self._h))
        self.n_stages = 0

    def bytecode(self, stage: int) -> tuple[np.ndarray, int]:
        """(program records as an (n, 4) uint32 array, shared slot count) of a stage."""
        slots = C.c_uint32()
        n = self._check(self.lib.pqw_stage_bytecode(self._h, stage, None, 0, C.byref(slots)))
        buf = (_Ins * max(n, 1))()
        self._check(self.lib.pqw_stage_bytecode(self._h, stage, buf, n, C.byref(slots)))
        arr = np.frombuffer(buf, dtype=np.uint32, count=4 * n).reshape(n, 4).copy()
        return arr, int(slots.value)

    def support(self, stage: int, obl: int) -> list[int]:
        n = self._check(self.lib.pqw_obligation_support(self._h, stage, obl, None, 0))
        out = np.zeros(max(n, 1), dtype=np.uint32)
        self._check(self.lib.pqw_obligation_support(self._h, stage, obl, _ptr(out, C.c_uint32), n))
        return [int(x) for x in out[:n]]

    # -- device ----------------------------------------------------------------
    def upload(self):
        self._check(self.lib.pqw_upload(self._h))

    def launch(self, n_witness: int, stream: int | None = None):
        self._check(self.lib.pqw_launch(self._h, n_witness, C.c_void_p(stream or 0)))

    def results(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        n = self.n_stages
        fb = np.zeros(max(n, 1), dtype=np.uint64)
        nv = np.zeros(max(n, 1), dtype=np.uint32)
        nb = np.zeros(max(n, 1), dtype=np.uint32)
        self._check(self.lib.pqw_results(self._h, _ptr(fb, C.c_uint64), _ptr(nv, C.c_uint32),
                                         _ptr(nb, C.c_uint32), n))
        return fb[:n], nv[:n], nb[:n]

    def probe(self, stage: int, witness: int, obl: int, n_vars: int):
        lhs, rhs = C.c_uint32(), C.c_uint32()
        vals = np.zeros(max(n_vars, 1), dtype=np.uint32)
        self._check(self.lib.pqw_probe(self._h, stage, witness, obl, C.byref(lhs), C.byref(rhs),
                                       _ptr(vals, C.c_uint32), max(n_vars, 1)))
        return int(lhs.value), int(rhs.value), vals[:n_vars]

    def confirm(self, stage: int, witness: int, envs: np.ndarray, tol: float = 1e-6):
        """Host confirmation of a refutation (pqw_confirm): (exact obligation or
        -1, env index or -1, replay obligation or -1, lhs, rhs, #uf obligations)."""
        envs = np.ascontiguousarray(envs, dtype=np.float64)
        out = np.zeros(4, dtype=np.int64)
        sides = np.zeros(2, dtype=np.float64)
        n_env = envs.shape[0] if envs.ndim == 2 else 0
        self._check(self.lib.pqw_confirm(self._h, stage, witness, _ptr(envs, C.c_double), n_env,
                                         tol, _ptr(out, C.c_int64), _ptr(sides, C.c_double)))
        return int(out[0]), int(out[1]), int(out[2]), float(sides[0]), float(sides[1]), int(out[3])

    def last_launch_ms(self) -> float:
        ms = C.c_float()
        self._check(self.lib.pqw_last_launch_ms(self._h, C.byref(ms)))
        return float(ms.value)

    def image_stats(self) -> dict:
        out = np.zeros(IMAGE_STATS_LEN, dtype=np.uint64)
        self._check(self.lib.pqw_image_stats(self._h, _ptr(out, C.c_uint64), out.size))
        n = N_BOPS
        return {"gpu_stages": int(out[0]), "instructions": int(out[1]),
                "max_slots": int(out[2]), "smem_slots": int(out[3]),
                "op_hist": {BOP_NAMES[i]: int(out[4 + i]) for i in range(n)},
                "unique_instructions": int(out[4 + n]), "cache_hits": int(out[5 + n]),
                "field_ops": {FIELD_CLASSES[i]: int(out[6 + n + i]) for i in range(5)},
                "max_spill_slots": int(out[11 + n]), "bundles": int(out[12 + n]),
                "waits": int(out[13 + n]), "h2d_bytes": int(out[14 + n]),
                "d2h_bytes": int(out[15 + n])}

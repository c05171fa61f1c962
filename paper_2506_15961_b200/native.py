"""Native plan core: the verify pipeline's stage construction and lowering in C++.

Binding of the pqw_plan_* entry points (include/planeq_witness.h). A Plan is
packed once into flat arrays -- names as NUL-separated UTF-8, shapes,
per-node kind codes and encoded attributes, lineage -- and handed to the
library, which then does what the reference does per plan and per stage on
the host (validate_concrete, entry_order, build_stages, stage interface and
obligations: pkg/src/planeq/shapes.py:35-45, stages.py:79-176, :267-340) on
host threads, and queues every stage's tensor-op program into an Engine.

The Python host code (opshape.validate_concrete, stages.build_stages,
stages.lower_stage) stays the drop-in API and the definition: the native
core must produce the same stages and, word for word, the same programs
(tests/test_native_plan.py). When the library declines a plan (PQW_EPLAN:
something the reference would reject, or an attribute the packer cannot
encode), the caller runs the Python host code, which raises the reference's
exception with the reference's message.

Attribute encoding per kind (int64 words; "cid" indexes the plan's table of
distinct rational constants):
  scale [cid(factor)]  shift [cid(addend)]  full [cid(value), ndim, *shape]
  pow [exponent]  div [den_positive]  softmax [axis]  create_mask [size]
  transpose [*perm]  view/expand [ndim, *shape]  embedding_grad [vocab]
  sum/mean [keepdims, 0] (all axes) | [keepdims, 1, n, *axes]
  einsum [len(spec), *code points]  chunk [axis, parts, index]
  all_reduce [group]  all_gather/reduce_scatter [group, axis]
  all_to_all [group, split_axis, concat_axis]     (group = len(attrs["group"]))
"""

from __future__ import annotations

import ctypes as C
from collections import defaultdict
from fractions import Fraction
from itertools import chain
from operator import attrgetter

import numpy as np

from . import field as F
from .engine import Engine, load_library
from .errors import EngineError
from .graph import Graph
from .plan import Plan
from .stages import OPCODE, Stage

E_PLAN = -5

_I64P = C.POINTER(C.c_int64)
_I32P = C.POINTER(C.c_int32)
_U8P = C.POINTER(C.c_uint8)


class _GraphDesc(C.Structure):
    _fields_ = [("n_tensors", C.c_int64), ("tensor_names", C.c_char_p),
                ("tensor_ndim", _I32P), ("tensor_dims", _I64P), ("tensor_flags", _U8P),
                ("n_nodes", C.c_int64), ("node_ids", C.c_char_p), ("node_kind", _I32P),
                ("node_nin", _I32P), ("node_nout", _I32P), ("node_inputs", C.c_char_p),
                ("node_outputs", C.c_char_p), ("node_nattr", _I32P), ("node_attrs", _I64P),
                ("node_device", _I32P), ("node_seq", _I64P), ("n_inputs", C.c_int64),
                ("input_names", C.c_char_p), ("tensor_names_len", C.c_int64),
                ("node_ids_len", C.c_int64), ("node_inputs_len", C.c_int64),
                ("node_outputs_len", C.c_int64), ("input_names_len", C.c_int64)]


class _LineageDesc(C.Structure):
    _fields_ = [("n_entries", C.c_int64), ("logical_names", C.c_char_p), ("mode", _U8P),
                ("n_shards", _I32P), ("shard_names", C.c_char_p), ("shard_ndim", _I32P),
                ("ranges", _I64P)]


def _bind(lib):
    if getattr(lib, "_pqw_plan_bound", False):
        return lib
    vp = C.c_void_p
    lib.pqw_plan_create.argtypes = [C.POINTER(_GraphDesc), C.POINTER(_GraphDesc),
                                    C.POINTER(_LineageDesc), _I64P, C.c_size_t,
                                    C.POINTER(vp)]
    lib.pqw_plan_create.restype = C.c_int
    lib.pqw_plan_destroy.argtypes = [vp]
    lib.pqw_plan_destroy.restype = None
    lib.pqw_plan_validate.argtypes = [vp]
    lib.pqw_plan_validate.restype = C.c_int
    lib.pqw_plan_check_lineage.argtypes = [vp, _I64P]
    lib.pqw_plan_check_lineage.restype = C.c_int
    lib.pqw_plan_build_stages.argtypes = [vp, _I64P]
    lib.pqw_plan_build_stages.restype = C.c_int
    lib.pqw_plan_stage_target.argtypes = [vp, C.c_int]
    lib.pqw_plan_stage_target.restype = C.c_int
    lib.pqw_plan_stage_nodes.argtypes = [vp, C.c_int, C.c_int, _I32P, C.c_size_t]
    lib.pqw_plan_stage_nodes.restype = C.c_long
    lib.pqw_plan_uncovered.argtypes = [vp, C.c_int, _I32P, C.c_size_t]
    lib.pqw_plan_uncovered.restype = C.c_long
    lib.pqw_plan_add_stages.argtypes = [vp, vp, C.c_uint64, _I32P, C.c_size_t, _I32P]
    lib.pqw_plan_add_stages.restype = C.c_int
    lib.pqw_plan_stage_program.argtypes = [vp, C.c_int, C.c_uint64, _I32P, C.c_size_t, _I64P,
                                           C.c_size_t, C.POINTER(C.c_uint64), C.c_size_t, _I64P]
    lib.pqw_plan_stage_program.restype = C.c_int
    lib._pqw_plan_bound = True
    return lib


class PlanDeclined(Exception):
    """The native core does not take this plan; run the Python host code."""


class _Consts:
    """Distinct rational attributes of a plan (Fraction-keyed, like _Lowerer.const)."""

    def __init__(self):
        self.idx: dict[tuple[int, int], int] = {}
        self.triples: list[tuple[int, int, int]] = []

    def __call__(self, v) -> int:
        q = Fraction(v)
        key = (q.numerator, q.denominator)
        got = self.idx.get(key)
        if got is None:
            got = len(self.triples)
            self.triples.append(F.const_triple(q))
            self.idx[key] = got
        return got


def _shape_words(s) -> list[int]:
    return [len(s), *map(int, s)]


def _reduce_words(a) -> list[int]:
    axes = a.get("axes")
    keep = 1 if a.get("keepdims") else 0
    if axes is None:
        return [keep, 0]
    return [keep, 1, len(axes), *map(int, axes)]


_ENC = {
    "scale": lambda a, c: [c(a["factor"])],
    "shift": lambda a, c: [c(a["addend"])],
    "full": lambda a, c: [c(a["value"]), *_shape_words(a["shape"])],
    "pow": lambda a, c: [int(a.get("exponent", 0))],
    "div": lambda a, c: [1 if a.get("den_positive") else 0],
    "softmax": lambda a, c: [int(a.get("axis", -1))],
    "create_mask": lambda a, c: [int(a["size"])],
    "transpose": lambda a, c: [int(p) for p in a["perm"]],
    "view": lambda a, c: _shape_words(a["shape"]),
    "expand": lambda a, c: _shape_words(a["shape"]),
    "embedding_grad": lambda a, c: [int(a["vocab"])],
    "sum": lambda a, c: _reduce_words(a),
    "mean": lambda a, c: _reduce_words(a),
    "einsum": lambda a, c: [len(a["spec"]), *map(ord, a["spec"])],
    "chunk": lambda a, c: [int(a["axis"]), int(a["parts"]), int(a["index"])],
    "all_reduce": lambda a, c: [len(a["group"])],
    "all_gather": lambda a, c: [len(a["group"]), int(a["axis"])],
    "reduce_scatter": lambda a, c: [len(a["group"]), int(a["axis"])],
    "all_to_all": lambda a, c: [len(a["group"]), int(a["split_axis"]), int(a["concat_axis"])],
}


_KIND = defaultdict(lambda: -1, OPCODE)
_NONE_TO_M1 = {None: -1}


def _joined(names) -> bytes:
    return ("\0".join(names) + "\0").encode()


def _zjoin(names, n: int) -> bytes:
    """n names, each NUL-terminated (empty for n == 0, so slices concatenate)."""
    return _joined(names) if n else b""


_CONST_KINDS = (OPCODE["scale"], OPCODE["shift"], OPCODE["full"])


def _pack_tensors(tv: list) -> dict:
    nt = len(tv)
    shapes = list(map(attrgetter("shape"), tv))
    flags = np.zeros(nt, np.uint8)
    is_int = np.fromiter(map("int".__eq__, map(attrgetter("dtype"), tv)), np.bool_, nt)
    for i in np.flatnonzero(is_int).tolist():
        flags[i] = 1 | (2 if tv[i].meta.get("enum") == "position" else 0)
    return dict(ndim=np.fromiter(map(len, shapes), np.int32, nt),
                dims=np.fromiter(chain.from_iterable(shapes), np.int64), flags=flags)


def _pack_nodes(nodes: list) -> dict:
    """Columns of a node slice; rational attributes get slice-local constant ids
    (the "consts" list of (num, den) keys), remapped to plan ids by the caller."""
    nn = len(nodes)
    consts = _Consts()
    kinds = list(map(attrgetter("kind"), nodes))
    ins = list(map(attrgetter("inputs"), nodes))
    outs = list(map(attrgetter("outputs"), nodes))
    nattr = [0] * nn
    words: list[int] = []
    attrs = list(map(attrgetter("attrs"), nodes))
    for i, enc in enumerate(map(_ENC.get, kinds)):
        if enc is not None:
            w = enc(attrs[i], consts)
            nattr[i] = len(w)
            words.extend(w)
    devs = list(map(attrgetter("device"), nodes))
    nin = np.fromiter(map(len, ins), np.int32, nn)
    nout = np.fromiter(map(len, outs), np.int32, nn)
    return dict(kind=np.fromiter(map(_KIND.__getitem__, kinds), np.int32, nn), nin=nin,
                nout=nout, nattr=np.array(nattr, dtype=np.int32),
                attrs=np.array(words, dtype=np.int64),
                device=np.fromiter(map(_NONE_TO_M1.get, devs, devs), np.int32, nn),
                seq=np.fromiter(map(attrgetter("seq"), nodes), np.int64, nn),
                ids=_zjoin(map(attrgetter("id"), nodes), nn),
                ins=_zjoin(chain.from_iterable(ins), int(nin.sum())),
                outs=_zjoin(chain.from_iterable(outs), int(nout.sum())),
                consts=list(consts.idx))


def _ext():
    try:
        from . import _pqw_pack
        return _pqw_pack
    except ImportError:
        return None


def _pack_columns(g: Graph, consts: _Consts) -> tuple[dict, tuple[int, int, int]]:
    """Flat columns of a graph: through the C++ packer (csrc/pack.cpp) when it
    is built, else the Python restatement above."""
    ext = _ext()
    if ext is not None:
        d = ext.pack_graph(g, OPCODE, lambda v: consts(v))
        cols = {k: d[k] for k in ("tn", "ids", "ins", "outs", "inputs")}
        for k, dt in (("ndim", np.int32), ("dims", np.int64), ("flags", np.uint8),
                      ("kind", np.int32), ("nin", np.int32), ("nout", np.int32),
                      ("nattr", np.int32), ("attrs", np.int64), ("device", np.int32),
                      ("seq", np.int64)):
            cols[k] = np.frombuffer(d[k], dtype=dt)
        return cols, d["counts"]
    tv = list(g.tensors.values())
    t = _pack_tensors(tv)
    t["tn"] = _zjoin(g.tensors, len(tv))  # the dict keys: what node inputs name
    n = _pack_nodes(g.nodes)
    if n["consts"]:  # slice-local constant ids -> plan ids
        remap = np.array([consts(Fraction(a, b)) for a, b in n["consts"]], dtype=np.int64)
        off = np.cumsum(n["nattr"], dtype=np.int64) - n["nattr"]
        at = off[np.isin(n["kind"], _CONST_KINDS) & (n["nattr"] > 0)]
        n["attrs"][at] = remap[n["attrs"][at]]
    cols = {**t, **n, "inputs": _zjoin(g.inputs, len(g.inputs))}
    return cols, (len(tv), len(g.nodes), len(g.inputs))


def _pack_graph(g: Graph, consts: _Consts, keep: list) -> _GraphDesc:
    cols, (nt, nn, ng) = _pack_columns(g, consts)
    arrs = {k: np.ascontiguousarray(cols[k] if cols[k].size else np.zeros(1, cols[k].dtype))
            for k in ("ndim", "dims", "flags", "kind", "nin", "nout", "nattr", "attrs",
                      "device", "seq")}
    strs = {k: cols[k] or b"\0" for k in ("tn", "ids", "ins", "outs", "inputs")}
    keep.append((arrs, strs))

    def p(a, t):
        return a.ctypes.data_as(t)
    return _GraphDesc(nt, strs["tn"], p(arrs["ndim"], _I32P), p(arrs["dims"], _I64P),
                      p(arrs["flags"], _U8P), nn, strs["ids"], p(arrs["kind"], _I32P),
                      p(arrs["nin"], _I32P), p(arrs["nout"], _I32P), strs["ins"], strs["outs"],
                      p(arrs["nattr"], _I32P), p(arrs["attrs"], _I64P), p(arrs["device"], _I32P),
                      p(arrs["seq"], _I64P), ng, strs["inputs"],
                      *(_names_len(strs[k]) for k in ("tn", "ids", "ins", "outs", "inputs")))


def _names_len(b) -> int:
    """Byte length of a NUL-joined names buffer through its last NUL (the
    library then need not scan for it), 0 when unknown."""
    return len(b) if isinstance(b, (bytes, bytearray)) and (not b or b[-1] == 0) else 0


def _lineage_columns(lineage) -> tuple:
    """(mode, n_shards, sdim, ranges, (names, shard names)) of a lineage: through
    the C++ packer when it is built, else in Python."""
    ext = _ext()
    if ext is not None and hasattr(ext, "pack_lineage") and isinstance(lineage, dict):
        d = ext.pack_lineage(lineage)
        return (np.frombuffer(d["mode"], np.uint8), np.frombuffer(d["n_shards"], np.int32),
                np.frombuffer(d["sdim"], np.int32), np.frombuffer(d["ranges"], np.int64),
                (d["names"], d["shard_names"]))
    entries = list(lineage.values())
    mode = np.array([0 if e.mode == "full" else 1 if e.mode == "partial" else 2 for e in entries]
                    or [0], dtype=np.uint8)
    n_sh = np.array([len(e.shards) for e in entries] or [0], dtype=np.int32)
    shards = [s for e in entries for s in e.shards]
    sdim = np.array([len(s.ranges) for s in shards] or [0], dtype=np.int32)
    ranges = np.fromiter(chain.from_iterable(chain.from_iterable(s.ranges) for s in shards),
                         np.int64)
    return mode, n_sh, sdim, ranges, (_joined(lineage), _joined(s.tensor for s in shards))


def _pack_lineage(lineage, keep: list) -> _LineageDesc:
    mode, n_sh, sdim, ranges, strs = _lineage_columns(lineage)
    n = len(lineage)
    mode, n_sh, sdim = (a if a.size else np.zeros(1, a.dtype) for a in (mode, n_sh, sdim))
    if not ranges.size:
        ranges = np.zeros(2, np.int64)
    strs = tuple(x or b"\0" for x in strs)
    keep.append((mode, n_sh, sdim, ranges, strs))
    return _LineageDesc(n, strs[0], mode.ctypes.data_as(_U8P),
                        n_sh.ctypes.data_as(_I32P), strs[1], sdim.ctypes.data_as(_I32P),
                        ranges.ctypes.data_as(_I64P))


class NativePlan:
    """A plan inside the native core. Raises PlanDeclined when it cannot be
    packed (the Python host code then handles the plan)."""

    def __init__(self, plan: Plan):
        self.lib = _bind(load_library())
        self.plan = plan
        self.h = C.c_void_p()
        keep: list = []
        consts = _Consts()
        try:
            lg = _pack_graph(plan.logical, consts, keep)
            pg = _pack_graph(plan.parallel, consts, keep)
            ln = _pack_lineage(plan.lineage, keep)
        except (KeyError, TypeError, ValueError, OverflowError, AttributeError,
                ZeroDivisionError, UnicodeError) as e:
            raise PlanDeclined(f"plan not packable: {type(e).__name__}: {e}") from e
        tri = np.array(consts.triples or [(0, 0, 0)], dtype=np.int64).reshape(-1, 3)
        rc = self.lib.pqw_plan_create(C.byref(lg), C.byref(pg), C.byref(ln),
                                      tri.ctypes.data_as(_I64P), len(consts.triples),
                                      C.byref(self.h))
        if rc < 0:
            raise EngineError(self.lib.pqw_last_error().decode(errors="replace"))
        self.n_stages = 0
        self._ltensors: list[str] | None = None
        self._ptensors: list[str] | None = None

    def close(self):
        if self.h:
            self.lib.pqw_plan_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _err(self) -> str:
        return self.lib.pqw_last_error().decode(errors="replace")

    def validate(self) -> bool:
        """validate_concrete on both graphs; False: the plan is not well formed."""
        rc = self.lib.pqw_plan_validate(self.h)
        if rc == E_PLAN:
            self.declined = self._err()
            return False
        if rc < 0:
            raise EngineError(self._err())
        return True

    def lineage_clean(self) -> bool:
        """True iff validate_lineage would report no problem (else the host's
        validate_lineage gives the reference's messages)."""
        out = (C.c_int64 * 2)()
        if self.lib.pqw_plan_check_lineage(self.h, out) < 0:
            raise EngineError(self._err())
        return out[0] == 0 and out[1] == 0

    def build_stages(self) -> bool:
        """Stage construction; False: stage construction would raise."""
        out = (C.c_int64 * 3)()
        rc = self.lib.pqw_plan_build_stages(self.h, out)
        if rc == E_PLAN:
            self.declined = self._err()
            return False
        if rc < 0:
            raise EngineError(self._err())
        self.n_stages = int(out[0])
        self._n_unc = (int(out[1]), int(out[2]))
        return True

    def _ints(self, fn, *args) -> np.ndarray:
        n = fn(self.h, *args, None, 0)
        if n < 0:
            raise EngineError(self._err())
        buf = np.empty(max(int(n), 1), dtype=np.int32)
        fn(self.h, *args, buf.ctypes.data_as(_I32P), buf.size)
        return buf[: int(n)]

    def ltensor_names(self) -> list[str]:
        if self._ltensors is None:
            self._ltensors = list(self.plan.logical.tensors)
        return self._ltensors

    def ptensor_names(self) -> list[str]:
        if self._ptensors is None:
            self._ptensors = list(self.plan.parallel.tensors)
        return self._ptensors

    def target(self, i: int) -> str:
        t = self.lib.pqw_plan_stage_target(self.h, i)
        if t < 0:
            raise EngineError(self._err())
        return self.ltensor_names()[t]

    def targets(self) -> list[str]:
        names = self.ltensor_names()
        return [names[self.lib.pqw_plan_stage_target(self.h, i)] for i in range(self.n_stages)]

    def stage_nodes(self, i: int, side: int) -> np.ndarray:
        return self._ints(self.lib.pqw_plan_stage_nodes, i, side)

    def uncovered(self) -> dict[str, list[str]]:
        lg, pg = self.plan.logical.nodes, self.plan.parallel.nodes
        return {"logical": [lg[i].id for i in self._ints(self.lib.pqw_plan_uncovered, 0)],
                "parallel": [pg[i].id for i in self._ints(self.lib.pqw_plan_uncovered, 1)]}

    def stage(self, i: int) -> Stage:
        """Stage i as the host's Stage record (slices, boundaries; assumed and
        owned lists are left empty -- see stages() for the full records)."""
        lg, pg = self.plan.logical.nodes, self.plan.parallel.nodes
        ln, pn = self.ltensor_names(), self.ptensor_names()
        return Stage(self.target(i), [lg[v] for v in self.stage_nodes(i, 0)],
                     [pg[v] for v in self.stage_nodes(i, 1)],
                     [ln[t] for t in self.stage_nodes(i, 2)],
                     [pn[t] for t in self.stage_nodes(i, 3)], [])

    def stages(self) -> list[Stage]:
        """Every stage with the fields stages.build_stages fills (assumed
        checkpoints, owned node ids), computed from the native slices."""
        from .stages import entry_order, shard_owner
        order = entry_order(self.plan)
        rank = {t: i for i, t in enumerate(order)}
        owner = shard_owner(self.plan, order)
        out: list[Stage] = []
        claimed_l: set[str] = set()
        claimed_p: set[str] = set()
        for i in range(self.n_stages):
            st = self.stage(i)
            st.assumed = sorted(set(st.l_inputs) | {owner[b] for b in st.p_inputs}, key=rank.get)
            st.owned_logical = sorted(n.id for n in st.logical_nodes if n.id not in claimed_l)
            claimed_l.update(st.owned_logical)
            st.owned_parallel = sorted(n.id for n in st.parallel_nodes if n.id not in claimed_p)
            claimed_p.update(st.owned_parallel)
            out.append(st)
        return out

    def add_stages(self, eng: Engine, seed: int, which: list[int] | None = None) -> np.ndarray:
        """Lower stages (all, or the listed ones) into `eng`; per stage its engine
        index, or E_PLAN where the host's lowering raises."""
        if which is None:
            n, ptr = self.n_stages, None
        else:
            arr = np.asarray(which, dtype=np.int32)
            n, ptr = arr.size, arr.ctypes.data_as(_I32P)
        idx = np.empty(max(n, 1), dtype=np.int32)
        rc = self.lib.pqw_plan_add_stages(self.h, eng._h, seed & F.MASK64, ptr, n,
                                          idx.ctypes.data_as(_I32P))
        if rc < 0:
            raise EngineError(self._err())
        idx = idx[:n]
        eng.n_stages += int((idx >= 0).sum())
        return idx

    def stage_program(self, i: int, seed: int) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """(ir, consts, var_keys) of stage i -- stages.lower_stage's output."""
        lens = (C.c_int64 * 3)()
        rc = self.lib.pqw_plan_stage_program(self.h, i, seed & F.MASK64, None, 0, None, 0, None,
                                             0, lens)
        if rc == E_PLAN:
            raise PlanDeclined(self._err())
        if rc < 0:
            raise EngineError(self._err())
        ir = np.empty(max(lens[0], 1), np.int32)
        cs = np.empty((max(lens[1], 1), 3), np.int64)
        vk = np.empty(max(lens[2], 1), np.uint64)
        self.lib.pqw_plan_stage_program(self.h, i, seed & F.MASK64, ir.ctypes.data_as(_I32P),
                                        ir.size, cs.ctypes.data_as(_I64P), cs.shape[0],
                                        vk.ctypes.data_as(C.POINTER(C.c_uint64)), vk.size, lens)
        return ir[: lens[0]], cs[: lens[1]], vk[: lens[2]]

"""The C-ABI library loads on a CPU-only host and exports every declared symbol."""

import ctypes
import os
import re

from paper_2506_15961_b200 import engine

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "planeq_witness.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(pqw_\w+)\s*\(", text, re.M)))


def test_header_and_binding_agree(lib):
    decl = declared_functions()
    assert decl, "no functions parsed from the header"
    assert sorted(engine.EXPORTS) == decl


def test_every_symbol_exported(lib):
    raw = ctypes.CDLL(engine.LIB_PATH)
    for name in declared_functions():
        assert hasattr(raw, name), name


def test_abi_and_device_count_without_gpu(lib):
    assert lib.pqw_abi_version() == engine.ABI_VERSION
    assert engine.device_count() >= 0


def test_compile_only_works_without_device(lib):
    import numpy as np
    from paper_2506_15961_b200.stages import IR_MAGIC, OPCODE, T_CHECK, T_VARS
    # x (2 vars) ; y = x + x ; check y == scale(x, 2)
    consts = np.array([[2, 2, 1]], dtype=np.int64)
    ir = [IR_MAGIC, 3, 4, 2, 1, 2, 1, 2, 1, 2,
          T_VARS, 0, 1, 1, 0, 0,
          OPCODE["add"], 2, 1, 0, 0, 0, 1,
          OPCODE["scale"], 1, 1, 1, 0, 2, 0]
    ir += [T_CHECK, 2, 0, 1, 1, 2, 0]
    e = engine.Engine(0, 1, (1, 2, 3))
    c = e.add_stage(np.array(ir, dtype=np.int32), consts, np.array([5, 6], dtype=np.uint64))
    assert c.obligations == 2 and c.status in (engine.STAGE_OK, engine.STAGE_PROVEN)
    code, slots = e.bytecode(c.index)
    assert code[-1, 0] == 0  # END
    e.close()


def test_malformed_program_is_rejected(lib):
    import numpy as np
    import pytest
    from paper_2506_15961_b200.errors import EngineError
    e = engine.Engine(0, 1, (1, 2, 3))
    with pytest.raises(EngineError):
        e.add_stage(np.array([1, 2, 3], dtype=np.int32), np.zeros((0, 3), np.int64),
                    np.zeros(0, np.uint64))
    e.close()


def test_compilation_is_deferred_and_status_resolves(lib):
    """pqw_stage_add only queues the program (status PENDING); the first
    status query compiles every pending stage; identical texts share one
    compiled program."""
    import ctypes as C
    import numpy as np
    from paper_2506_15961_b200.stages import IR_MAGIC, OPCODE, T_CHECK, T_VARS
    consts = np.array([[2, 2, 1]], dtype=np.int64)
    ir = np.array([IR_MAGIC, 3, 4, 2, 1, 2, 1, 2, 1, 2,
                   T_VARS, 0, 1, 1, 0, 0,
                   OPCODE["add"], 2, 1, 0, 0, 0, 1,
                   OPCODE["scale"], 1, 1, 1, 0, 2, 0,
                   T_CHECK, 2, 0, 1, 1, 2, 0], dtype=np.int32)
    e = engine.Engine(0, 1, (1, 2, 3))
    raw = np.zeros(16, dtype=np.int64)
    keys = np.array([5, 6], dtype=np.uint64)
    idx = e.lib.pqw_stage_add(e._h, ir.ctypes.data_as(C.POINTER(C.c_int32)), ir.size,
                              consts.ctypes.data_as(C.POINTER(C.c_int64)), 1,
                              keys.ctypes.data_as(C.POINTER(C.c_uint64)), 2,
                              raw.ctypes.data_as(C.POINTER(C.c_int64)))
    assert idx == 0 and raw[0] == engine.STAGE_PENDING and raw[13] == 2
    e.n_stages += 1
    dup = e.add_stage(ir, consts, keys)              # same text: a cache hit
    a, b = e.stage_status(0), dup
    assert a.status == b.status and a.obligations == b.obligations == 2
    assert e.image_stats()["cache_hits"] == 1
    e.close()


def test_front_end_errors_surface_at_status(lib):
    import numpy as np
    import pytest
    from paper_2506_15961_b200.errors import EngineError
    from paper_2506_15961_b200.stages import IR_MAGIC
    e = engine.Engine(0, 1, (1, 2, 3))
    # a valid header followed by a truncated op stream
    c = e.add_stage(np.array([IR_MAGIC, 1, 1, 0, 1, 2, 99], dtype=np.int32),
                    np.zeros((0, 3), np.int64), np.zeros(0, np.uint64))
    with pytest.raises(EngineError):
        _ = c.status
    e.close()


def _scale_check_program(c_lhs, c_rhs):
    """x (2 vars); obligations scale(x, c_lhs) == scale(x, c_rhs) (c = None: x itself)."""
    import numpy as np
    from paper_2506_15961_b200 import field as F
    from paper_2506_15961_b200.stages import IR_MAGIC, OPCODE, T_CHECK, T_VARS
    consts, ops, n_t = [], [T_VARS, 0, 1, 1, 0, 0], 1
    sides = []
    for c in (c_lhs, c_rhs):
        if c is None:
            sides.append(0)
            continue
        consts.append(F.const_triple(c))
        ops += [OPCODE["scale"], 1, 1, 1, 0, n_t, len(consts) - 1]
        sides.append(n_t)
        n_t += 1
    ops += [T_CHECK, 2, 0, 1, sides[0], sides[1], 0]
    head = [IR_MAGIC, n_t, 1 + sum(c is not None for c in (c_lhs, c_rhs)) + 1, 2]
    ir = head + [1, 2] * n_t + ops
    return (np.array(ir, dtype=np.int32), np.array(consts or [(0, 0, 0)], dtype=np.int64)[:len(consts)],
            np.array([5, 6], dtype=np.uint64))


def test_constants_that_collide_mod_p_are_not_decided(lib):
    """Distinct exact constants with one image in F_p (or a nonzero multiple of
    p): the field cannot separate what they scale, so the stage is LOSSY
    (reported unknown) instead of closing or passing as equal."""
    P = (1 << 31) - 1
    e = engine.Engine(0, 1, (1, 2, 3))
    for lhs, rhs in ((1, 1 - P), (P, 0), (2, 2 + P)):
        c = e.add_stage(*_scale_check_program(lhs, rhs))
        assert c.status == engine.STAGE_LOSSY, (lhs, rhs)
    # the same constant on both sides still closes at compile time
    c = e.add_stage(*_scale_check_program(3, 3))
    assert c.status == engine.STAGE_PROVEN
    e.close()


def test_identities_fold_on_exact_values(lib):
    """x * c with c congruent to 1 mod p but not 1 is not folded to x: no
    compile-time proof of x == scale(x, 1 - p)."""
    P = (1 << 31) - 1
    e = engine.Engine(0, 1, (1, 2, 3))
    c = e.add_stage(*_scale_check_program(None, 1 - P))
    assert c.status != engine.STAGE_PROVEN
    c = e.add_stage(*_scale_check_program(None, 1))
    assert c.status == engine.STAGE_PROVEN
    e.close()

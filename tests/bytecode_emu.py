"""TEST INFRASTRUCTURE ONLY: numpy emulation of the engine's scalar bytecode.

Lets the CPU test suite check the host compiler's output (straight-line F_p
bytecode, exported through pqw_stage_bytecode) against the independent oracle
without a GPU. Semantics mirror the device interpreter in
paper_2506_15961_b200/csrc/witness_kernel.cu (run_item); the product never
calls this.
"""

from __future__ import annotations

import numpy as np

from oracle import m31

OPS = ("END", "CONST", "VAR", "ADD", "SUB", "MUL", "NEG", "DIV", "HASH", "ACC_MUL", "ACC_MAC",
       "ACC_LD", "ACC_ADD", "ACC_ST", "CHK", "DEN", "ACC_MACF", "INV", "ACC_MUL2", "ACC_MAC2")
FN = ("EXP", "RSQRT", "SIGMOID")


def run(code: np.ndarray, n_slots: int, var_keys: np.ndarray, var_base: int, seed: int,
        witnesses: np.ndarray):
    """Returns (valid mask [W], first bad obligation per witness [W] or -1)."""
    W = len(witnesses)
    slots = np.zeros((max(n_slots, 1), W), dtype=np.uint64)
    valid = np.ones(W, dtype=bool)
    bad = np.full(W, -1, dtype=np.int64)
    acc = np.zeros(W, dtype=object)
    w1 = np.asarray(witnesses, dtype=np.uint64) + np.uint64(1)
    for op, dst, a, b in code:
        name = OPS[op]
        if name == "END":
            break
        if name == "CONST":
            slots[dst] = a
        elif name == "VAR":
            key = np.uint64(var_keys[a])  # VAR operands are stage-relative
            with np.errstate(over="ignore"):
                slots[dst] = m31.to_field(m31.mix64(key + w1 * m31.GOLDEN))
        elif name == "ADD":
            slots[dst] = m31.add(slots[a], slots[b])
        elif name == "SUB":
            slots[dst] = m31.sub(slots[a], slots[b])
        elif name == "MUL":
            slots[dst] = m31.mul(slots[a], slots[b])
        elif name == "NEG":
            slots[dst] = (m31.P - slots[a]) % m31.P
        elif name == "DIV":
            slots[dst] = m31.mul(slots[a], m31.inv(slots[b]))
        elif name == "INV":
            slots[dst] = m31.inv(slots[a])
        elif name == "HASH":
            slots[dst] = m31.uf(seed, FN[b], slots[a])
        elif name == "ACC_LD":
            acc = slots[a].astype(object)
        elif name == "ACC_ADD":
            acc = acc + slots[a].astype(object)
        elif name == "ACC_MUL":
            acc = slots[a].astype(object) * slots[b].astype(object)
        elif name in ("ACC_MAC", "ACC_MACF"):
            if name == "ACC_MACF":
                acc = np.array([(int(v) & m31.PI) + (int(v) >> 31) for v in acc], dtype=object)
            acc = acc + slots[a].astype(object) * slots[b].astype(object)
            assert all(int(v) < (1 << 64) for v in acc), "accumulator overflow"
        elif name == "ACC_MUL2":
            c, d = dst & 0xFFFF, dst >> 16
            acc = slots[a].astype(object) * slots[b].astype(object) + \
                slots[c].astype(object) * slots[d].astype(object)
            assert all(int(v) < (1 << 64) for v in acc), "accumulator overflow"
        elif name == "ACC_MAC2":
            c, d = dst & 0xFFFF, dst >> 16
            acc = np.array([(int(v) & m31.PI) + (int(v) >> 31) for v in acc], dtype=object)
            acc = acc + slots[a].astype(object) * slots[b].astype(object) + \
                slots[c].astype(object) * slots[d].astype(object)
            assert all(int(v) < (1 << 64) for v in acc), "accumulator overflow"
        elif name == "ACC_ST":
            slots[dst] = np.array([int(v) % m31.PI for v in acc], dtype=np.uint64)
        elif name == "CHK":
            diff = slots[a] != slots[b]
            newbad = diff & (bad < 0)
            bad[newbad] = dst
        elif name == "DEN":
            valid &= slots[a] != 0
        else:
            raise ValueError(name)
    return valid, bad

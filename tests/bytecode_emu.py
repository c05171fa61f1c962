"""TEST INFRASTRUCTURE ONLY: numpy emulation of the engine's cooperative bytecode.

Lets the CPU test suite check the host compiler's output (barrier-phased F_p
bytecode, one stream per warp, exported through pqw_stage_bytecode) against
the independent oracle without a GPU. Semantics mirror the device interpreter
in paper_2506_15961_b200/csrc/interp.cuh (run_stream / eval_kernel): the warps
of one phase run in arbitrary order (here: warp 0 first, then 1, ...; the test
also runs them in reverse to catch cross-warp hazards), each with its own
64-bit accumulator, all sharing one value file. The product never calls this.
"""

from __future__ import annotations

import numpy as np

from oracle import m31

OPS = ("END", "CONST", "VAR", "ADD", "SUB", "MUL", "NEG", "DIV", "HASH", "ACC_MUL", "ACC_MAC",
       "ACC_LD", "ACC_ADD", "ACC_ST", "CHK", "DEN", "ACC_MACF", "INV", "ACC_MUL2", "ACC_MAC2",
       "BAR")
FN = ("EXP", "RSQRT", "SIGMOID")


def streams(code: np.ndarray, n_warps: int) -> list[list[list[tuple]]]:
    """Split a cooperative program into per-warp lists of phases."""
    flat = code.reshape(-1)
    table = [int(x) for x in flat[:n_warps]]
    out = []
    for w in range(n_warps):
        pc = table[w]
        phases, cur = [], []
        while True:
            op, d, a, b = (int(x) for x in code[pc])
            pc += 1
            if OPS[op] in ("BAR", "END"):
                phases.append(cur)
                cur = []
                if OPS[op] == "END":
                    break
                continue
            cur.append((op, d, a, b))
        out.append(phases)
    return out


def run(code: np.ndarray, n_slots: int, var_keys: np.ndarray, var_base: int, seed: int,
        witnesses: np.ndarray, n_warps: int = 8, reverse: bool = False):
    """Returns (valid mask [W], first bad obligation per witness [W] or -1)."""
    W = len(witnesses)
    slots = np.zeros((max(n_slots, 1), W), dtype=np.uint64)
    valid = np.ones(W, dtype=bool)
    bad = np.full(W, -1, dtype=np.int64)
    w1 = np.asarray(witnesses, dtype=np.uint64) + np.uint64(1)
    per_warp = streams(code, n_warps)
    n_phases = len(per_warp[0])
    assert all(len(s) == n_phases for s in per_warp), "warps disagree on the phase count"
    order = list(range(n_warps))[::-1] if reverse else list(range(n_warps))
    for ph in range(n_phases):
        for w in order:
            acc = None
            for op, dst, a, b in per_warp[w][ph]:
                name = OPS[op]
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
                    upd = diff & ((bad < 0) | (bad > dst))
                    bad[upd] = dst
                elif name == "DEN":
                    valid &= slots[a] != 0
                else:
                    raise ValueError(name)
    return valid, bad

"""TEST INFRASTRUCTURE ONLY: numpy emulation of the engine's v4 stage programs.

Lets the CPU test suite check the host compiler's output (isa.hpp programs:
one instruction stream per warp, bundles of independent ops, explicit
WAIT/SIGNAL between warps; exported through pqw_stage_bytecode) against the
independent oracle without a GPU. Semantics mirror the device interpreter in
paper_2506_15961_b200/csrc/interp.cuh: all warps share one value file; a warp
blocked in WAIT does not advance. The warps are interleaved instruction by
instruction under a chosen policy -- "random" (seeded), "ahead" (run the
lowest runnable warp until it blocks) or "behind" (the highest) -- so a
missing wait (a read before the producer wrote, or a slot overwritten before
its last reader read it) shows up as a wrong value under some policy. The
product never calls this.
"""

from __future__ import annotations

import numpy as np

from oracle import m31

OPS = ("END", "DOT", "SUM", "SUB", "NEG", "HASH", "INV", "VAR", "CONST", "CHK", "DEN",
       "FILL", "SPILL", "WAIT", "SIGNAL")
FN = ("EXP", "RSQRT", "SIGMOID")
SLOT = 128
GROUP = 8


def fields(op: str, k: int) -> int:
    return {"DOT": 1 + 2 * k, "SUM": 1 + k, "SUB": 3, "CHK": 3, "NEG": 2, "HASH": 2, "INV": 2,
            "VAR": 2, "CONST": 2, "FILL": 2, "SPILL": 2, "DEN": 1}.get(op, 0)


def decode(code: np.ndarray, n_warps: int) -> list[list[tuple]]:
    """Per warp: list of (op, fn, k, aux, signal, cols) where cols[f] is the u32
    array of field f over the bundle's n ops and signal the progress published
    after the bundle (header.w; for WAIT: a second wait, 0 for none; a WAIT's
    third wait, header.y, is returned as k)."""
    flat = code.reshape(-1)
    out = []
    for w in range(n_warps):
        pc = int(flat[w])
        ins = []
        while True:
            h = code[pc]
            pc += 1
            op = OPS[int(h[0]) & 0xFF]
            fn = (int(h[0]) >> 8) & 0xFF
            k = int(h[0]) >> 16
            n = int(h[1])
            aux = int(h[2])
            sig = int(h[3])
            if op == "WAIT":  # header.y of a WAIT is its third wait, not an op count
                k, n = n, 0
            elif n >> 13:  # a second folded wait in header.y >> 13: (warp + 1) << 13 | count
                w2 = n >> 13
                aux = [aux, ((w2 >> 13) << 24) | (w2 & 0x1FFF)]
                n &= 0x1FFF
            nf = fields(op, k)
            ng = (n + GROUP - 1) // GROUP
            cols = [np.zeros(ng * GROUP, dtype=np.int64) for _ in range(nf)]
            for g in range(ng):
                for f in range(nf):
                    rec = code[pc:pc + 2].reshape(-1)
                    cols[f][g * GROUP:(g + 1) * GROUP] = rec
                    pc += 2
            cols = [c[:n] for c in cols]
            ins.append((op, fn, k, aux, sig, cols))
            if op == "END":
                break
        out.append(ins)
    return out


def run(code: np.ndarray, n_slots: int, var_keys: np.ndarray, var_base: int, seed: int,
        witnesses: np.ndarray, n_warps: int = 16, policy: str = "random", rng_seed: int = 0,
        n_spill: int | None = None):
    """Returns (valid mask [W], first bad obligation per witness [W] or -1)."""
    W = len(witnesses)
    streams = decode(code, n_warps)
    if n_spill is None:  # global spill slots the program addresses
        n_spill = 1 + max([int(c.max()) // SLOT for st in streams
                           for op, _f, _k, _a, _s, cols in st if op in ("FILL", "SPILL")
                           for c in (cols[1] if op == "FILL" else cols[0],) if len(c)] or [0])
    sm = np.zeros((max(n_slots, 1), W), dtype=np.uint64)
    gm = np.zeros((max(n_spill, 1), W), dtype=np.uint64)
    valid = np.ones(W, dtype=bool)
    bad = np.full(W, -1, dtype=np.int64)
    w1 = np.asarray(witnesses, dtype=np.uint64) + np.uint64(1)
    pc = [0] * n_warps
    prog = [0] * n_warps
    rng = np.random.default_rng(rng_seed)
    P = np.uint64(m31.PI)

    def s(off):
        assert off % SLOT == 0
        return int(off) // SLOT

    def runnable(w):
        op, fn, k, aux, sig, cols = streams[w][pc[w]]
        if op == "END":
            return False
        if op == "WAIT":  # up to three waits (aux, sig, k): (warp + 1) << 24 | progress
            return all(not x or prog[(x >> 24) - 1] >= (x & 0xFFFFFF) for x in (aux, sig, k))
        if aux:  # one or two waits folded into the bundle header
            return all(prog[(a >> 24) - 1] >= (a & 0xFFFFFF)
                       for a in (aux if isinstance(aux, list) else [aux]))
        return True

    def step(w):
        nonlocal valid
        op, fn, k, aux, sig, cols = streams[w][pc[w]]
        pc[w] += 1
        n = len(cols[0]) if cols else 0
        if op == "DOT":
            for i in range(n):
                acc = np.zeros(W, dtype=np.uint64)
                for j in range(k):
                    acc = (acc + sm[s(cols[1 + 2 * j][i])] * sm[s(cols[2 + 2 * j][i])] % P) % P
                sm[s(cols[0][i])] = acc
        elif op == "SUM":
            for i in range(n):
                acc = np.zeros(W, dtype=np.uint64)
                for j in range(k):
                    acc = (acc + sm[s(cols[1 + j][i])]) % P
                sm[s(cols[0][i])] = acc
        elif op == "SUB":
            for i in range(n):
                sm[s(cols[0][i])] = m31.sub(sm[s(cols[1][i])], sm[s(cols[2][i])])
        elif op == "NEG":
            for i in range(n):
                sm[s(cols[0][i])] = (P - sm[s(cols[1][i])]) % P
        elif op == "HASH":
            for i in range(n):
                sm[s(cols[0][i])] = m31.uf(seed, FN[fn], sm[s(cols[1][i])])
        elif op == "INV":
            # Montgomery batch inversion, exactly as the device does it
            acc = np.ones(W, dtype=np.uint64)
            for i in range(n):
                acc = acc * sm[s(cols[1][i])] % P
                sm[s(cols[0][i])] = acc
            if fn:  # the guarded operands' DEN check (their DEN ops were dropped)
                valid &= acc != 0
            inv = m31.inv(acc)
            for i in range(n - 1, 0, -1):
                prev = sm[s(cols[0][i - 1])].copy()
                a = sm[s(cols[1][i])].copy()
                sm[s(cols[0][i])] = inv * prev % P
                inv = inv * a % P
            if n:
                sm[s(cols[0][0])] = inv
        elif op == "VAR":
            for i in range(n):
                key = np.uint64(var_keys[int(cols[1][i])])  # stage-relative
                with np.errstate(over="ignore"):
                    sm[s(cols[0][i])] = m31.to_field(m31.mix64(key + w1 * m31.GOLDEN))
        elif op == "CONST":
            for i in range(n):
                sm[s(cols[0][i])] = np.uint64(int(cols[1][i]))
        elif op == "CHK":
            for i in range(n):
                diff = sm[s(cols[1][i])] != sm[s(cols[2][i])]
                o = int(cols[0][i])
                upd = diff & ((bad < 0) | (bad > o))
                bad[upd] = o
        elif op == "DEN":
            for i in range(n):
                valid &= sm[s(cols[0][i])] != 0
        elif op == "FILL":
            for i in range(n):
                sm[s(cols[0][i])] = gm[s(cols[1][i])]
        elif op == "SPILL":
            for i in range(n):
                gm[s(cols[0][i])] = sm[s(cols[1][i])]
        elif op == "WAIT":
            return
        else:
            raise ValueError(op)
        if sig:
            assert sig >= prog[w], "progress must be monotone"
            prog[w] = sig

    while True:
        live = [w for w in range(n_warps) if runnable(w)]
        if not live:
            assert all(streams[w][pc[w]][0] == "END" for w in range(n_warps)), "deadlock"
            break
        if policy == "random":
            w = int(rng.choice(live))
        elif policy == "ahead":
            w = live[0]
        else:
            w = live[-1]
        step(w)
    return valid, bad

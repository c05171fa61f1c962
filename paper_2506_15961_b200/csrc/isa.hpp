// isa.hpp -- the v4 stage-program format shared by the host back end
// (schedule.cpp), the sm_100a interpreter (interp.cuh) and, restated, the CPU
// test emulator (tests/bytecode_emu.py).
//
// A stage program is a table of NW u32 stream offsets (in 16-byte records,
// padded to whole records) followed by NW instruction streams, one per warp of
// the CTA that evaluates the stage for a tile of 32 witnesses (one per lane)
// out of one shared value file.
//
// Instruction = one header record + payload records.
//   header.x = op | fn << 8 | k << 16,  header.y = n (ops in the bundle, low
//   13 bits) | a second folded wait << 13 ((warp + 1) << 13 | progress < 2^13),
//   header.z = a wait folded into the bundle ((warp + 1) << 24 | progress; 0:
//   none), header.w = progress this warp publishes after the bundle (0: none)
//   -- a WAIT instruction carries up to three waits in that encoding, in z, w
//   and y ((producer warp + 1) << 24 | progress; 0 in w or y: none there).
// A bundle holds n independent ops of one kind. Its payload is ceil(n / 8)
// groups; a group lists, field by field, 8 u32 values (two records) for the 8
// ops of the group (unused entries of the last group are 0):
//   DOT k   D, A0, B0, ..., A(k-1), B(k-1)    d = sum_j a_j * b_j  (k = 1: multiply)
//   SUM k   D, A0, ..., A(k-1)                d = sum_j a_j        (k = 2: add)
//   SUB     D, A, B        NEG  D, A          HASH fn   D, A       (d = f_fn(a))
//   INV     D, A           batched: every d_i = a_i^-1 via one inversion (fn 1: the
//                          operands are guarded denominators; a zero product
//                          invalidates the witness, standing in for their DENs)
//   VAR     D, V (stage-relative var index)   CONST     D, C (residue)
//   CHK     O (obligation id), A, B           DEN       A
//   FILL    D, G (global spill slot -> shared)  SPILL   G, A (shared -> global)
//   WAIT    (no payload) wait until warp z has published progress >= w
//   END     end of stream
// Shared operands are byte offsets slot * 128 into the value file (slot s of
// the file is 32 consecutive u32, lane l's witness at +4l); global operands
// are byte offsets into the CTA's spill region laid out the same way.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define PQW_ISA_HD __host__ __device__
#else
#define PQW_ISA_HD
#endif

namespace pqw {

enum IsaOp : uint32_t {
  I_END = 0,
  I_DOT,
  I_SUM,
  I_SUB,
  I_NEG,
  I_HASH,
  I_INV,
  I_VAR,
  I_CONST,
  I_CHK,
  I_DEN,
  I_FILL,
  I_SPILL,
  I_WAIT,
  I_SIGNAL,
  I_NUM_OPS
};

constexpr uint32_t SLOT_BYTES = 128;  // one value for 32 witnesses
constexpr uint32_t GROUP = 8;         // ops per payload group
constexpr uint32_t MAX_K = 64;        // max pairs of a DOT / terms of a SUM

// Fields (of 8 u32 = two records) per payload group.
PQW_ISA_HD inline constexpr uint32_t isa_fields(uint32_t op, uint32_t k) {
  return op == I_DOT ? 1 + 2 * k
       : op == I_SUM ? 1 + k
       : (op == I_SUB || op == I_CHK) ? 3
       : (op == I_NEG || op == I_HASH || op == I_INV || op == I_VAR || op == I_CONST ||
          op == I_FILL || op == I_SPILL) ? 2
       : op == I_DEN ? 1
       : 0;
}

PQW_ISA_HD inline constexpr uint32_t isa_header(uint32_t op, uint32_t fn, uint32_t k) {
  return op | (fn << 8) | (k << 16);
}

}  // namespace pqw

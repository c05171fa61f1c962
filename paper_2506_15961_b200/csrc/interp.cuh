// interp.cuh -- the sm_100a bytecode interpreter (device code of witness_kernel.cu).
//
// Cooperative execution. A work item is (stage, tile of 32 witnesses). The CTA
// (NW warps) evaluates the stage for the tile's 32 witnesses -- one witness per
// lane -- out of ONE value file shared by all its warps: slot s of the file is
// 32 consecutive u32 (128 B, one conflict-free LDS/STS per warp access) in
// shared memory for s < smem_slots, or in the CTA's global spill region. The
// compiler split the stage program into NW instruction streams and into phases
// (list scheduling in depth-first order, so the live set stays that of a
// sequential evaluation): within a phase the warps' instructions are mutually
// independent, a BAR ends the phase (named CTA barrier), so the warps of the
// CTA supply the instruction-level parallelism that one witness lacks while
// the whole live set of a stage -- up to ~1600 values -- stays on chip.
//
// The grid is persistent (SMs x occupancy) and pulls items from an atomic
// counter; stages are ordered by descending cost. Decode is a warp-uniform
// broadcast 128-bit load (instruction streams are shared by all CTAs working
// on the same program, so they live in L1/L2), prefetched one ahead, plus an
// indirect branch that never diverges.
#pragma once

#include <stdint.h>

#include "../../include/planeq_witness.h"
#include "field.hpp"

namespace pqw {
namespace {

constexpr int NW = 8;               // warps per CTA (must equal the compile-time n_warps)
constexpr int BLOCK = 32 * NW;
constexpr int TW = 32;              // witnesses per work item (one per lane)

struct StageDesc {
  uint32_t code_off;
  uint32_t n_slots;
  uint32_t var_base;
  uint32_t result;  // index into result arrays
};

struct Params {
  const uint4* code;
  const StageDesc* stages;
  const uint32_t* work;      // stage-desc index per work stage
  const uint64_t* var_keys;
  const uint64_t* fn_keys;   // 3 entries
  uint32_t* counter;         // work-item counter
  uint32_t* scratch;         // per-CTA spill value files
  unsigned long long* first_bad;
  uint32_t* n_valid;
  uint32_t* n_bad;
  uint32_t n_items;
  uint32_t tiles;            // work items per stage
  uint32_t n_witness;
  uint32_t smem_slots;       // fast slots (shared memory)
  uint32_t overflow_slots;   // per-CTA spill capacity in slots
  // probe mode
  uint32_t probe_w;
  uint32_t probe_obl;
  uint32_t* probe_out;       // [lhs, rhs]
  uint32_t* probe_vars;
};

__device__ __forceinline__ void cta_bar() { asm volatile("bar.sync 1, %0;" ::"r"(BLOCK) : "memory"); }

// Runs this warp's stream of the stage program for witness w = tile*32 + lane,
// folding the lane's definedness and first failing obligation into valid/bad.
template <bool PROBE>
__device__ __forceinline__ void run_stream(const Params& p, const StageDesc& sd, uint32_t* sfile,
                                           uint32_t* gfile, uint32_t w, bool& valid,
                                           uint32_t& bad) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t nsm = p.smem_slots;
  auto ld = [&](uint32_t s) -> uint32_t {
    if (s < nsm) return sfile[s * 32u + lane];
    return gfile[(size_t)(s - nsm) * 32u + lane];
  };
  auto st = [&](uint32_t s, uint32_t v) {
    if (s < nsm)
      sfile[s * 32u + lane] = v;
    else
      gfile[(size_t)(s - nsm) * 32u + lane] = v;
  };
  const uint4* base = p.code + sd.code_off;
  const uint32_t off = __ldg(reinterpret_cast<const uint32_t*>(base) + warp);
  const uint4* code = base + off;
  uint64_t acc = 0;
  uint4 nxt = __ldg(code);
  for (uint32_t pc = 0;; ++pc) {
    const uint4 in = nxt;
    nxt = __ldg(code + pc + 1);  // every stream ends with END and the image is padded
    switch (in.x) {
      case PQW_B_END:
        return;
      case PQW_B_BAR:
        cta_bar();
        break;
      case PQW_B_CONST:
        st(in.y, in.z);
        break;
      case PQW_B_VAR: {
        const uint32_t v = witness_value(__ldg(p.var_keys + sd.var_base + in.z), w);
        if (PROBE && w == p.probe_w) p.probe_vars[in.z] = v;
        st(in.y, v);
        break;
      }
      case PQW_B_ADD:
        st(in.y, fadd(ld(in.z), ld(in.w)));
        break;
      case PQW_B_SUB:
        st(in.y, fsub(ld(in.z), ld(in.w)));
        break;
      case PQW_B_MUL:
        st(in.y, fmul(ld(in.z), ld(in.w)));
        break;
      case PQW_B_NEG:
        st(in.y, fneg(ld(in.z)));
        break;
      case PQW_B_DIV:
        st(in.y, fmul(ld(in.z), finv(ld(in.w))));
        break;
      case PQW_B_INV:
        st(in.y, finv(ld(in.z)));
        break;
      case PQW_B_HASH:
        st(in.y, uf_apply(__ldg(p.fn_keys + in.w), ld(in.z)));
        break;
      case PQW_B_ACC_LD:
        acc = ld(in.z);
        break;
      case PQW_B_ACC_ADD:
        acc += ld(in.z);
        break;
      case PQW_B_ACC_MUL:
        acc = (uint64_t)ld(in.z) * ld(in.w);
        break;
      case PQW_B_ACC_MACF:
        acc = ffold64(acc);
        // fallthrough
      case PQW_B_ACC_MAC:
        acc += (uint64_t)ld(in.z) * ld(in.w);
        break;
      case PQW_B_ACC_MUL2:  // acc = a*b + c*d  (< 2^63)
        acc = (uint64_t)ld(in.z) * ld(in.w) + (uint64_t)ld(in.y & 0xFFFFu) * ld(in.y >> 16);
        break;
      case PQW_B_ACC_MAC2:  // acc = fold(acc) + a*b + c*d  (< 2^34 + 2^63)
        acc = ffold64(acc) + (uint64_t)ld(in.z) * ld(in.w) +
              (uint64_t)ld(in.y & 0xFFFFu) * ld(in.y >> 16);
        break;
      case PQW_B_ACC_ST:
        st(in.y, fred64(acc));
        break;
      case PQW_B_CHK: {
        const uint32_t a = ld(in.z), b = ld(in.w);
        if (PROBE && in.y == p.probe_obl && w == p.probe_w) {
          p.probe_out[0] = a;
          p.probe_out[1] = b;
        }
        if (a != b) bad = min(bad, in.y);
        break;
      }
      case PQW_B_DEN:
        if (ld(in.z) == 0) valid = false;
        break;
      default:
        return;  // unreachable for a well-formed image
    }
  }
}

template <bool PROBE>
__global__ void __launch_bounds__(BLOCK) eval_kernel(Params p) {
  extern __shared__ uint32_t sfile[];
  __shared__ uint32_t s_item;
  __shared__ uint32_t s_invalid;     // lanes with a vanished denominator (bitmask)
  __shared__ uint32_t s_bad[32];     // first failing obligation per lane
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t warp = threadIdx.x >> 5;
  uint32_t* gfile = p.scratch + (size_t)blockIdx.x * p.overflow_slots * 32u;
  for (;;) {
    if (threadIdx.x == 0) s_item = PROBE ? 0u : atomicAdd(p.counter, 1u);
    if (threadIdx.x < 32) s_bad[threadIdx.x] = 0xFFFFFFFFu;
    if (threadIdx.x == 0) s_invalid = 0;
    __syncthreads();
    const uint32_t item = s_item;
    if (item >= p.n_items) break;
    const uint32_t stage = PROBE ? p.work[0] : p.work[item / p.tiles];
    const uint32_t tile = PROBE ? p.probe_w / 32u : item % p.tiles;
    const StageDesc sd = p.stages[stage];
    const uint32_t w = tile * 32u + lane;
    bool valid = PROBE ? (w == p.probe_w) : (w < p.n_witness);
    uint32_t bad = 0xFFFFFFFFu;
    run_stream<PROBE>(p, sd, sfile, gfile, w, valid, bad);
    // merge the warps' verdicts for each lane
    const uint32_t inval = __ballot_sync(0xFFFFFFFFu, !valid);
    if (lane == 0 && inval) atomicOr(&s_invalid, inval);
    if (bad != 0xFFFFFFFFu) atomicMin(&s_bad[lane], bad);
    __syncthreads();
    if (!PROBE && warp == 0) {
      const bool ok = !((s_invalid >> lane) & 1u) && w < p.n_witness;
      const uint32_t b = s_bad[lane];
      uint32_t nv = ok, nb = ok && b != 0xFFFFFFFFu;
      unsigned long long best = nb ? (((unsigned long long)w << 32) | b) : ~0ull;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        nv += __shfl_down_sync(0xFFFFFFFFu, nv, o);
        nb += __shfl_down_sync(0xFFFFFFFFu, nb, o);
        const unsigned long long t = __shfl_down_sync(0xFFFFFFFFu, best, o);
        best = t < best ? t : best;
      }
      if (lane == 0) {
        if (nv) atomicAdd(p.n_valid + sd.result, nv);
        if (nb) atomicAdd(p.n_bad + sd.result, nb);
        if (best != ~0ull) atomicMin(p.first_bad + sd.result, best);
      }
    }
    __syncthreads();  // the value file and s_* are reused by the next item
    if (PROBE) break;
  }
}

// -- integer-pipe ceiling: register-resident field arithmetic, no decode, no memory.
// KIND 0: fmul chains, 1: fadd chains, 2: keyed hash (mix64 + to_field).
template <int KIND>
__global__ void __launch_bounds__(256) peak_kernel(uint32_t* sink, int iters, uint32_t salt) {
  uint32_t a[8], b[8];
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    a[j] = (t * 2654435761u + j * 40503u + salt) % P;
    b[j] = (t * 2246822519u + j * 9973u + 7u) % P;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (KIND == 0) a[j] = fmul(a[j], b[j]);
        else if (KIND == 1) a[j] = fadd(a[j], b[j]);
        else a[j] = uf_apply(0x9E3779B97F4A7C15ull + b[j], a[j]);
      }
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) x ^= a[j];
  if (x == salt * 2654435761u + 1u) sink[t] = x;  // opaque to the compiler: keeps chains live
}

}  // namespace
}  // namespace pqw

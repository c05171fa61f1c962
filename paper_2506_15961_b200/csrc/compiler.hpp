// compiler.hpp -- host-side stage compiler: tensor-op program -> scalar F_p bytecode.
#pragma once
#include <stdint.h>

#include <memory>
#include <string>
#include <vector>

#include "../../include/planeq_witness.h"

namespace pqw {

struct CompiledStage {
  int status = PQW_STAGE_OK;
  int64_t info = -1;
  uint32_t n_obligations = 0;
  uint32_t n_fast = 0;
  uint32_t n_residual = 0;
  uint32_t n_slots = 0;        // fast slots [0, smem_slots) + spill slots after them
  uint32_t n_fast_slots = 0;   // fast slots actually used
  uint32_t n_warps = 1;        // cooperative streams (one per warp of the CTA)
  uint32_t n_phases = 0;       // barrier-separated phases of the schedule
  uint32_t n_vars = 0;
  uint32_t var_base = 0;       // first global var index of this stage
  uint64_t degree = 0;
  uint64_t field_ops = 0;      // field operations per witness (roofline numerator)
  int64_t const_lhs = 0, const_rhs = 0, exact_lhs = INT64_MIN, exact_rhs = INT64_MIN;
  // terminated by PQW_B_END when status == OK; shared between stages whose
  // programs are identical (VAR operands are stage-relative)
  std::shared_ptr<std::vector<pqw_ins>> code = std::make_shared<std::vector<pqw_ins>>();
};

// Compile one stage into a cooperative program: `n_warps` instruction streams
// (one per warp of a CTA that evaluates 32 witnesses, one per lane) separated
// into barrier phases, sharing one value file. Code layout: ceil(n_warps/4)
// records holding the n_warps u32 stream offsets, then the streams; each has
// one PQW_B_BAR per phase boundary and ends with PQW_B_END. Slots below
// `smem_slots` are the fast (shared-memory) file; the allocator gives them to
// the busiest values per phase of lifetime and spills the rest to slots >=
// smem_slots. VAR operands are stage-relative. Throws std::runtime_error on
// malformed input.
CompiledStage compile_stage(const int32_t* ir, size_t ir_len, const int64_t* consts,
                            size_t n_consts, uint32_t n_vars, uint32_t var_base,
                            const uint64_t fn_keys[3], uint32_t smem_slots, uint32_t n_warps);

// Defaults (overridable per engine: PQW_FAST_SLOTS, PQW_WARPS env vars): a
// 1600-slot fast file is 200 KB of shared memory for 32 witnesses.
constexpr uint32_t DEFAULT_FAST_SLOTS = 1600;
constexpr uint32_t DEFAULT_WARPS = 8;

// Variables (global indices) in the cone of obligation `obl`, by backward
// slicing the bytecode.
std::vector<uint32_t> obligation_support(const CompiledStage& st, uint32_t obl);

}  // namespace pqw

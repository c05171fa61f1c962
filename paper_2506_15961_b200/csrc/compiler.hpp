// compiler.hpp -- host-side stage compiler: tensor-op program -> v4 F_p program.
#pragma once
#include <stdint.h>

#include <memory>
#include <string>
#include <vector>

#include "../../include/planeq_witness.h"
#include "isa.hpp"
#include "schedule.hpp"

namespace pqw {

struct CompiledStage {
  int status = PQW_STAGE_OK;
  int64_t info = -1;
  uint32_t n_obligations = 0;
  uint32_t n_fast = 0;
  uint32_t n_residual = 0;
  uint32_t n_slots = 0;        // shared-memory slots of the value file
  uint32_t n_spill = 0;        // global spill slots
  uint32_t n_spilled_values = 0;
  uint32_t n_bundles = 0;
  uint32_t n_waits = 0;
  uint64_t makespan = 0;       // cost-model length of the schedule
  uint32_t n_warps = 1;        // instruction streams (one per warp of the CTA)
  uint32_t n_vars = 0;
  uint32_t var_base = 0;       // first global var index of this stage
  uint64_t degree = 0;
  uint64_t field_ops = 0;      // field operations per witness (sum of cls)
  uint64_t cls[5] = {0, 0, 0, 0, 0};  // per witness: mul, add, hash, inv, cmp
  uint64_t op_hist[I_NUM_OPS] = {};
  int64_t const_lhs = 0, const_rhs = 0, exact_lhs = INT64_MIN, exact_rhs = INT64_MIN;
  // isa.hpp program (table + NW streams) when status == OK; shared between
  // stages whose programs are identical (VAR operands are stage-relative)
  std::shared_ptr<std::vector<pqw_ins>> code = std::make_shared<std::vector<pqw_ins>>();
  std::shared_ptr<const Dag> dag;  // scheduling units, for obligation support
};

// Compile one stage into an isa.hpp program of `n_warps` instruction streams
// sharing a value file of at most `smem_slots` shared-memory slots (values
// that do not fit are kept in global memory). VAR operands are
// stage-relative. Throws std::runtime_error on malformed input.
CompiledStage compile_stage(const int32_t* ir, size_t ir_len, const int64_t* consts,
                            size_t n_consts, uint32_t n_vars, uint32_t var_base,
                            const uint64_t fn_keys[3], uint32_t smem_slots, uint32_t n_warps,
                            const SchedOptions& sched);

// Defaults (overridable per engine: PQW_FAST_SLOTS, PQW_WARPS, PQW_WINDOW,
// PQW_BMAX, PQW_XLAT env vars): 1680 slots = 210 KB of shared memory, which
// leaves room for the per-warp code rings (16 x 1 KB).
constexpr uint32_t DEFAULT_FAST_SLOTS = 1680;
constexpr uint32_t DEFAULT_WARPS = 16;

// Variables (stage-relative indices) in the cone of obligation `obl`.
std::vector<uint32_t> obligation_support(const CompiledStage& st, uint32_t obl);

}  // namespace pqw

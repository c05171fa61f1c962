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
  uint32_t n_vars = 0;
  uint32_t var_base = 0;       // first global var index of this stage
  uint64_t degree = 0;
  uint64_t field_ops = 0;      // field operations per witness (roofline numerator)
  int64_t const_lhs = 0, const_rhs = 0, exact_lhs = INT64_MIN, exact_rhs = INT64_MIN;
  // terminated by PQW_B_END when status == OK; shared between stages whose
  // programs are identical (VAR operands are stage-relative)
  std::shared_ptr<std::vector<pqw_ins>> code = std::make_shared<std::vector<pqw_ins>>();
};

// Compile one stage. `var_base` is the global index of the stage's first
// variable (VAR instructions carry global indices). Slots below `smem_slots`
// are the fast (shared-memory) file; the allocator gives them to the busiest
// short-lived values and spills the rest to slots >= smem_slots. Throws
// std::runtime_error on malformed input.
CompiledStage compile_stage(const int32_t* ir, size_t ir_len, const int64_t* consts,
                            size_t n_consts, uint32_t n_vars, uint32_t var_base,
                            const uint64_t fn_keys[3], uint32_t smem_slots);

// Default fast-slot count (overridable per engine, PQW_FAST_SLOTS env var).
constexpr uint32_t DEFAULT_FAST_SLOTS = 24;

// Variables (global indices) in the cone of obligation `obl`, by backward
// slicing the bytecode.
std::vector<uint32_t> obligation_support(const CompiledStage& st, uint32_t obl);

}  // namespace pqw

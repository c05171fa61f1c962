// schedule.hpp -- host back end of the stage compiler: value DAG -> v4 program.
#pragma once
#include <stdint.h>

#include <vector>

#include "../../include/planeq_witness.h"
#include "isa.hpp"

namespace pqw {

// One scheduling unit: a value definition, an obligation check or a
// definedness test. Operands name the units that define them.
struct DagUnit {
  uint32_t op = I_END;  // I_DOT, I_SUM, I_SUB, I_NEG, I_HASH, I_INV, I_VAR, I_CONST, I_CHK, I_DEN
  uint32_t fn = 0;      // HASH: function index
  uint32_t k = 0;       // DOT: pairs, SUM: terms
  uint32_t aux = 0;     // VAR: stage-relative index, CONST: residue, CHK: obligation id
  uint32_t arg0 = 0;    // operands: pool[arg0 .. arg0 + nargs)
  uint32_t nargs = 0;
  bool guarded = false;  // INV: the operand is a checked denominator (batchable)
  bool defines() const { return op != I_CHK && op != I_DEN; }
};

// Units in priority order (a topological order: operands come first).
struct Dag {
  std::vector<DagUnit> units;
  std::vector<uint32_t> pool;
};

struct SchedOptions {
  uint32_t n_warps = 16;
  uint32_t smem_slots = 1760;  // shared-memory value file capacity (slots)
  uint32_t window = 0;         // look-ahead in units past the lowest unscheduled one (0: adaptive)
  uint32_t bmax = 32;          // max ops per bundle
  uint32_t xlat = 32;          // cost-model penalty of a cross-warp dependence
  uint32_t bundle_base = 600;  // cost-model constant per bundle (dispatch + latency; measured best on 405B)
  uint32_t spill_cost = 8;     // cost-model weight of one FILL/SPILL op when choosing a window
  uint32_t pick_scan = 0;      // >0: pick the longest-path unit among that many eligible ones
  uint32_t active_warps = 32;  // warps that receive work (the rest run empty streams)
};

struct Program {
  std::vector<pqw_ins> code;   // table + streams (isa.hpp)
  uint32_t n_slots = 0;        // shared slots used
  uint32_t n_spill = 0;        // global spill slots used
  uint32_t n_spilled_values = 0;
  uint32_t n_remat = 0;        // VAR/CONST ops recomputed at readers instead of filled
  uint32_t n_bundles = 0;
  uint32_t n_waits = 0;        // (warp, count) pairs waited on
  uint64_t makespan = 0;       // cost-model length of the schedule
  uint64_t cls[5] = {0, 0, 0, 0, 0};  // field ops per witness: mul, add, hash, inv, cmp
  uint64_t op_hist[I_NUM_OPS] = {};   // ops per kind (bundled ops, not records)
};

// Throws std::runtime_error on malformed DAGs.
Program schedule_program(const Dag& dag, const SchedOptions& opt);

}  // namespace pqw

// compiler.hpp -- host-side stage compiler: tensor-op program -> v4 F_p program.
#pragma once
#include "pool.hpp"
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/planeq_witness.h"
#include "isa.hpp"
#include "schedule.hpp"

namespace pqw {

// Back-end output (isa.hpp program + its statistics), shared by every stage
// whose program text is identical; filled by finalize_stage.
struct StageBackend {
  Program prog;
  bool ready = false;
};

struct CompiledStage {
  int status = PQW_STAGE_OK;
  int64_t info = -1;
  uint32_t n_obligations = 0;
  uint32_t n_fast = 0;
  uint32_t n_residual = 0;
  uint32_t n_warps = 1;        // instruction streams (one per warp of the CTA)
  uint32_t n_vars = 0;
  uint32_t var_base = 0;       // first global var index of this stage
  uint64_t degree = 0;
  int64_t const_lhs = 0, const_rhs = 0, exact_lhs = INT64_MIN, exact_rhs = INT64_MIN;
  std::shared_ptr<const Dag> dag;         // scheduling units (status == OK)
  SchedOptions sched;                     // back-end options it was compiled with
  std::shared_ptr<StageBackend> be = std::make_shared<StageBackend>();
  const Program& prog() const { return be->prog; }
};

// Compile one stage: the front end (symbolic execution into a value DAG,
// value numbering, obligation classification) runs now; the back end that
// turns the DAG into an isa.hpp program of `n_warps` instruction streams
// sharing a value file of at most `smem_slots` shared-memory slots runs in
// finalize_stage (the engine batches those over host threads). VAR operands
// are stage-relative. Throws std::runtime_error on malformed input.
CompiledStage compile_stage(const int32_t* ir, size_t ir_len, const int64_t* consts,
                            size_t n_consts, uint32_t n_vars, uint32_t var_base,
                            const uint64_t fn_keys[3], uint32_t smem_slots, uint32_t n_warps,
                            const SchedOptions& sched);

// Defaults (overridable per engine: PQW_FAST_SLOTS, PQW_WARPS, PQW_WINDOW,
// PQW_BMAX, PQW_XLAT env vars): 1680 slots = 210 KB of shared memory, which
// leaves room for the per-warp code rings (16 x 1 KB).
constexpr uint32_t DEFAULT_FAST_SLOTS = 1800;
constexpr uint32_t DEFAULT_WARPS = 16;

// Host confirmation of a refutation (pqw_confirm in include/planeq_witness.h):
// re-runs the front end; returns -1 when the program has no value graph.
int confirm_stage(const int32_t* ir, size_t ir_len, const int64_t* consts, size_t n_consts,
                  uint32_t n_vars, const uint64_t fn_keys[3], const uint64_t* var_keys,
                  uint32_t witness, const double* env_vals, size_t n_env, double tol,
                  int64_t out[4], double sides[2]);

// Run the back end of a stage compiled with status OK (idempotent).
void finalize_stage(CompiledStage& st);

// Back-end sharing between stages whose value DAGs are equal.
uint64_t dag_hash(const Dag& d);
bool same_dag(const Dag& a, const Dag& b);
bool same_sched(const SchedOptions& a, const SchedOptions& b);

// f(i) for i in [0, n) on up to hardware_concurrency host threads
template <class F>
void host_parallel_for(size_t n, F&& f) {
  const unsigned nt =
      (unsigned)std::min<size_t>(n, std::max(1u, std::thread::hardware_concurrency()));
  std::atomic<size_t> next{0};
  run_on_threads(nt, [&](unsigned) {
    for (size_t i; (i = next.fetch_add(1)) < n;) f(i);
  });
}

// Variables (stage-relative indices) in the cone of obligation `obl`.
std::vector<uint32_t> obligation_support(const CompiledStage& st, uint32_t obl);

}  // namespace pqw

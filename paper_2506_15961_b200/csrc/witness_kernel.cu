// witness_kernel.cu -- host side of the sm_100a stage-discharge engine: the
// extern "C" API of include/planeq_witness.h (compile, upload, launch, results,
// probe). The device interpreter lives in interp.cuh.
#include <cuda_runtime.h>
#include <malloc.h>
#include <sched.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <atomic>
#include <mutex>
#include <thread>
#include <numeric>
#include <string>
#include <unordered_map>
#include <vector>

#include "compiler.hpp"
#include "field.hpp"

#include "interp.cuh"

namespace pqw {
namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CU(call)                                                              \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess)                                                    \
      return fail(PQW_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

}  // namespace

int set_last_error(int code, const std::string& msg) { return fail(code, msg); }

// Device memory of uploaded images comes from a per-device pool of blocks
// that outlive engines: verify_plan creates an engine per call, and a fresh
// cudaMalloc/cudaFree of ~30 MB per call measured 30-150 ms of variance.
// A returned block is reused by the next upload that fits in it; at most two
// blocks per device stay cached.
std::mutex g_pool_mu;
std::unordered_map<int, std::vector<std::pair<void*, size_t>>> g_pool;

void* arena_get(int device, size_t need, size_t* got) {
  {
    std::lock_guard<std::mutex> l(g_pool_mu);
    auto& v = g_pool[device];
    size_t best = SIZE_MAX;
    for (size_t i = 0; i < v.size(); ++i)
      if (v[i].second >= need && (best == SIZE_MAX || v[i].second < v[best].second)) best = i;
    if (best != SIZE_MAX) {
      auto blk = v[best];
      v.erase(v.begin() + (long)best);
      *got = blk.second;
      return blk.first;
    }
  }
  void* p = nullptr;
  const size_t bytes = need + need / 4;  // headroom for the next, slightly larger image
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    // drop the cached blocks and retry at the exact size
    std::vector<std::pair<void*, size_t>> drop;
    {
      std::lock_guard<std::mutex> l(g_pool_mu);
      drop.swap(g_pool[device]);
    }
    for (auto& b : drop) cudaFree(b.first);
    if (cudaMalloc(&p, need) != cudaSuccess) return nullptr;
    *got = need;
    return p;
  }
  *got = bytes;
  return p;
}

void arena_put(int device, void* p, size_t bytes) {
  cudaSetDevice(device);
  cudaDeviceSynchronize();  // no launch of the owning engine may still use it
  std::lock_guard<std::mutex> l(g_pool_mu);
  auto& v = g_pool[device];
  v.push_back({p, bytes});
  if (v.size() > 2) {  // keep the two largest
    std::sort(v.begin(), v.end(), [](auto& a, auto& b) { return a.second > b.second; });
    for (size_t i = 2; i < v.size(); ++i) cudaFree(v[i].first);
    v.resize(2);
  }
}
}  // namespace pqw

struct pqw_engine {
  int device = 0;
  uint64_t seed = 0;
  uint64_t fn_keys[3] = {0, 0, 0};
  std::vector<pqw::CompiledStage> stages;
  // deferred front ends: per stage, the stage it duplicates (-1: compile its
  // own text, kept in cache_src) and its var base; front_done once compiled
  std::vector<int> alias;
  std::vector<uint8_t> active;   // pqw_stage_select: only active stages are scheduled/uploaded
  std::vector<uint32_t> pend_nvars, pend_base;
  std::vector<char> front_done;
  size_t n_front_pending = 0;
  std::vector<uint64_t> var_keys;
  // program cache: text hash -> first stage compiled from it (+ its source for exact compare)
  std::unordered_map<uint64_t, size_t> cache;
  std::unordered_map<size_t, std::pair<std::vector<int32_t>, std::vector<int64_t>>> cache_src;
  uint64_t cache_hits = 0;
  uint64_t n_code_unique = 0;
  // device image
  bool uploaded = false;
  std::vector<int> gpu_stage_of;   // result index -> stage index
  uint4* d_code = nullptr;
  pqw::StageDesc* d_stages = nullptr;
  uint32_t* d_work = nullptr;
  uint64_t* d_var_keys = nullptr;
  uint64_t* d_fn_keys = nullptr;
  uint32_t* d_counter = nullptr;
  uint32_t* d_scratch = nullptr;
  unsigned long long* d_first_bad = nullptr;
  uint32_t* d_n_valid = nullptr;
  uint32_t* d_n_bad = nullptr;
  uint32_t* d_probe = nullptr;
  size_t scratch_bytes = 0;
  uint64_t h2d_bytes = 0;  // bytes the last pqw_upload copied host -> device
  uint32_t n_gpu_stages = 0;
  uint32_t max_slots = 0;
  uint32_t smem_slots = 0;
  uint32_t n_warps = pqw::DEFAULT_WARPS;
  uint32_t sleep_ns = 32;
  uint32_t fast_slots = pqw::DEFAULT_FAST_SLOTS;  // shared value-file capacity (slots)
  uint32_t spill_slots = 0;                        // per-CTA global spill capacity
  pqw::SchedOptions sched;
  uint32_t grid = 0;
  uint64_t n_code = 0;
  uint64_t op_hist[PQW_B_NUM_OPS] = {};
  uint64_t cls[5] = {};
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool timed = false;
  std::vector<unsigned long long> h_first_bad;
  std::vector<uint32_t> h_valid, h_bad;
  bool results_ready = false;
  unsigned long long* d_prof_last = nullptr;

  void* arena = nullptr;     // one device block holding every buffer of the image
  size_t arena_bytes = 0;

  void free_device() {
    if (arena) pqw::arena_put(device, arena, arena_bytes);
    arena = nullptr;
    arena_bytes = 0;
    d_code = nullptr;
    d_stages = nullptr;
    d_work = nullptr;
    d_var_keys = nullptr;
    d_fn_keys = nullptr;
    d_counter = nullptr;
    d_scratch = nullptr;
    d_first_bad = nullptr;
    d_n_valid = nullptr;
    d_n_bad = nullptr;
    d_probe = nullptr;
    uploaded = false;
    results_ready = false;
  }
};

using pqw::fail;

// Run the compiler back end of every pending program, spread over host threads
// (identical programs share one back end). PQW_THREADS caps the thread count.
extern "C" {
static int finalize_front(pqw_engine* e);
}

static int finalize_all(pqw_engine* e) {
  {
    int rc = finalize_front(e);
    if (rc != PQW_OK) return rc;
  }
  std::vector<pqw::CompiledStage*> todo;
  std::unordered_map<const pqw::StageBackend*, int> seen;
  for (size_t i = 0; i < e->stages.size(); ++i) {
    auto& st = e->stages[i];
    if (e->active[i] && st.status == PQW_STAGE_OK && !st.be->ready &&
        seen.emplace(st.be.get(), 1).second)
      todo.push_back(&st);
  }
  if (todo.empty()) return PQW_OK;
  // Programs whose texts differ but whose value DAGs are equal (the front end
  // erases the difference: interface order, names) get one back end:
  // schedule_program is a function of the DAG and the options only.
  {
    std::vector<uint64_t> h(todo.size());
    pqw::host_parallel_for(todo.size(), [&](size_t i) { h[i] = pqw::dag_hash(*todo[i]->dag); });
    std::unordered_map<uint64_t, std::vector<size_t>> reps;
    std::unordered_map<const pqw::StageBackend*, std::shared_ptr<pqw::StageBackend>> same;
    std::vector<pqw::CompiledStage*> kept;
    for (size_t i = 0; i < todo.size(); ++i) {
      auto& cand = reps[h[i]];
      bool dup = false;
      for (size_t r : cand) {
        if (pqw::same_dag(*todo[r]->dag, *todo[i]->dag) &&
            pqw::same_sched(todo[r]->sched, todo[i]->sched)) {
          same.emplace(todo[i]->be.get(), todo[r]->be);
          dup = true;
          break;
        }
      }
      if (!dup) {
        cand.push_back(i);
        kept.push_back(todo[i]);
      }
    }
    if (!same.empty())
      for (size_t i = 0; i < e->stages.size(); ++i) {
        auto it = same.find(e->stages[i].be.get());
        if (it != same.end()) e->stages[i].be = it->second;
      }
    todo.swap(kept);
  }
  static const bool timing = getenv("PQW_TIMING") != nullptr;
  // largest first, handed out through a shared counter
  std::sort(todo.begin(), todo.end(), [](const pqw::CompiledStage* a, const pqw::CompiledStage* b) {
    return a->dag->units.size() > b->dag->units.size();
  });
  // the CPUs this process may run on (hardware_concurrency reports the host's)
  unsigned nt = std::max(1u, std::thread::hardware_concurrency());
  {
    cpu_set_t cs;
    if (sched_getaffinity(0, sizeof(cs), &cs) == 0) nt = std::max(1, CPU_COUNT(&cs));
  }
  if (const char* s = getenv("PQW_THREADS")) nt = std::max(1, atoi(s));
  nt = std::min<unsigned>(nt, (unsigned)todo.size());
  std::atomic<size_t> next{0};
  std::mutex err_mu;
  std::string err;
  auto work = [&]() {
    for (;;) {
      const size_t i = next.fetch_add(1);
      if (i >= todo.size()) return;
      try {
        const auto t0 = std::chrono::steady_clock::now();
        pqw::finalize_stage(*todo[i]);
        if (timing)
          fprintf(stderr, "PQW_TIMING back end %zu units %.1f ms\n", todo[i]->dag->units.size(),
                  std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                      .count());
      } catch (const std::exception& ex) {
        std::lock_guard<std::mutex> g(err_mu);
        if (err.empty()) err = ex.what();
      }
    }
  };
  pqw::run_on_threads(nt, [&](unsigned) { work(); });
  if (!err.empty()) return fail(PQW_EINVAL, std::string("stage compile: ") + err);
  return PQW_OK;
}

extern "C" {

int pqw_abi_version(void) { return PQW_ABI_VERSION; }

const char* pqw_last_error(void) { return pqw::g_err.c_str(); }

int pqw_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int pqw_engine_create(int device, uint64_t seed, const uint64_t fn_keys[3], pqw_engine** out) {
  if (!out || !fn_keys) return fail(PQW_EINVAL, "null argument");
  {
    // the compiler allocates and frees large scratch vectors per program on
    // many threads: keep them in the heap instead of mmap/munmap round trips
    static std::once_flag once;
    std::call_once(once, [] {
      mallopt(M_MMAP_THRESHOLD, 512 << 20);
      mallopt(M_TRIM_THRESHOLD, 1 << 30);
    });
  }
  auto* e = new pqw_engine();
  e->device = device;
  e->seed = seed;
  for (int i = 0; i < 3; ++i) e->fn_keys[i] = fn_keys[i];
  auto env = [](const char* name, int lo, int hi, uint32_t& out) {
    if (const char* s = getenv(name)) {
      int v = atoi(s);
      if (v >= lo && v <= hi) out = (uint32_t)v;
    }
  };
  env("PQW_WARPS", 8, 32, e->n_warps);
  if (e->n_warps != 8 && e->n_warps != 16 && e->n_warps != 32) e->n_warps = pqw::DEFAULT_WARPS;
  // the shared value file gets what the per-warp code rings leave of 227 KB
  e->fast_slots = std::min<uint32_t>(
      pqw::DEFAULT_FAST_SLOTS, (232448u - 512u - e->n_warps * pqw::RING_BYTES) / pqw::SLOT_BYTES);
  env("PQW_FAST_SLOTS", 16, 1800, e->fast_slots);
  env("PQW_WINDOW", 1, 1 << 20, e->sched.window);
  env("PQW_BMAX", 1, 4096, e->sched.bmax);
  env("PQW_XLAT", 0, 1 << 20, e->sched.xlat);
  env("PQW_BUNDLE_BASE", 0, 1 << 20, e->sched.bundle_base);
  env("PQW_SPILL_COST", 0, 1 << 20, e->sched.spill_cost);
  env("PQW_SLEEP", 0, 100000, e->sleep_ns);
  env("PQW_PICK", 0, 1 << 20, e->sched.pick_scan);
  *out = e;
  return PQW_OK;
}

void pqw_engine_destroy(pqw_engine* e) {
  if (!e) return;
  if (e->uploaded || e->d_code) {
    cudaSetDevice(e->device);
    e->free_device();
  }
  if (e->ev0) cudaEventDestroy(e->ev0);
  if (e->ev1) cudaEventDestroy(e->ev1);
  delete e;
}

}  // extern "C"

namespace pqw {
// Key of the program cache: a cheap multiply-xorshift over the text's 64-bit
// words (it runs over every stage's text), the full mix only finalises.
uint64_t program_hash(const int32_t* ir, size_t ir_len, const int64_t* consts, size_t n_consts,
                      size_t n_vars) {
  auto absorb = [](uint64_t h, uint64_t w) {
    h = (h ^ w) * 0x9E3779B97F4A7C15ull;
    return h ^ (h >> 29);
  };
  uint64_t h = 0x5157ull ^ ir_len ^ ((uint64_t)n_consts << 32) ^ ((uint64_t)n_vars << 48);
  size_t i = 0;
  for (; i + 2 <= ir_len; i += 2) {
    uint64_t w;
    std::memcpy(&w, ir + i, 8);
    h = absorb(h, w);
  }
  if (i < ir_len) h = absorb(h, (uint32_t)ir[i]);
  for (size_t j = 0; j < 3 * n_consts; ++j) h = absorb(h, (uint64_t)consts[j]);
  return mix64(h);
}

// The program text the engine caches under hash h and the stage compiled
// from it; false if none.
bool cached_program(const pqw_engine* e, uint64_t h, const std::vector<int32_t>** ir,
                    const std::vector<int64_t>** consts, int* stage) {
  auto it = e->cache.find(h);
  if (it == e->cache.end()) return false;
  const auto& src = e->cache_src.at(it->second);
  *ir = &src.first;
  *consts = &src.second;
  *stage = (int)it->second;
  return true;
}

// pqw_stage_add with the hash already computed. same >= 0: the caller has
// checked that this program's text equals stage `same`'s (no lookup or
// compare here). own_ir/own_consts: the text may be moved from them when the
// engine keeps it.
int stage_add_hashed(pqw_engine* e, const int32_t* ir, size_t ir_len, const int64_t* consts,
                     size_t n_consts, const uint64_t* var_keys, size_t n_vars, uint64_t h,
                     int same, std::vector<int32_t>* own_ir, std::vector<int64_t>* own_consts,
                     int64_t out_status[16]) {
  const uint32_t base = (uint32_t)e->var_keys.size();
  const int idx = (int)e->stages.size();
  int alias = -1;
  if (same >= 0) {
    alias = e->alias[(size_t)same] >= 0 ? e->alias[(size_t)same] : same;
    e->cache_hits++;
  } else {
    auto it = e->cache.find(h);
    if (it != e->cache.end()) {
      const auto& ent = e->cache_src[it->second];
      if (ent.first.size() == ir_len && std::equal(ent.first.begin(), ent.first.end(), ir) &&
          ent.second.size() == 3 * n_consts &&
          std::equal(ent.second.begin(), ent.second.end(), consts)) {
        alias = (int)it->second;
        e->cache_hits++;
      }
    }
    if (alias < 0) {
      if (it == e->cache.end()) e->cache.emplace(h, (size_t)idx);
      auto& dst = e->cache_src[(size_t)idx];
      if (own_ir) dst.first = std::move(*own_ir);
      else dst.first.assign(ir, ir + ir_len);
      if (own_consts) dst.second = std::move(*own_consts);
      else dst.second.assign(consts, consts + 3 * n_consts);
    }
  }
  e->stages.emplace_back();
  e->alias.push_back(alias);
  e->active.push_back(1);
  e->pend_nvars.push_back((uint32_t)n_vars);
  e->pend_base.push_back(base);
  e->front_done.push_back(0);
  e->n_front_pending++;
  e->var_keys.insert(e->var_keys.end(), var_keys, var_keys + n_vars);
  for (int i = 0; i < 16; ++i) out_status[i] = 0;
  out_status[0] = PQW_STAGE_PENDING;
  out_status[13] = (int64_t)n_vars;
  e->uploaded = false;
  return idx;
}
}  // namespace pqw

extern "C" {

int pqw_stage_add(pqw_engine* e, const int32_t* ir, size_t ir_len, const int64_t* consts,
                  size_t n_consts, const uint64_t* var_keys, size_t n_vars,
                  int64_t out_status[16]) {
  if (!e || !ir || !out_status) return fail(PQW_EINVAL, "null argument");
  if (n_vars && !var_keys) return fail(PQW_EINVAL, "null var_keys");
  if (n_consts && !consts) return fail(PQW_EINVAL, "null consts");
  if (ir_len < 4 || ir[0] != 0x50515701) return fail(PQW_EINVAL, "stage compile: bad program magic");
  // identical programs (e.g. the same layer repeated) compile once: the cache
  // key is the program text; a hit shares the compiled program and only
  // rebases vars. The compilation itself is deferred: every distinct program
  // is compiled on a host thread pool at the first pqw_stage_status,
  // pqw_upload or inspection call.
  const uint64_t h = pqw::program_hash(ir, ir_len, consts, n_consts, n_vars);
  return pqw::stage_add_hashed(e, ir, ir_len, consts, n_consts, var_keys, n_vars, h, -1, nullptr,
                               nullptr, out_status);
}

// Compile the front ends of every pending stage (distinct programs on host
// threads, duplicates copy their original and rebase their vars).
static int finalize_front(pqw_engine* e) {
  if (!e->n_front_pending) return PQW_OK;
  std::vector<size_t> todo;
  for (size_t i = 0; i < e->stages.size(); ++i)
    if (!e->front_done[i] && e->alias[i] < 0) todo.push_back(i);
  // longest texts first (the pool's critical path is its largest program)
  std::stable_sort(todo.begin(), todo.end(), [&](size_t a, size_t b) {
    return e->cache_src.at(a).first.size() > e->cache_src.at(b).first.size();
  });
  static const bool timing = getenv("PQW_TIMING") != nullptr;
  const auto t_front = std::chrono::steady_clock::now();
  unsigned nt = std::max(1u, std::thread::hardware_concurrency());
  {
    cpu_set_t cs;
    if (sched_getaffinity(0, sizeof(cs), &cs) == 0) nt = std::max(1, CPU_COUNT(&cs));
  }
  if (const char* s = getenv("PQW_THREADS")) nt = std::max(1, atoi(s));
  nt = std::max(1u, std::min<unsigned>(nt, (unsigned)todo.size()));
  std::atomic<size_t> next{0};
  std::mutex err_mu;
  std::string err;
  auto work = [&]() {
    for (;;) {
      const size_t k = next.fetch_add(1);
      if (k >= todo.size()) return;
      const size_t i = todo[k];
      const auto& src = e->cache_src.at(i);
      try {
        e->stages[i] = pqw::compile_stage(src.first.data(), src.first.size(), src.second.data(),
                                          src.second.size() / 3, e->pend_nvars[i], e->pend_base[i],
                                          e->fn_keys, e->fast_slots, e->n_warps, e->sched);
        e->front_done[i] = 1;
      } catch (const std::exception& ex) {
        std::lock_guard<std::mutex> g(err_mu);
        if (err.empty()) err = "stage " + std::to_string(i) + " compile: " + ex.what();
      }
    }
  };
  pqw::run_on_threads(nt, [&](unsigned) { work(); });
  if (timing)
    fprintf(stderr, "PQW_TIMING front ends %zu programs %.1f ms (largest %zu words)\n", todo.size(),
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_front)
                .count(),
            todo.empty() ? (size_t)0 : e->cache_src.at(todo[0]).first.size());
  if (!err.empty()) return fail(PQW_EINVAL, err);
  for (size_t i = 0; i < e->stages.size(); ++i) {
    if (e->front_done[i]) continue;
    e->stages[i] = e->stages[(size_t)e->alias[i]];
    e->stages[i].var_base = e->pend_base[i];
    e->front_done[i] = 1;
  }
  e->n_front_pending = 0;
  return PQW_OK;
}

int pqw_stage_select(pqw_engine* e, const uint8_t* active, size_t n) {
  if (!e || !active) return fail(PQW_EINVAL, "null argument");
  if (n != e->stages.size()) return fail(PQW_EINVAL, "select: one flag per stage");
  e->active.assign(active, active + n);
  e->uploaded = false;
  return PQW_OK;
}

int64_t pqw_stage_cost(pqw_engine* e, int stage) {
  if (!e) return fail(PQW_EINVAL, "null engine");
  if (stage < 0 || (size_t)stage >= e->stages.size()) return fail(PQW_EINVAL, "bad stage");
  {
    int rc = finalize_front(e);
    if (rc != PQW_OK) return rc;
  }
  const auto& st = e->stages[stage];
  if (st.status != PQW_STAGE_OK || !st.dag) return 0;
  return (int64_t)st.dag->units.size();
}

int pqw_stage_status(pqw_engine* e, int stage, int64_t out_status[16]) {
  if (!e || !out_status) return fail(PQW_EINVAL, "null argument");
  if (stage < 0 || (size_t)stage >= e->stages.size()) return fail(PQW_EINVAL, "bad stage");
  {
    int rc = finalize_front(e);
    if (rc != PQW_OK) return rc;
  }
  const auto& st = e->stages[stage];
  for (int i = 0; i < 16; ++i) out_status[i] = 0;
  out_status[0] = st.status;
  out_status[1] = st.info;
  out_status[2] = st.n_obligations;
  out_status[3] = st.n_fast;
  out_status[4] = st.n_residual;
  out_status[7] = (int64_t)std::min<uint64_t>(st.degree, (uint64_t)INT64_MAX);
  out_status[8] = st.const_lhs;
  out_status[9] = st.const_rhs;
  out_status[10] = st.exact_lhs;
  out_status[11] = st.exact_rhs;
  out_status[13] = st.n_vars;
  if (st.status == PQW_STAGE_OK && st.be->ready) {
    const auto& pr = st.prog();
    out_status[5] = (int64_t)pr.code.size();
    out_status[6] = pr.n_slots;
    out_status[12] = (int64_t)(pr.cls[0] + pr.cls[1] + pr.cls[2] + pr.cls[3] + pr.cls[4]);
    out_status[14] = pr.n_spill;
    out_status[15] = pr.n_bundles;
  }
  return PQW_OK;
}

int pqw_reset(pqw_engine* e) {
  if (!e) return fail(PQW_EINVAL, "null engine");
  if (e->d_code) {
    cudaSetDevice(e->device);
    e->free_device();
  }
  e->stages.clear();
  e->alias.clear();
  e->active.clear();
  e->pend_nvars.clear();
  e->pend_base.clear();
  e->front_done.clear();
  e->n_front_pending = 0;
  e->var_keys.clear();
  e->cache.clear();
  e->cache_src.clear();
  e->cache_hits = 0;
  e->gpu_stage_of.clear();
  e->n_gpu_stages = 0;
  return PQW_OK;
}

long pqw_stage_bytecode(pqw_engine* e, int stage, pqw_ins* out, size_t cap, uint32_t* n_slots) {
  if (!e || stage < 0 || (size_t)stage >= e->stages.size()) return fail(PQW_EINVAL, "bad stage");
  {
    int rc = finalize_front(e);
    if (rc != PQW_OK) return rc;
  }
  const auto& st = e->stages[stage];
  try {
    pqw::finalize_stage(e->stages[stage]);
  } catch (const std::exception& ex) {
    return fail(PQW_EINVAL, std::string("stage compile: ") + ex.what());
  }
  const auto& code = st.prog().code;
  if (n_slots) *n_slots = st.prog().n_slots;
  if (out) std::memcpy(out, code.data(), std::min(cap, code.size()) * sizeof(pqw_ins));
  return (long)code.size();
}

long pqw_obligation_support(pqw_engine* e, int stage, uint32_t obl, uint32_t* out, size_t cap) {
  if (!e || stage < 0 || (size_t)stage >= e->stages.size()) return fail(PQW_EINVAL, "bad stage");
  {
    int rc = finalize_front(e);
    if (rc != PQW_OK) return rc;
  }
  const auto& st = e->stages[stage];
  auto vars = pqw::obligation_support(st, obl);
  if (out)
    for (size_t i = 0; i < std::min(cap, vars.size()); ++i) out[i] = vars[i];
  return (long)vars.size();
}

int pqw_upload(pqw_engine* e) {
  if (!e) return fail(PQW_EINVAL, "null engine");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= e->device) {
    cudaGetLastError();
    return fail(PQW_ENODEV, "no CUDA device for the witness engine");
  }
  {
    int rc = finalize_all(e);
    if (rc != PQW_OK) return rc;
  }
  CU(cudaSetDevice(e->device));
  e->free_device();
  // stages that need the GPU, longest first (LPT order for the work queue)
  std::vector<int> ids;
  for (size_t i = 0; i < e->stages.size(); ++i)
    if (e->active[i] && e->stages[i].status == PQW_STAGE_OK) ids.push_back((int)i);
  std::stable_sort(ids.begin(), ids.end(), [&](int a, int b) {
    return e->stages[a].prog().code.size() > e->stages[b].prog().code.size();
  });
  e->gpu_stage_of = ids;
  e->n_gpu_stages = (uint32_t)ids.size();
  std::vector<pqw_ins> code;
  std::vector<pqw::StageDesc> descs;
  std::vector<uint32_t> work;
  std::unordered_map<const std::vector<pqw_ins>*, uint32_t> placed;  // shared programs: one copy
  e->max_slots = 0;
  e->spill_slots = 0;
  e->n_code = 0;
  std::fill(std::begin(e->op_hist), std::end(e->op_hist), 0);
  std::fill(std::begin(e->cls), std::end(e->cls), 0);
  for (size_t r = 0; r < ids.size(); ++r) {
    const auto& st = e->stages[ids[r]];
    if (st.n_warps != e->n_warps) return fail(PQW_EINVAL, "stage compiled for another warp count");
    const auto& pr = st.prog();
    auto pit = placed.find(&pr.code);
    uint32_t off;
    if (pit == placed.end()) {
      off = (uint32_t)code.size();
      placed.emplace(&pr.code, off);
      code.insert(code.end(), pr.code.begin(), pr.code.end());
    } else {
      off = pit->second;
    }
    descs.push_back({off, pr.n_slots, st.var_base, (uint32_t)r});
    work.push_back((uint32_t)r);
    e->max_slots = std::max(e->max_slots, pr.n_slots);
    e->spill_slots = std::max(e->spill_slots, pr.n_spill);
    e->n_code += pr.code.size();
    for (int i = 0; i < PQW_B_NUM_OPS; ++i) e->op_hist[i] += pr.op_hist[i];
    for (int i = 0; i < 5; ++i) e->cls[i] += pr.cls[i];
  }
  e->n_code_unique = code.size();
  if (code.empty()) code.push_back(pqw_ins{PQW_B_END, 0, 0, 0});
  // the code rings fetch whole 32-record chunks, up to two past a stream's END
  for (uint32_t i = 0; i < 2 * 32; ++i) code.push_back(pqw_ins{PQW_B_END, 0, 0, 0});
  if (descs.empty()) descs.push_back({0, 0, 0, 0});
  if (work.empty()) work.push_back(0);

  // two attributes, not cudaGetDeviceProperties (which queries everything and
  // costs tens of milliseconds per call)
  int smem_optin = 0, n_sm = 0;
  CU(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, e->device));
  CU(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, e->device));
  // the shared value file is as large as the largest stage needs (at most the
  // capacity the stages were compiled for); spills live in per-CTA scratch
  const size_t slot_bytes = pqw::SLOT_BYTES;
  e->smem_slots = std::max<uint32_t>(e->max_slots, 1);
  const size_t smem_bytes = (size_t)e->smem_slots * slot_bytes + (size_t)e->n_warps * pqw::RING_BYTES;
  if (smem_bytes + 512 > (size_t)smem_optin)
    return fail(PQW_EINVAL, "value file does not fit in shared memory");
  int per_sm = 0;
  auto setup = [&](auto kern_false, auto kern_true, int threads) -> cudaError_t {
    cudaError_t err = cudaFuncSetAttribute(kern_false, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem_bytes);
    if (err == cudaSuccess)
      err = cudaFuncSetAttribute(kern_true, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem_bytes);
    if (err == cudaSuccess)
      err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern_false, threads, smem_bytes);
    return err;
  };
  if (e->n_warps == 32)
    CU(setup(pqw::eval_kernel<32, false>, pqw::eval_kernel<32, true>, 32 * 32));
  else if (e->n_warps == 16)
    CU(setup(pqw::eval_kernel<16, false>, pqw::eval_kernel<16, true>, 16 * 32));
  else
    CU(setup(pqw::eval_kernel<8, false>, pqw::eval_kernel<8, true>, 8 * 32));
  if (per_sm < 1) per_sm = 1;
  e->grid = (uint32_t)(n_sm * per_sm);

  // one block for the whole image (pooled across engines, see arena_get)
  const size_t nk = std::max<size_t>(e->var_keys.size(), 1);
  const size_t nr = std::max<size_t>(ids.size(), 1);
  e->scratch_bytes = (size_t)e->grid * std::max<uint32_t>(e->spill_slots, 1) * slot_bytes;
  const size_t sizes[11] = {code.size() * sizeof(pqw_ins), descs.size() * sizeof(pqw::StageDesc),
                            work.size() * sizeof(uint32_t), nk * sizeof(uint64_t),
                            3 * sizeof(uint64_t), sizeof(uint32_t), e->scratch_bytes,
                            nr * sizeof(unsigned long long), nr * sizeof(uint32_t),
                            nr * sizeof(uint32_t), 2 * sizeof(uint32_t)};
  size_t offs[11], total = 0;
  for (int i = 0; i < 11; ++i) {
    offs[i] = total;
    total += (sizes[i] + 255) & ~(size_t)255;
  }
  e->arena = pqw::arena_get(e->device, total, &e->arena_bytes);
  if (!e->arena) return fail(PQW_ECUDA, "device allocation of the image failed");
  char* base = static_cast<char*>(e->arena);
  e->d_code = reinterpret_cast<uint4*>(base + offs[0]);
  e->d_stages = reinterpret_cast<pqw::StageDesc*>(base + offs[1]);
  e->d_work = reinterpret_cast<uint32_t*>(base + offs[2]);
  e->d_var_keys = reinterpret_cast<uint64_t*>(base + offs[3]);
  e->d_fn_keys = reinterpret_cast<uint64_t*>(base + offs[4]);
  e->d_counter = reinterpret_cast<uint32_t*>(base + offs[5]);
  e->d_scratch = reinterpret_cast<uint32_t*>(base + offs[6]);
  e->d_first_bad = reinterpret_cast<unsigned long long*>(base + offs[7]);
  e->d_n_valid = reinterpret_cast<uint32_t*>(base + offs[8]);
  e->d_n_bad = reinterpret_cast<uint32_t*>(base + offs[9]);
  e->d_probe = reinterpret_cast<uint32_t*>(base + offs[10]);
  CU(cudaMemcpy(e->d_code, code.data(), code.size() * sizeof(pqw_ins), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(e->d_stages, descs.data(), descs.size() * sizeof(pqw::StageDesc),
                cudaMemcpyHostToDevice));
  CU(cudaMemcpy(e->d_work, work.data(), work.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
  if (!e->var_keys.empty())
    CU(cudaMemcpy(e->d_var_keys, e->var_keys.data(), e->var_keys.size() * sizeof(uint64_t),
                  cudaMemcpyHostToDevice));
  CU(cudaMemcpy(e->d_fn_keys, e->fn_keys, 3 * sizeof(uint64_t), cudaMemcpyHostToDevice));
  e->h2d_bytes = code.size() * sizeof(pqw_ins) + descs.size() * sizeof(pqw::StageDesc) +
                 work.size() * sizeof(uint32_t) + e->var_keys.size() * sizeof(uint64_t) +
                 3 * sizeof(uint64_t);
  if (!e->ev0) CU(cudaEventCreate(&e->ev0));
  if (!e->ev1) CU(cudaEventCreate(&e->ev1));
  e->uploaded = true;
  e->results_ready = false;
  return PQW_OK;
}

static int launch_eval(pqw_engine* e, const pqw::Params& p, uint32_t grid, bool probe,
                       cudaStream_t s) {
  const size_t smem_bytes =
      (size_t)e->smem_slots * pqw::SLOT_BYTES + (size_t)e->n_warps * pqw::RING_BYTES;
  if (e->n_warps == 32) {
    if (probe) pqw::eval_kernel<32, true><<<1, 32 * 32, smem_bytes, s>>>(p);
    else pqw::eval_kernel<32, false><<<grid, 32 * 32, smem_bytes, s>>>(p);
  } else if (e->n_warps == 16) {
    if (probe) pqw::eval_kernel<16, true><<<1, 16 * 32, smem_bytes, s>>>(p);
    else pqw::eval_kernel<16, false><<<grid, 16 * 32, smem_bytes, s>>>(p);
  } else {
    if (probe) pqw::eval_kernel<8, true><<<1, 8 * 32, smem_bytes, s>>>(p);
    else pqw::eval_kernel<8, false><<<grid, 8 * 32, smem_bytes, s>>>(p);
  }
  CU(cudaGetLastError());
  return PQW_OK;
}

int pqw_launch(pqw_engine* e, uint32_t n_witness, void* stream) {
  if (!e) return fail(PQW_EINVAL, "null engine");
  if (!e->uploaded) return fail(PQW_ESTATE, "pqw_launch before pqw_upload");
  if (n_witness == 0) return fail(PQW_EINVAL, "n_witness must be positive");
  CU(cudaSetDevice(e->device));
  cudaStream_t s = (cudaStream_t)stream;
  const size_t nr = std::max<size_t>(e->n_gpu_stages, 1);
  CU(cudaMemsetAsync(e->d_first_bad, 0xFF, nr * sizeof(unsigned long long), s));
  CU(cudaMemsetAsync(e->d_n_valid, 0, nr * sizeof(uint32_t), s));
  CU(cudaMemsetAsync(e->d_n_bad, 0, nr * sizeof(uint32_t), s));
  CU(cudaMemsetAsync(e->d_counter, 0, sizeof(uint32_t), s));
  e->results_ready = false;
  e->timed = false;
  if (e->n_gpu_stages == 0) return PQW_OK;
  pqw::Params p{};
  p.code = reinterpret_cast<const uint4*>(e->d_code);
  p.stages = e->d_stages;
  p.work = e->d_work;
  p.var_keys = e->d_var_keys;
  p.fn_keys = e->d_fn_keys;
  p.counter = e->d_counter;
  p.scratch = e->d_scratch;
  p.first_bad = e->d_first_bad;
  p.n_valid = e->d_n_valid;
  p.n_bad = e->d_n_bad;
  p.tiles = (n_witness + pqw::TW - 1) / pqw::TW;
  p.n_items = e->n_gpu_stages * p.tiles;
  p.n_witness = n_witness;
  p.spill_slots = std::max<uint32_t>(e->spill_slots, 1);
  p.file_bytes = e->smem_slots * pqw::SLOT_BYTES;
  p.sleep_ns = e->sleep_ns;
#ifdef PQW_PROF
  static unsigned long long* d_prof = nullptr;
  if (!d_prof) CU(cudaMalloc(&d_prof, 80 * sizeof(unsigned long long)));
  CU(cudaMemsetAsync(d_prof, 0, 80 * sizeof(unsigned long long), s));
  p.prof = d_prof;
  e->d_prof_last = d_prof;
#endif
  uint32_t grid = std::min<uint32_t>(e->grid, std::max<uint32_t>(p.n_items, 1));
  CU(cudaEventRecord(e->ev0, s));
  int rc = launch_eval(e, p, grid, false, s);
  if (rc != PQW_OK) return rc;
  CU(cudaEventRecord(e->ev1, s));
  e->timed = true;
  return PQW_OK;
}

int pqw_results(pqw_engine* e, uint64_t* first_bad, uint32_t* n_valid, uint32_t* n_bad,
                size_t n_stages) {
  if (!e) return fail(PQW_EINVAL, "null engine");
  if (n_stages != e->stages.size()) return fail(PQW_EINVAL, "n_stages must equal stage count");
  if (!e->uploaded) return fail(PQW_ESTATE, "no uploaded image");
  CU(cudaSetDevice(e->device));
  const size_t nr = e->n_gpu_stages;
  e->h_first_bad.resize(nr);
  e->h_valid.resize(nr);
  e->h_bad.resize(nr);
  if (e->timed) CU(cudaEventSynchronize(e->ev1));
  CU(cudaDeviceSynchronize());
  if (nr) {
    CU(cudaMemcpy(e->h_first_bad.data(), e->d_first_bad, nr * sizeof(unsigned long long),
                  cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(e->h_valid.data(), e->d_n_valid, nr * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(e->h_bad.data(), e->d_n_bad, nr * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  }
#ifdef PQW_PROF
  if (e->d_prof_last) {
    unsigned long long pr[80];
    CU(cudaMemcpy(pr, e->d_prof_last, sizeof(pr), cudaMemcpyDeviceToHost));
    fprintf(stderr, "PQW_PROF warp-cycles: item %.3e wait %.3e (%.1f%%) end-barrier %.3e (%.1f%%)\n",
            (double)pr[0], (double)pr[1], 100.0 * pr[1] / pr[0], (double)pr[2], 100.0 * pr[2] / pr[0]);
    static const char* names[18] = {"DOT1", "DOT2", "DOTk", "SUM2", "SUMk", "SUB", "NEG", "HASH",
                                    "INV", "VAR", "CONST", "CHK", "DEN", "FILL", "SPILL", "WAIT",
                                    "?", "?"};
    for (int c = 0; c < 16; ++c) {
      const unsigned long long* q = pr + 8 + 4 * c;
      if (!q[2]) continue;
      fprintf(stderr, "PQW_PROF %-5s bundles %10llu groups %10llu cyc/group %8.1f cyc/bundle %8.1f "
              "dispatch/bundle %7.1f share %.1f%%\n", names[c], q[2], q[1],
              q[1] ? (double)q[0] / q[1] : 0.0, (double)q[0] / q[2], (double)q[3] / q[2],
              100.0 * (q[0] + q[3]) / pr[0]);
    }
  }
#endif
  for (size_t i = 0; i < n_stages; ++i) {
    if (first_bad) first_bad[i] = ~0ull;
    if (n_valid) n_valid[i] = 0;
    if (n_bad) n_bad[i] = 0;
  }
  for (size_t r = 0; r < nr; ++r) {
    int sidx = e->gpu_stage_of[r];
    if (first_bad) first_bad[sidx] = e->h_first_bad[r];
    if (n_valid) n_valid[sidx] = e->h_valid[r];
    if (n_bad) n_bad[sidx] = e->h_bad[r];
  }
  return PQW_OK;
}

int pqw_probe(pqw_engine* e, int stage, uint32_t witness, uint32_t obl, uint32_t* lhs,
              uint32_t* rhs, uint32_t* var_vals, size_t n_vars) {
  if (!e || stage < 0 || (size_t)stage >= e->stages.size()) return fail(PQW_EINVAL, "bad stage");
  if (!e->uploaded) return fail(PQW_ESTATE, "pqw_probe before pqw_upload");
  const auto& st = e->stages[stage];
  if (st.status != PQW_STAGE_OK) return fail(PQW_EINVAL, "stage has no GPU program");
  if (var_vals && n_vars < st.n_vars) return fail(PQW_EINVAL, "var_vals too short");
  CU(cudaSetDevice(e->device));
  uint32_t r = 0;
  for (; r < e->n_gpu_stages; ++r)
    if (e->gpu_stage_of[r] == stage) break;
  uint32_t* d_vars = nullptr;
  CU(cudaMalloc(&d_vars, std::max<size_t>(st.n_vars, 1) * sizeof(uint32_t)));
  // variables the program never reads (pruned by value numbering) keep this
  // marker (not a field element) and get their value from the host below
  CU(cudaMemset(d_vars, 0xFF, std::max<size_t>(st.n_vars, 1) * sizeof(uint32_t)));
  uint32_t* d_work1 = nullptr;
  CU(cudaMalloc(&d_work1, sizeof(uint32_t)));
  CU(cudaMemcpy(d_work1, &r, sizeof(uint32_t), cudaMemcpyHostToDevice));
  uint32_t init[2] = {0xFFFFFFFFu, 0xFFFFFFFFu};
  CU(cudaMemcpy(e->d_probe, init, sizeof(init), cudaMemcpyHostToDevice));
  pqw::Params p{};
  p.code = reinterpret_cast<const uint4*>(e->d_code);
  p.stages = e->d_stages;
  p.work = d_work1;
  p.var_keys = e->d_var_keys;
  p.fn_keys = e->d_fn_keys;
  p.counter = e->d_counter;
  p.scratch = e->d_scratch;
  p.n_items = 1;
  p.tiles = 1;
  p.n_witness = witness + 1;
  p.spill_slots = std::max<uint32_t>(e->spill_slots, 1);
  p.file_bytes = e->smem_slots * pqw::SLOT_BYTES;
  p.sleep_ns = e->sleep_ns;
  p.probe_w = witness;
  p.probe_obl = obl;
  p.probe_out = e->d_probe;
  p.probe_vars = d_vars;
  {
    int rc = launch_eval(e, p, 1, true, 0);
    if (rc != PQW_OK) return rc;
  }
  CU(cudaDeviceSynchronize());
  uint32_t got[2];
  CU(cudaMemcpy(got, e->d_probe, sizeof(got), cudaMemcpyDeviceToHost));
  if (lhs) *lhs = got[0];
  if (rhs) *rhs = got[1];
  if (var_vals && st.n_vars) {
    CU(cudaMemcpy(var_vals, d_vars, st.n_vars * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    for (uint32_t i = 0; i < st.n_vars; ++i)
      if (var_vals[i] == 0xFFFFFFFFu)
        var_vals[i] = pqw::witness_value(e->var_keys[st.var_base + i], witness);
  }
  cudaFree(d_vars);
  cudaFree(d_work1);
  return PQW_OK;
}

int pqw_confirm(pqw_engine* e, int stage, uint32_t witness, const double* env_vals, size_t n_env,
                double tol, int64_t out[4], double sides[2]) {
  if (!e || !out || !sides || (n_env && !env_vals)) return fail(PQW_EINVAL, "null argument");
  if (stage < 0 || (size_t)stage >= e->stages.size()) return fail(PQW_EINVAL, "bad stage");
  {
    int rc = finalize_front(e);
    if (rc != PQW_OK) return rc;
  }
  const size_t root = e->alias[stage] < 0 ? (size_t)stage : (size_t)e->alias[stage];
  auto it = e->cache_src.find(root);
  if (it == e->cache_src.end()) return fail(PQW_ESTATE, "stage program not retained");
  const auto& src = it->second;
  const uint32_t base = e->pend_base[stage], nv = e->pend_nvars[stage];
  try {
    int rc = pqw::confirm_stage(src.first.data(), src.first.size(), src.second.data(),
                                src.second.size() / 3, nv, e->fn_keys,
                                e->var_keys.data() + base, witness, env_vals, n_env, tol, out,
                                sides);
    if (rc < 0) return fail(PQW_ESTATE, "stage has no value graph");
  } catch (const std::exception& ex) {
    return fail(PQW_EINVAL, std::string("confirm: ") + ex.what());
  }
  return PQW_OK;
}

int pqw_last_launch_ms(pqw_engine* e, float* ms) {
  if (!e || !ms) return fail(PQW_EINVAL, "null argument");
  if (!e->timed) {
    *ms = 0.f;
    return PQW_OK;
  }
  CU(cudaSetDevice(e->device));
  CU(cudaEventSynchronize(e->ev1));
  CU(cudaEventElapsedTime(ms, e->ev0, e->ev1));
  return PQW_OK;
}

int pqw_image_stats(pqw_engine* e, uint64_t* out, size_t cap) {
  if (!e || !out) return fail(PQW_EINVAL, "null argument");
  constexpr int N = PQW_B_NUM_OPS;
  uint64_t buf[PQW_IMAGE_STATS_LEN] = {};
  {
    int rc = finalize_all(e);
    if (rc != PQW_OK) return rc;
  }
  uint64_t n_gpu = 0, n_code = 0, max_slots = 0, max_spill = 0, bundles = 0, waits = 0;
  for (size_t si = 0; si < e->stages.size(); ++si) {
    const auto& st = e->stages[si];
    if (st.status != PQW_STAGE_OK || !e->active[si]) continue;
    n_gpu++;
    const auto& pr = st.prog();
    n_code += pr.code.size();
    max_slots = std::max<uint64_t>(max_slots, pr.n_slots);
    max_spill = std::max<uint64_t>(max_spill, pr.n_spill);
    bundles += pr.n_bundles;
    waits += pr.n_waits;
    for (int i = 0; i < N; ++i) buf[4 + i] += pr.op_hist[i];
    for (int i = 0; i < 5; ++i) buf[6 + N + i] += pr.cls[i];
  }
  buf[0] = n_gpu;
  buf[1] = n_code;
  buf[2] = max_slots;
  buf[3] = e->smem_slots;
  buf[4 + N] = e->n_code_unique;
  buf[5 + N] = e->cache_hits;
  buf[11 + N] = max_spill;
  buf[12 + N] = bundles;
  buf[13 + N] = waits;
  buf[14 + N] = e->h2d_bytes;
  buf[15 + N] = (uint64_t)e->n_gpu_stages * (sizeof(unsigned long long) + 2 * sizeof(uint32_t));
  std::memcpy(out, buf, std::min(cap, (size_t)PQW_IMAGE_STATS_LEN) * sizeof(uint64_t));
  return PQW_OK;
}

int pqw_peak_fieldops(int device, double out[4]) {
  if (!out) return fail(PQW_EINVAL, "null argument");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= device) {
    cudaGetLastError();
    return fail(PQW_ENODEV, "no CUDA device");
  }
  CU(cudaSetDevice(device));
  cudaDeviceProp prop;
  CU(cudaGetDeviceProperties(&prop, device));
  const int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 2048;
  uint32_t* sink = nullptr;
  CU(cudaMalloc(&sink, (size_t)blocks * threads * sizeof(uint32_t)));
  cudaEvent_t e0, e1;
  CU(cudaEventCreate(&e0));
  CU(cudaEventCreate(&e1));
  for (int kind = 0; kind < 4; ++kind) {
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      int it = kind == 2 ? iters / 8 : kind == 3 ? iters / 32 : iters;
      CU(cudaEventRecord(e0));
      if (kind == 0) pqw::peak_kernel<0><<<blocks, threads>>>(sink, it, rep);
      else if (kind == 1) pqw::peak_kernel<1><<<blocks, threads>>>(sink, it, rep);
      else if (kind == 2) pqw::peak_kernel<2><<<blocks, threads>>>(sink, it, rep);
      else pqw::peak_kernel<3><<<blocks, threads>>>(sink, it, rep);
      CU(cudaEventRecord(e1));
      CU(cudaEventSynchronize(e1));
      float ms = 0;
      CU(cudaEventElapsedTime(&ms, e0, e1));
      if (rep > 0 && ms < best) best = ms;  // rep 0 warms up
    }
    double n_ops = (double)blocks * threads * (kind == 2 ? iters / 8 : kind == 3 ? iters / 32 : iters) * 16 * 8;
    out[kind] = n_ops / (best * 1e-3);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  return PQW_OK;
}

}  // extern "C"

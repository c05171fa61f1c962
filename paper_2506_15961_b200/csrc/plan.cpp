// plan.cpp -- native plan core: stage construction and lowering (pqw_plan_* C-ABI).
//
// What the reference does on the host before deciding anything, per plan and
// per stage, done once here over flat arrays:
//   validate_concrete  pkg/src/planeq/shapes.py:35-45 (shape rule of every node,
//                      rules of ops.py:100-909 as restated in opshape.py)
//   entry_order        pkg/src/planeq/stages.py:79-88
//   build_stages       pkg/src/planeq/stages.py:91-138 (backward slices cut at
//                      checkpoints, graph.py:303-328; topo order graph.py:96-150)
//   stage lowering     pkg/src/planeq/stages.py:144-176 + :267-340 (interface,
//                      both sub-DFGs, obligations) -- emits, word for word, the
//                      tensor-op program paper_2506_15961_b200/stages.py
//                      lower_stage emits, so pqw_stage_add cannot tell them apart.
// Any input the reference would reject yields PQW_EPLAN; the Python host then
// runs its own checks, which raise the reference's exception and message.
#include <sched.h>
#include <sys/mman.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <queue>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "../../include/planeq_witness.h"
#include "field.hpp"
#include "pool.hpp"

namespace pqw {
int set_last_error(int code, const std::string& msg);  // witness_kernel.cu (pqw_last_error)
// engine side of pqw_stage_add (witness_kernel.cu)
uint64_t program_hash(const int32_t* ir, size_t ir_len, const int64_t* consts, size_t n_consts,
                      size_t n_vars);
bool cached_program(const pqw_engine* e, uint64_t h, const std::vector<int32_t>** ir,
                    const std::vector<int64_t>** consts, int* stage);
int stage_add_hashed(pqw_engine* e, const int32_t* ir, size_t ir_len, const int64_t* consts,
                     size_t n_consts, const uint64_t* var_keys, size_t n_vars, uint64_t h,
                     int same, std::vector<int32_t>* own_ir, std::vector<int64_t>* own_consts,
                     int64_t out_status[16]);
namespace {

int pfail(int code, const std::string& msg) { return set_last_error(code, msg); }

struct PlanError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

constexpr int32_t IR_MAGIC = 0x50515701;

// encoded attribute layouts (paper_2506_15961_b200/native.py pack_attrs)
bool is_elementwise2(int k) {
  return k == PQW_T_ADD || k == PQW_T_SUB || k == PQW_T_MUL || k == PQW_T_DIV ||
         k == PQW_T_DROPOUT || k == PQW_T_SILU_GRAD;
}
bool is_unary(int k) {
  return k == PQW_T_IDENTITY || k == PQW_T_SCALE || k == PQW_T_SHIFT || k == PQW_T_POW ||
         k == PQW_T_RSQRT || k == PQW_T_SILU || k == PQW_T_MOVE;
}
bool is_comm(int k) {
  return k == PQW_T_ALL_REDUCE || k == PQW_T_ALL_GATHER || k == PQW_T_REDUCE_SCATTER ||
         k == PQW_T_ALL_TO_ALL;
}

int64_t pymod(int64_t a, int64_t m) {
  int64_t r = a % m;
  return r < 0 ? r + m : r;
}

// Storage of the plan's big columns (tens of MB on the 405B plan): no
// value-initialisation on resize -- the columns are filled by parallel copies,
// so their pages are first touched on the workers -- and transparent huge
// pages for blocks of 4 MB and more.
template <class T>
struct ColAlloc {
  using value_type = T;
  static constexpr size_t BIG = 4u << 20, H = 2u << 20;
  ColAlloc() = default;
  template <class U>
  ColAlloc(const ColAlloc<U>&) {}
  T* allocate(size_t n) {
    const size_t b = n * sizeof(T);
    if (b < BIG) return static_cast<T*>(::operator new(b));
    const size_t r = (b + H - 1) & ~(H - 1);
    void* q = std::aligned_alloc(H, r);
    if (!q) throw std::bad_alloc();
    madvise(q, r, MADV_HUGEPAGE);
    return static_cast<T*>(q);
  }
  void deallocate(T* q, size_t n) {
    if (n * sizeof(T) < BIG)
      ::operator delete(q);
    else
      std::free(q);
  }
  template <class U, class... A>
  void construct(U* q, A&&... a) {
    if constexpr (sizeof...(A) == 0 && std::is_trivially_copyable_v<U>)
      return;  // left for the filling copy
    else
      ::new (static_cast<void*>(q)) U(std::forward<A>(a)...);
  }
  friend bool operator==(const ColAlloc&, const ColAlloc&) { return true; }
  friend bool operator!=(const ColAlloc&, const ColAlloc&) { return false; }
};
template <class T>
using Col = std::vector<T, ColAlloc<T>>;

unsigned host_threads(size_t work) {
  unsigned nt = std::max(1u, std::thread::hardware_concurrency());
  cpu_set_t cs;
  if (sched_getaffinity(0, sizeof(cs), &cs) == 0) nt = std::max(1, CPU_COUNT(&cs));
  if (const char* s = getenv("PQW_THREADS")) nt = std::max(1, atoi(s));
  return (unsigned)std::max<size_t>(1, std::min<size_t>(nt, work));
}

template <class F>
void parallel_for(size_t n, F&& f) {
  const unsigned nt = host_threads(n);
  std::atomic<size_t> next{0};
  run_on_threads(nt, [&](unsigned tid) {
    for (;;) {
      const size_t i = next.fetch_add(1);
      if (i >= n) return;
      f(i, tid);
    }
  });
}

template <class T, class A>
void par_copy(std::vector<T, A>& v, const T* src, size_t n) {
  v.resize(n);
  const size_t chunk = (1u << 20) / sizeof(T);
  parallel_for((n + chunk - 1) / chunk, [&](size_t c, unsigned) {
    const size_t a = c * chunk, e = std::min(n, a + chunk);
    std::memcpy(v.data() + a, src + a, (e - a) * sizeof(T));
  });
}

// Byte length of n NUL-terminated names: a word-at-a-time count of the NULs
// (aligned 8-byte reads never cross into a page past the buffer's last one).
size_t names_len(const char* s, int64_t n) {
  if (n <= 0) return 0;
  const char* p = s;
  int64_t left = n;
  while ((reinterpret_cast<uintptr_t>(p) & 7u) != 0) {
    if (*p++ == 0 && --left == 0) return (size_t)(p - s);
  }
  constexpr uint64_t L7 = 0x7F7F7F7F7F7F7F7Full;
  for (;;) {
    uint64_t w;
    std::memcpy(&w, p, 8);
    const uint64_t z = ~(((w & L7) + L7) | w | L7);  // 0x80 in every zero byte
    const int c = __builtin_popcountll(z);
    if (c < left) {
      left -= c;
      p += 8;
      continue;
    }
    for (int b = 0; b < 8; ++b)
      if (p[b] == 0 && --left == 0) return (size_t)(p + b + 1 - s);
  }
}

// K chunks of a names buffer cut at name boundaries, with the index of each
// chunk's first name (cut and first have K + 1 entries).
void cut_names(const char* s, size_t len, unsigned K, std::vector<size_t>& cut,
               std::vector<size_t>& first) {
  cut.assign(K + 1, len);
  cut[0] = 0;
  for (unsigned k = 1; k < K; ++k) {
    size_t c = std::max(len * k / K, cut[k - 1]);
    while (c < len && c > 0 && s[c - 1] != 0) ++c;  // start right after a NUL
    cut[k] = c;
  }
  first.assign(K + 1, 0);
  parallel_for(K, [&](size_t k, unsigned) {
    size_t c = 0;
    for (size_t i = cut[k]; i < cut[k + 1]; ++i) c += s[i] == 0;
    first[k + 1] = c;
  });
  for (unsigned k = 0; k < K; ++k) first[k + 1] += first[k];
}

// copy the n NUL-separated names once, then view into the copy
void split_names(const char* s, int64_t n, Col<char>& store, Col<std::string_view>& out,
                 int64_t known_len = 0) {
  const size_t len = known_len > 0 ? (size_t)known_len : names_len(s, n);
  par_copy(store, s, len);
  out.resize((size_t)n);
  const unsigned K = host_threads(std::max<size_t>(1, len / (1u << 20)));
  std::vector<size_t> cut, first;
  cut_names(store.data(), len, K, cut, first);
  parallel_for(K, [&](size_t k, unsigned) {
    size_t idx = first[k];
    for (size_t i = cut[k]; i < cut[k + 1] && idx < (size_t)n; ++idx) {
      const size_t l = std::strlen(store.data() + i);
      out[idx] = std::string_view(store.data() + i, l);
      i += l + 1;
    }
  });
}

// Open-addressing name -> index table, built in parallel (CAS on the slots)
// and then read from many threads.
struct NameTable {
  Col<uint64_t> hs;                            // hash per name index
  std::unique_ptr<std::atomic<int32_t>[]> slot;  // name index per slot, -1 empty
  const Col<std::string_view>* names = nullptr;
  uint64_t mask = 0;

  static uint64_t h(std::string_view s) {
    uint64_t x = 0xCBF29CE484222325ull;
    size_t i = 0;
    for (; i + 8 <= s.size(); i += 8) {
      uint64_t w;
      std::memcpy(&w, s.data() + i, 8);
      x = (x ^ w) * 0x100000001B3ull;
      x ^= x >> 29;
    }
    for (; i < s.size(); ++i) x = (x ^ (unsigned char)s[i]) * 0x100000001B3ull;
    return mix64(x ^ s.size());
  }
  // returns false on a duplicate name
  bool build(const Col<std::string_view>& ns) {
    names = &ns;
    size_t cap = 16;
    while (cap < ns.size() * 2) cap <<= 1;
    mask = cap - 1;
    slot.reset(new std::atomic<int32_t>[cap]);
    hs.resize(ns.size());
    const size_t chunk = 65536;
    const size_t nc = (std::max(ns.size(), cap) + chunk - 1) / chunk;
    parallel_for(nc, [&](size_t c, unsigned) {
      for (size_t k = c * chunk; k < std::min(cap, (c + 1) * chunk); ++k)
        slot[k].store(-1, std::memory_order_relaxed);
      for (size_t i = c * chunk; i < std::min(ns.size(), (c + 1) * chunk); ++i) hs[i] = h(ns[i]);
    });
    std::atomic<bool> unique{true};
    parallel_for((ns.size() + chunk - 1) / chunk, [&](size_t c, unsigned) {
      for (size_t i = c * chunk; i < std::min(ns.size(), (c + 1) * chunk); ++i) {
        for (uint64_t k = hs[i] & mask;; k = (k + 1) & mask) {
          int32_t cur = slot[k].load(std::memory_order_acquire);
          if (cur < 0) {
            if (slot[k].compare_exchange_strong(cur, (int32_t)i, std::memory_order_acq_rel))
              break;
            // lost the race: cur now holds the winner, compare with it below
          }
          if (hs[(size_t)cur] == hs[i] && ns[(size_t)cur] == ns[i]) {
            unique.store(false, std::memory_order_relaxed);
            break;
          }
        }
      }
    });
    return unique.load();
  }
  int32_t find(std::string_view s) const {
    const uint64_t hv = h(s);
    for (uint64_t k = hv & mask;; k = (k + 1) & mask) {
      const int32_t cur = slot[k].load(std::memory_order_relaxed);
      if (cur < 0) return -1;
      if (hs[(size_t)cur] == hv && (*names)[(size_t)cur] == s) return cur;
    }
  }
};

struct GraphData {
  Col<char> tstore, nstore;
  Col<std::string_view> tname, nid;
  Col<int64_t> dim_off, dims;
  Col<uint8_t> tflags;
  Col<int32_t> kind;
  Col<int64_t> in_off, out_off, attr_off;
  Col<int32_t> ins, outs;  // tensor indices, -1 unresolved
  Col<int64_t> attrs;
  Col<int32_t> device;
  Col<int64_t> seq;
  std::vector<uint8_t> is_input;
  std::vector<int32_t> producer;   // tensor -> node, -1 none
  NameTable index;
  bool resolved = true;            // every node input/output names a tensor
  bool unique_producers = true;
  std::string problem;

  size_t nt() const { return tname.size(); }
  size_t nn() const { return kind.size(); }
  std::vector<int64_t> shape_vec(int32_t t) const {
    return std::vector<int64_t>(dims.begin() + dim_off[t], dims.begin() + dim_off[t + 1]);
  }
  int32_t find(std::string_view s) const { return index.find(s); }
  // topological key (graph.py:136 rank: device or -1, seq, id)
  bool before(int32_t a, int32_t b) const {
    if (device[a] != device[b]) return device[a] < device[b];
    if (seq[a] != seq[b]) return seq[a] < seq[b];
    return nid[a] < nid[b];
  }

  // n NUL-terminated names -> tensor indices, read in place: the buffer is cut
  // into chunks at name boundaries, names counted per chunk, then resolved in
  // parallel (no copy of the names is kept)
  template <class V>
  void resolve(const char* names, int64_t n, V& out, int64_t known_len = 0) {
    out.resize((size_t)n);
    if (n == 0) return;
    const size_t len = known_len > 0 ? (size_t)known_len : names_len(names, n);
    const unsigned K = host_threads(std::max<size_t>(1, len / (1u << 20)));
    std::vector<size_t> cut, first;
    cut_names(names, len, K, cut, first);
    std::atomic<bool> all{true};
    parallel_for(K, [&](size_t k, unsigned) {
      size_t idx = first[k];
      for (size_t i = cut[k]; i < cut[k + 1] && idx < (size_t)n; ++idx) {
        const size_t l = std::strlen(names + i);
        out[idx] = find(std::string_view(names + i, l));
        if (out[idx] < 0) all = false;
        i += l + 1;
      }
    });
    if (!all) resolved = false;
  }

  void load(const pqw_graph_desc& d) {
    static const bool timing = getenv("PQW_TIMING") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto t0 = now();
    auto lap = [&](const char* what) {
      if (!timing) return;
      auto t = now();
      fprintf(stderr, "PQW_TIMING load %s %.1f ms\n", what,
              std::chrono::duration<double, std::milli>(t - t0).count());
      t0 = t;
    };
    split_names(d.tensor_names, d.n_tensors, tstore, tname, d.tensor_names_len);
    lap("tensor names");
    if (!index.build(tname)) {
      resolved = false;
      problem = "duplicate tensor id";
    }
    lap("tensor table");
    dim_off.resize((size_t)d.n_tensors + 1);
    dim_off[0] = 0;
    for (int64_t i = 0; i < d.n_tensors; ++i) dim_off[i + 1] = dim_off[i] + d.tensor_ndim[i];
    par_copy(dims, d.tensor_dims, (size_t)dim_off.back());
    par_copy(tflags, d.tensor_flags, (size_t)d.n_tensors);
    lap("  tensor dims");
    const size_t n = (size_t)d.n_nodes;
    split_names(d.node_ids, d.n_nodes, nstore, nid, d.node_ids_len);
    lap("  node ids");
    par_copy(kind, d.node_kind, n);
    par_copy(device, d.node_device, n);
    par_copy(seq, d.node_seq, n);
    lap("  kind/device/seq");
    in_off.resize(n + 1);
    out_off.resize(n + 1);
    attr_off.resize(n + 1);
    in_off[0] = out_off[0] = attr_off[0] = 0;
    for (size_t i = 0; i < n; ++i) {
      in_off[i + 1] = in_off[i] + d.node_nin[i];
      out_off[i + 1] = out_off[i] + d.node_nout[i];
      attr_off[i + 1] = attr_off[i] + d.node_nattr[i];
    }
    par_copy(attrs, d.node_attrs, (size_t)attr_off[n]);
    lap("node columns");
    resolve(d.node_inputs, in_off[n], ins, d.node_inputs_len);
    resolve(d.node_outputs, out_off[n], outs, d.node_outputs_len);
    lap("resolve io");
    {
      std::vector<int32_t> gin;
      const bool keep = resolved;
      resolve(d.input_names, d.n_inputs, gin, d.input_names_len);
      resolved = keep;  // graph.inputs may name anything (it is only a set of ids)
      is_input.assign(nt(), 0);
      for (int32_t t : gin)
        if (t >= 0) is_input[t] = 1;
    }
    producer.assign(nt(), -1);
    for (size_t v = 0; v < n; ++v)
      for (int64_t j = out_off[v]; j < out_off[v + 1]; ++j) {
        int32_t t = outs[j];
        if (t < 0) continue;
        if (producer[t] >= 0) unique_producers = false;
        producer[t] = (int32_t)v;
      }
    lap("inputs+producers");
    // node ids must be unique for the (device, seq, id) order to be total
    NameTable ids;
    if (!ids.build(nid)) {
      resolved = false;
      problem = "duplicate node id";
    }
    lap("node id table");
  }
};

struct Entry {
  int32_t logical = -1;  // logical tensor
  uint8_t mode = 0;
  std::vector<int32_t> shards;                      // parallel tensors
  std::vector<std::vector<std::pair<int64_t, int64_t>>> ranges;
};

struct StageRec {
  int32_t target = -1;   // logical tensor
  int32_t entry = -1;
  std::vector<int32_t> lnodes, pnodes;  // topo order
  std::vector<int32_t> l_inputs, p_inputs;  // sorted by name
};

// Per-thread scratch: generation-stamped marks over tensors and nodes.
struct Marks {
  // calloc'd: a fresh large block is untouched zero pages, so a per-thread
  // Marks over a million-node graph costs only the pages its slices visit
  uint32_t* stamp = nullptr;
  size_t n = 0;
  uint32_t gen = 0;
  Marks() = default;
  Marks(const Marks&) = delete;
  Marks& operator=(const Marks&) = delete;
  ~Marks() { std::free(stamp); }
  void reset(size_t m) {
    if (m != n || !stamp) {
      std::free(stamp);
      stamp = static_cast<uint32_t*>(std::calloc(std::max<size_t>(m, 1), sizeof(uint32_t)));
      if (!stamp) throw std::bad_alloc();
      n = m;
      gen = 0;
    }
    if (++gen == 0) {
      std::memset(stamp, 0, n * sizeof(uint32_t));
      gen = 1;
    }
  }
  bool test(size_t i) const { return stamp[i] == gen; }
  bool set(size_t i) {  // true if newly set
    if (stamp[i] == gen) return false;
    stamp[i] = gen;
    return true;
  }
};

}  // namespace
}  // namespace pqw

struct pqw_plan {
  pqw::GraphData L, P;
  std::vector<pqw::Entry> entries;
  std::vector<int32_t> entry_of_logical;  // logical tensor -> entry, -1
  std::vector<int64_t> consts;             // triples
  bool lineage_ok = true;
  bool validated = false;
  bool built = false;
  std::vector<int32_t> order;              // entry_order (entry indices)
  std::vector<int32_t> owner;              // parallel tensor -> earliest claiming entry
  std::vector<pqw::StageRec> stages;
  std::vector<int32_t> uncovered[2];
};

namespace pqw {
namespace {

// ---- validate_concrete -------------------------------------------------------

using Shape = std::vector<int64_t>;

int64_t volume(const Shape& s) {
  int64_t v = 1;
  for (auto d : s) v *= d;
  return v;
}

struct ShapeFail {};

void want(bool c) {
  if (!c) throw ShapeFail{};
}

// einsum spec (code points) -> subscripts, rhs; as opshape.einsum_parse
void einsum_split(const int64_t* a, int64_t n, size_t n_in, std::vector<std::vector<int64_t>>& subs,
                  std::vector<int64_t>& rhs) {
  std::vector<int64_t> sp;
  for (int64_t i = 0; i < n; ++i)
    if (a[i] != ' ') sp.push_back(a[i]);
  int arrows = 0;
  size_t at = 0;
  for (size_t i = 0; i + 1 < sp.size(); ++i)
    if (sp[i] == '-' && sp[i + 1] == '>') {
      arrows++;
      at = i;
    }
  if (arrows != 1) throw PlanError("einsum spec");
  subs.assign(1, {});
  for (size_t i = 0; i < at; ++i) {
    if (sp[i] == ',') subs.emplace_back();
    else subs.back().push_back(sp[i]);
  }
  rhs.assign(sp.begin() + at + 2, sp.end());
  if (subs.size() != n_in) throw ShapeFail{};
}

std::vector<Shape> infer(int k, const int64_t* a, int64_t na, const std::vector<Shape>& ins) {
  auto at = [&](int64_t i) -> int64_t {
    if (i >= na) throw PlanError("attribute words");
    return a[i];
  };
  if (k < PQW_T_ADD || k > PQW_T_ALL_TO_ALL) throw PlanError("unknown operator");
  if (is_elementwise2(k)) {
    want(ins.size() == 2);
    want(ins[1] == ins[0]);
    return {ins[0]};
  }
  if (is_unary(k)) {
    want(ins.size() == 1);
    if (k == PQW_T_POW) want(at(0) >= 1);
    return {ins[0]};
  }
  switch (k) {
    case PQW_T_SOFTMAX: {
      want(ins.size() == 1);
      const int64_t ax = at(0);
      want(ax == -1 || ax == (int64_t)ins[0].size() - 1);
      want(!ins[0].empty() && ins[0].back() >= 2);
      return {ins[0]};
    }
    case PQW_T_CREATE_MASK: {
      want(ins.empty());
      const int64_t s = at(0);
      want(s >= 2);
      return {Shape{s, s}};
    }
    case PQW_T_APPLY_MASK: {
      want(ins.size() == 2);
      const Shape &x = ins[0], &m = ins[1];
      want(m.size() == 2 && m[0] == m[1]);
      want(x.size() >= 2 && x[x.size() - 2] == m[0] && x[x.size() - 1] == m[1]);
      return {x};
    }
    case PQW_T_VIEW: {
      want(ins.size() == 1);
      Shape t(a + 1, a + 1 + at(0));
      want(volume(ins[0]) == volume(t));
      return {t};
    }
    case PQW_T_TRANSPOSE: {
      want(ins.size() == 1);
      Shape perm(a, a + na), sorted = perm;
      std::sort(sorted.begin(), sorted.end());
      want(sorted.size() == ins[0].size());
      for (size_t i = 0; i < sorted.size(); ++i) want(sorted[i] == (int64_t)i);
      Shape out;
      for (auto p : perm) out.push_back(ins[0][p]);
      return {out};
    }
    case PQW_T_EXPAND: {
      if (ins.empty()) throw PlanError("expand without input");
      Shape t(a + 1, a + 1 + at(0));
      const Shape& s = ins[0];
      want(t.size() == s.size());
      for (size_t i = 0; i < s.size(); ++i) want(s[i] == t[i] || s[i] == 1);
      return {t};
    }
    case PQW_T_SUM:
    case PQW_T_MEAN: {
      want(ins.size() == 1);
      const int64_t r = (int64_t)ins[0].size();
      const bool keep = at(0) != 0;
      std::vector<char> red((size_t)r, 0);
      if (at(1) == 0) {
        std::fill(red.begin(), red.end(), 1);
      } else {
        if (r == 0) throw PlanError("reduce of rank 0");
        for (int64_t i = 0; i < at(2); ++i) red[(size_t)pymod(at(3 + i), r)] = 1;
      }
      Shape out;
      for (int64_t ax = 0; ax < r; ++ax) {
        if (red[ax]) {
          if (keep) out.push_back(1);
        } else {
          out.push_back(ins[0][ax]);
        }
      }
      if (out.empty()) out.push_back(1);
      return {out};
    }
    case PQW_T_MATMUL: {
      want(ins.size() == 2);
      const Shape &x = ins[0], &y = ins[1];
      want(x.size() >= 2 && y.size() >= 2);
      want(y.size() == x.size() || y.size() == 2);
      if (y.size() == x.size())
        want(std::equal(x.begin(), x.end() - 2, y.begin()));
      want(x[x.size() - 1] == y[y.size() - 2]);
      Shape out(x.begin(), x.end() - 1);
      out.push_back(y.back());
      return {out};
    }
    case PQW_T_EINSUM: {
      std::vector<std::vector<int64_t>> subs;
      std::vector<int64_t> rhs;
      einsum_split(a + 1, at(0), ins.size(), subs, rhs);
      std::vector<std::pair<int64_t, int64_t>> extent;  // (char, extent) in first-seen order
      auto find = [&](int64_t ch) -> int64_t* {
        for (auto& e : extent)
          if (e.first == ch) return &e.second;
        return nullptr;
      };
      for (size_t i = 0; i < subs.size(); ++i) {
        want(subs[i].size() == ins[i].size());
        for (size_t j = 0; j < subs[i].size(); ++j) {
          int64_t* e = find(subs[i][j]);
          if (e) want(*e == ins[i][j]);
          else extent.push_back({subs[i][j], ins[i][j]});
        }
      }
      int64_t vol = 1;
      bool any = false;
      for (auto& e : extent)
        if (std::find(rhs.begin(), rhs.end(), e.first) == rhs.end()) {
          any = true;
          vol *= e.second;
        }
      if (any) want(vol >= 2);
      Shape out;
      for (auto ch : rhs) {
        int64_t* e = find(ch);
        if (!e) throw PlanError("einsum output index not in inputs");
        out.push_back(*e);
      }
      return {out};
    }
    case PQW_T_FULL: {
      want(ins.empty());
      return {Shape(a + 2, a + 2 + at(1))};
    }
    case PQW_T_CHUNK: {
      if (ins.empty()) throw PlanError("chunk without input");
      const int64_t r = (int64_t)ins[0].size();
      int64_t ax = at(0);
      if (ax < -r || ax >= r) throw PlanError("chunk axis");
      ax = pymod(ax, r);
      const int64_t parts = at(1), idx = at(2), d = ins[0][ax];
      want(parts >= 1 && idx >= 0 && idx < parts);
      want(d % parts == 0);
      Shape out = ins[0];
      out[ax] = d / parts;
      return {out};
    }
    case PQW_T_EMBEDDING: {
      want(ins.size() == 2);
      want(ins[0].size() == 2);
      want(ins[0][0] >= volume(ins[1]));
      Shape out = ins[1];
      out.push_back(ins[0][1]);
      return {out};
    }
    case PQW_T_EMBEDDING_GRAD: {
      if (ins.size() != 2) throw PlanError("embedding_grad arity");
      const Shape &g = ins[0], &ids = ins[1];
      want(!g.empty() && g.size() - 1 == ids.size() && std::equal(ids.begin(), ids.end(), g.begin()));
      const int64_t v = at(0);
      want(v >= volume(ids));
      return {Shape{v, g.back()}};
    }
    case PQW_T_GNORM_SQ:
      want(!ins.empty());
      return {Shape{1}};
    default:
      break;
  }
  // communication: group of n, n inputs, n outputs
  const int64_t n = at(0);
  want((int64_t)ins.size() == n);
  if (n == 0) throw PlanError("empty group");
  const int64_t r = (int64_t)ins[0].size();
  auto axis = [&](int64_t ax) {
    if (ax < -r || ax >= r) throw PlanError("axis out of range");
    return pymod(ax, r);
  };
  if (k == PQW_T_ALL_REDUCE) {
    for (auto& s : ins) want(s == ins[0]);
    return std::vector<Shape>((size_t)n, ins[0]);
  }
  if (k == PQW_T_ALL_GATHER) {
    // opshape.py compares s[:ax] + s[ax+1:] with Python slicing on the raw
    // axis (a negative axis -1 keeps the whole shape in the second slice)
    const int64_t ax = at(1);
    auto clamp = [](int64_t i, int64_t len) {
      if (i < 0) i += len;
      return std::min(std::max<int64_t>(i, 0), len);
    };
    auto off_axis = [&](const Shape& s) {
      const int64_t len = (int64_t)s.size();
      Shape o(s.begin(), s.begin() + clamp(ax, len));
      o.insert(o.end(), s.begin() + clamp(ax + 1, len), s.end());
      return o;
    };
    Shape base = ins[0];
    const Shape want_off = off_axis(base);
    int64_t total = 0;
    for (auto& s : ins) {
      want(off_axis(s) == want_off);
      const int64_t len = (int64_t)s.size();
      if (ax < -len || ax >= len) throw PlanError("axis out of range");
      total += s[(size_t)pymod(ax, len)];
    }
    base[(size_t)axis(ax)] = total;
    return std::vector<Shape>((size_t)n, base);
  }
  if (k == PQW_T_REDUCE_SCATTER) {
    const int64_t ax = axis(at(1));
    for (auto& s : ins) want(s == ins[0]);
    want(ins[0][ax] % n == 0);
    Shape out = ins[0];
    out[ax] /= n;
    return std::vector<Shape>((size_t)n, out);
  }
  const int64_t sa = axis(at(1)), ca = axis(at(2));
  for (auto& s : ins) want(s == ins[0]);
  want(ins[0][sa] % n == 0);
  Shape out = ins[0];
  out[sa] /= n;
  out[ca] *= n;
  return std::vector<Shape>((size_t)n, out);
}

// Python negative-index semantics are applied by the packer only where the
// reference normalises (softmax axis is compared raw); nothing else to do.

bool validate_graph(const GraphData& g, std::string& why) {
  if (!g.resolved) {
    why = g.problem.empty() ? "unresolved tensor name" : g.problem;
    return false;
  }
  // dangling inputs (graph.py topo_sort) and cycles
  const size_t n = g.nn();
  // Fast path: when every producer precedes its consumer in node order (a
  // graph built front to back), there is no cycle; only dangling inputs need
  // looking for. One parallel pass instead of the serial Kahn sweep below.
  {
    std::atomic<int> state{0};  // 0 forward, 1 dangling, 2 a backward edge
    const size_t chunk = 16384;
    parallel_for((n + chunk - 1) / chunk, [&](size_t c, unsigned) {
      for (size_t v = c * chunk; v < std::min(n, (c + 1) * chunk); ++v)
        for (int64_t j = g.in_off[v]; j < g.in_off[v + 1]; ++j) {
          const int32_t t = g.ins[j];
          if (g.is_input[t]) continue;
          const int32_t src = g.producer[t];
          if (src < 0) {
            state.store(1);
            return;
          }
          if ((size_t)src >= v) {
            int expect = 0;
            state.compare_exchange_strong(expect, 2);
          }
        }
    });
    if (state.load() == 1) {
      why = "dangling tensor";
      return false;
    }
    if (state.load() == 0) goto shapes;
  }
  {
  // successor lists in CSR form (no per-node allocation)
  std::vector<int32_t> indeg(n, 0), soff(n + 1, 0);
  for (size_t v = 0; v < n; ++v)
    for (int64_t j = g.in_off[v]; j < g.in_off[v + 1]; ++j) {
      const int32_t t = g.ins[j];
      if (g.is_input[t]) continue;
      const int32_t src = g.producer[t];
      if (src < 0) {
        why = "dangling tensor";
        return false;
      }
      indeg[v]++;
      soff[(size_t)src + 1]++;
    }
  for (size_t v = 0; v < n; ++v) soff[v + 1] += soff[v];
  {
    std::vector<int32_t> succ((size_t)soff[n]), fill(soff.begin(), soff.end() - 1);
    for (size_t v = 0; v < n; ++v)
      for (int64_t j = g.in_off[v]; j < g.in_off[v + 1]; ++j) {
        const int32_t t = g.ins[j];
        if (g.is_input[t]) continue;
        succ[(size_t)fill[(size_t)g.producer[t]]++] = (int32_t)v;
      }
    std::vector<int32_t> q;
    for (size_t v = 0; v < n; ++v)
      if (!indeg[v]) q.push_back((int32_t)v);
    size_t seen = 0;
    while (!q.empty()) {
      int32_t v = q.back();
      q.pop_back();
      seen++;
      for (int32_t i = soff[(size_t)v]; i < soff[(size_t)v + 1]; ++i)
        if (--indeg[(size_t)succ[(size_t)i]] == 0) q.push_back(succ[(size_t)i]);
    }
    if (seen != n) {
      why = "cycle";
      return false;
    }
  }
  }
shapes:
  auto same_shape = [&](int32_t a, int32_t b) {
    const int64_t la = g.dim_off[a + 1] - g.dim_off[a], lb = g.dim_off[b + 1] - g.dim_off[b];
    return la == lb && std::equal(g.dims.begin() + g.dim_off[a], g.dims.begin() + g.dim_off[a + 1],
                                  g.dims.begin() + g.dim_off[b]);
  };
  std::atomic<bool> ok{true};
  std::mutex mu;
  const size_t chunk = 4096;
  parallel_for((n + chunk - 1) / chunk, [&](size_t c, unsigned) {
    std::vector<Shape> ins;
    for (size_t v = c * chunk; v < std::min(n, (c + 1) * chunk) && ok.load(std::memory_order_relaxed); ++v) {
      const int k = g.kind[v];
      const int64_t ni = g.in_off[v + 1] - g.in_off[v], nov = g.out_off[v + 1] - g.out_off[v];
      // the common kinds without allocation: outputs equal the (shared) input shape
      if ((is_elementwise2(k) && ni == 2 &&
           same_shape(g.ins[g.in_off[v]], g.ins[g.in_off[v] + 1])) ||
          (is_unary(k) && ni == 1 &&
           (k != PQW_T_POW || (g.attr_off[v + 1] > g.attr_off[v] && g.attrs[g.attr_off[v]] >= 1)))) {
        bool good = true;
        for (int64_t j = 0; j < nov && j < 1; ++j)
          good = good && same_shape(g.outs[g.out_off[v] + j], g.ins[g.in_off[v]]);
        if (good) continue;
      }
      ins.clear();
      for (int64_t j = g.in_off[v]; j < g.in_off[v + 1]; ++j) ins.push_back(g.shape_vec(g.ins[j]));
      bool good = true;
      try {
        auto got = infer(k, g.attrs.data() + g.attr_off[v], g.attr_off[v + 1] - g.attr_off[v], ins);
        // zip(outputs, got): only the common prefix is compared (opshape.py)
        const int64_t no = g.out_off[v + 1] - g.out_off[v];
        for (int64_t j = 0; j < no && (size_t)j < got.size(); ++j)
          if (g.shape_vec(g.outs[g.out_off[v] + j]) != got[(size_t)j]) good = false;
      } catch (...) {
        good = false;
      }
      if (!good) {
        ok = false;
        std::lock_guard<std::mutex> l(mu);
        why = std::string("node ") + std::string(g.nid[v]);
      }
    }
  });
  return ok.load();
}

// ---- stage construction -------------------------------------------------------

// Deterministic Kahn order of `nodes` (graph.py topo_sort with the (device,
// seq, id) tie-break); `picked` marks exactly `nodes`. Throws PlanError on a
// dangling input or a cycle.
// `nodes` sorted ascending, all marked in `picked`; graph.py:96-150 order
// (Kahn's algorithm, ready nodes by (device, seq, id))
// Reusable per-thread buffers of topo_order (a stage's slice is a few hundred
// nodes; allocating them per call cost more than the sort itself).
std::atomic<uint64_t> topo_fast_hits{0};

struct TopoScratch {
  std::vector<int32_t> loc;  // node -> position in `nodes` (valid where picked)
  std::vector<int32_t> indeg, soff, src_of, dst_of, succ, fill, heap;
  std::vector<int32_t> dev;
  std::vector<int64_t> seq;
};

std::vector<int32_t> topo_order(const GraphData& g, const std::vector<int32_t>& nodes,
                                const Marks& picked, TopoScratch& S) {
  const size_t n = nodes.size();
  if (S.loc.size() < g.nn()) S.loc.resize(g.nn());
  for (size_t i = 0; i < n; ++i) S.loc[(size_t)nodes[i]] = (int32_t)i;
  // the (device, seq) part of the key, contiguous; ties fall back to the id
  S.dev.resize(n);
  S.seq.resize(n);
  for (size_t i = 0; i < n; ++i) {
    S.dev[i] = g.device[(size_t)nodes[i]];
    S.seq[i] = g.seq[(size_t)nodes[i]];
  }
  // in-edges within the slice as CSR of successors
  S.indeg.assign(n, 0);
  S.soff.assign(n + 1, 0);
  S.src_of.clear();
  S.dst_of.clear();
  for (size_t i = 0; i < n; ++i) {
    const int32_t v = nodes[i];
    for (int64_t j = g.in_off[v]; j < g.in_off[v + 1]; ++j) {
      const int32_t t = g.ins[j];
      if (g.is_input[t]) continue;
      const int32_t src = g.producer[t];
      if (src >= 0 && picked.test((size_t)src)) {
        S.indeg[i]++;
        const int32_t k = S.loc[(size_t)src];
        S.soff[(size_t)k + 1]++;
        S.src_of.push_back(k);
        S.dst_of.push_back((int32_t)i);
      } else if (src < 0) {
        throw PlanError("dangling tensor");
      }
    }
  }
  // Fast path: when the slice's nodes, ascending by index, are already in key
  // order and every in-slice edge points forward, that order is the Kahn order
  // (the smallest remaining key is always ready).
  {
    bool sorted_topo = true;
    for (size_t i = 1; i < n && sorted_topo; ++i)
      sorted_topo = (S.dev[i - 1] != S.dev[i]) ? S.dev[i - 1] < S.dev[i]
                  : (S.seq[i - 1] != S.seq[i]) ? S.seq[i - 1] < S.seq[i]
                  : g.nid[(size_t)nodes[i - 1]] < g.nid[(size_t)nodes[i]];
    for (size_t e = 0; e < S.src_of.size() && sorted_topo; ++e)
      sorted_topo = S.src_of[e] < S.dst_of[e];
    if (sorted_topo) {
      topo_fast_hits.fetch_add(1, std::memory_order_relaxed);
      return nodes;
    }
  }
  for (size_t i = 0; i < n; ++i) S.soff[i + 1] += S.soff[i];
  S.succ.resize(S.src_of.size());
  S.fill.assign(S.soff.begin(), S.soff.end() - 1);
  for (size_t e = 0; e < S.src_of.size(); ++e)
    S.succ[(size_t)S.fill[(size_t)S.src_of[e]]++] = S.dst_of[e];
  // g.before on slice positions (graph.py:136 rank: device, seq, id)
  auto before = [&](int32_t a, int32_t b) {
    if (S.dev[a] != S.dev[b]) return S.dev[a] < S.dev[b];
    if (S.seq[a] != S.seq[b]) return S.seq[a] < S.seq[b];
    return g.nid[(size_t)nodes[a]] < g.nid[(size_t)nodes[b]];
  };
  auto cmp = [&](int32_t a, int32_t b) { return before(b, a); };  // min-heap
  auto& heap = S.heap;
  heap.clear();
  for (size_t i = 0; i < n; ++i)
    if (!S.indeg[i]) heap.push_back((int32_t)i);
  std::make_heap(heap.begin(), heap.end(), cmp);
  std::vector<int32_t> out;
  out.reserve(n);
  while (!heap.empty()) {
    std::pop_heap(heap.begin(), heap.end(), cmp);
    const int32_t i = heap.back();
    heap.pop_back();
    out.push_back(nodes[i]);
    for (int32_t e = S.soff[(size_t)i]; e < S.soff[(size_t)i + 1]; ++e) {
      const int32_t s2 = S.succ[(size_t)e];
      if (--S.indeg[(size_t)s2] == 0) {
        heap.push_back(s2);
        std::push_heap(heap.begin(), heap.end(), cmp);
      }
    }
  }
  if (out.size() != n) throw PlanError("cycle");
  return out;
}

// graph.py backward_slice: nodes reached from roots without passing stop
// tensors; returns picked nodes (marked in `picked`) and the boundary.
void backward_slice(const GraphData& g, const std::vector<int32_t>& roots,
                    const std::function<bool(int32_t)>& stop, Marks& seen, Marks& picked,
                    std::vector<int32_t>& nodes, std::vector<int32_t>& boundary) {
  seen.reset(g.nt());
  picked.reset(g.nn());
  nodes.clear();
  boundary.clear();
  std::vector<int32_t> stack(roots.rbegin(), roots.rend());
  // (the reference pops from the end; order does not change the result sets)
  while (!stack.empty()) {
    const int32_t t = stack.back();
    stack.pop_back();
    if (!seen.set((size_t)t)) continue;
    const int32_t v = g.producer[t];
    const bool st = stop(t);
    if (st || v < 0) {
      if (st || g.is_input[t]) boundary.push_back(t);
      continue;
    }
    if (picked.set((size_t)v)) {
      nodes.push_back(v);
      for (int64_t j = g.in_off[v]; j < g.in_off[v + 1]; ++j) stack.push_back(g.ins[j]);
    }
  }
}

void sort_by_name(const GraphData& g, std::vector<int32_t>& ts) {
  std::sort(ts.begin(), ts.end(), [&](int32_t a, int32_t b) { return g.tname[a] < g.tname[b]; });
}

void build(pqw_plan* p) {
  static const bool timing = getenv("PQW_TIMING") != nullptr;
  auto lap = [t = std::chrono::steady_clock::now()](const char* what) mutable {
    const auto now = std::chrono::steady_clock::now();
    if (timing)
      fprintf(stderr, "PQW_TIMING build %s %.1f ms\n", what,
              std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  };
  const GraphData &L = p->L, &P = p->P;
  // entry_order: logical topological position of the producer, inputs first
  std::vector<int32_t> all(L.nn());
  for (size_t i = 0; i < all.size(); ++i) all[i] = (int32_t)i;
  Marks everything;
  everything.reset(L.nn());
  for (size_t i = 0; i < all.size(); ++i) everything.set(i);
  TopoScratch ts0;
  const auto lorder = topo_order(L, all, everything, ts0);
  std::vector<int64_t> pos(L.nn(), -1);
  for (size_t i = 0; i < lorder.size(); ++i) pos[lorder[i]] = (int64_t)i;
  const size_t ne = p->entries.size();
  p->order.resize(ne);
  for (size_t i = 0; i < ne; ++i) p->order[i] = (int32_t)i;
  auto epos = [&](int32_t e) {
    const int32_t v = L.producer[p->entries[e].logical];
    return v < 0 ? (int64_t)-1 : pos[v];
  };
  std::sort(p->order.begin(), p->order.end(), [&](int32_t a, int32_t b) {
    const int64_t pa = epos(a), pb = epos(b);
    if (pa != pb) return pa < pb;
    return L.tname[p->entries[a].logical] < L.tname[p->entries[b].logical];
  });
  std::vector<int32_t> rank(ne);
  for (size_t r = 0; r < ne; ++r) rank[p->order[r]] = (int32_t)r;
  // earliest checkpoint claiming each shard tensor
  p->owner.assign(P.nt(), -1);
  for (size_t r = ne; r-- > 0;)
    for (int32_t s : p->entries[p->order[r]].shards) p->owner[s] = p->order[r];
  // a shard is an "earlier shard" of stage r iff some entry of rank < r lists it:
  // first_rank[s] = smallest rank of an entry listing s
  std::vector<int32_t> first_rank(P.nt(), INT32_MAX);
  for (size_t r = 0; r < ne; ++r)
    for (int32_t s : p->entries[p->order[r]].shards)
      first_rank[s] = std::min(first_rank[s], (int32_t)r);
  lap("entry order");
  std::vector<int32_t> produced;  // ranks of produced checkpoints
  for (size_t r = 0; r < ne; ++r)
    if (L.producer[p->entries[p->order[r]].logical] >= 0) produced.push_back((int32_t)r);
  p->stages.assign(produced.size(), StageRec{});
  std::mutex err_mu;
  std::string err;
  const unsigned nt = host_threads(produced.size());
  std::vector<Marks> seen_l(nt), picked_l(nt), seen_p(nt), picked_p(nt);
  std::vector<TopoScratch> tscr(nt);
  std::vector<std::array<double, 6>> acc(nt, std::array<double, 6>{});
  parallel_for(produced.size(), [&](size_t si, unsigned tid) {
    auto tick = [&](int k, std::chrono::steady_clock::time_point& t) {
      if (!timing) return;
      const auto now = std::chrono::steady_clock::now();
      acc[tid][k] += std::chrono::duration<double, std::milli>(now - t).count();
      t = now;
    };
    auto tt = std::chrono::steady_clock::now();
    try {
      const int32_t r = produced[si];
      const Entry& e = p->entries[p->order[r]];
      StageRec& st = p->stages[si];
      st.target = e.logical;
      st.entry = p->order[r];
      std::vector<int32_t> nodes, bound;
      backward_slice(L, {e.logical},
                     [&](int32_t t) { return t != e.logical && p->entry_of_logical[t] >= 0; },
                     seen_l[tid], picked_l[tid], nodes, bound);
      tick(0, tt);
      std::sort(nodes.begin(), nodes.end());
      st.lnodes = topo_order(L, nodes, picked_l[tid], tscr[tid]);
      tick(1, tt);
      for (int32_t b : bound)
        if (p->entry_of_logical[b] < 0) throw PlanError("logical input has no checkpoint entry");
      sort_by_name(L, bound);
      st.l_inputs = bound;
      backward_slice(P, e.shards, [&](int32_t t) { return first_rank[t] < r; }, seen_p[tid],
                     picked_p[tid], nodes, bound);
      tick(2, tt);
      if (timing) acc[tid][5] += (double)nodes.size();
      std::sort(nodes.begin(), nodes.end());
      st.pnodes = topo_order(P, nodes, picked_p[tid], tscr[tid]);
      tick(3, tt);
      for (int32_t b : bound)
        if (!(first_rank[b] < r)) throw PlanError("parallel input is not a checkpoint shard");
      sort_by_name(P, bound);
      st.p_inputs = bound;
      tick(4, tt);
    } catch (const std::exception& ex) {
      std::lock_guard<std::mutex> l(err_mu);
      if (err.empty()) err = ex.what();
    }
  });
  if (!err.empty()) throw PlanError(err);
  if (timing) {
    std::array<double, 6> tot{};
    for (auto& a : acc)
      for (int k = 0; k < 6; ++k) tot[k] += a[k];
    fprintf(stderr, "PQW_TIMING slices (thread-ms) lslice %.1f ltopo %.1f pslice %.1f ptopo %.1f rest %.1f; parallel slice nodes %.0f; index-order fast path %llu\n",
            tot[0], tot[1], tot[2], tot[3], tot[4], tot[5], (unsigned long long)topo_fast_hits.load());
  }
  lap("slices");
  // ownership in stage order: a node belongs to the first stage whose slice has it
  for (int side = 0; side < 2; ++side) {
    const GraphData& g = side ? P : L;
    std::vector<char> claimed(g.nn(), 0);
    for (auto& st : p->stages)
      for (int32_t v : side ? st.pnodes : st.lnodes) claimed[v] = 1;
    auto& u = p->uncovered[side];
    u.clear();
    for (size_t v = 0; v < g.nn(); ++v)
      if (!claimed[v]) u.push_back((int32_t)v);
    std::sort(u.begin(), u.end(), [&](int32_t a, int32_t b) { return g.nid[a] < g.nid[b]; });
  }
  lap("uncovered");
}

// ---- lowering ---------------------------------------------------------------------

uint64_t fnv1a64(std::string_view a, std::string_view b) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (unsigned char c : a) h = (h ^ c) * 0x100000001B3ull;
  for (unsigned char c : b) h = (h ^ c) * 0x100000001B3ull;
  return h;
}

struct Program {
  std::vector<int32_t> ir;
  std::vector<int64_t> consts;
  std::vector<uint64_t> var_keys;
};

// tensor index -> local value, with O(1) reset: generation-stamped arrays
// that live per host thread across the stages it lowers
struct StampMap {
  std::vector<uint32_t> stamp;
  std::vector<int32_t> val;
  uint32_t gen = 0;
  void begin(size_t n) {
    if (stamp.size() < n) {
      stamp.assign(n, 0);
      val.assign(n, -1);
      gen = 0;
    }
    if (++gen == 0) {
      std::fill(stamp.begin(), stamp.end(), 0);
      gen = 1;
    }
  }
  int32_t get(int32_t k) const { return stamp[(size_t)k] == gen ? val[(size_t)k] : -1; }
  void set(int32_t k, int32_t v) {
    stamp[(size_t)k] = gen;
    val[(size_t)k] = v;
  }
};

struct LowerScratch {
  StampMap lt, pt, boxes, prod_l, prod_p;
};

struct Lowerer {
  const pqw_plan* p = nullptr;
  uint64_t seed = 0;
  std::vector<int64_t> sdims;          // local tensor shapes, flat
  std::vector<int32_t> soff{0};
  std::vector<int32_t> ops;
  int32_t n_ops = 0;
  std::vector<int64_t> consts;
  std::unordered_map<int64_t, int32_t> const_idx;  // plan const id -> stage const index
  std::vector<uint64_t> var_keys;
  int64_t n_vars = 0;
  StampMap* lt_ = nullptr;             // "L:" keys -> local tensor
  StampMap* pt_ = nullptr;             // "P:" keys -> local tensor
  StampMap* boxes_ = nullptr;          // logical tensor -> local tensor
  std::vector<int32_t> abuf;           // attribute words of the node being emitted

  int32_t temp(const int64_t* d, size_t n) {
    sdims.insert(sdims.end(), d, d + n);
    soff.push_back((int32_t)sdims.size());
    return (int32_t)soff.size() - 2;
  }
  int32_t temp(const Shape& s) { return temp(s.data(), s.size()); }
  size_t rank(int32_t t) const { return (size_t)(soff[(size_t)t + 1] - soff[(size_t)t]); }
  int32_t tensor(StampMap& m, int32_t key, const int64_t* d, size_t n) {
    const int32_t got = m.get(key);
    if (got >= 0) return got;
    const int32_t idx = temp(d, n);
    m.set(key, idx);
    return idx;
  }
  int32_t tensor(StampMap& m, int32_t key, const Shape& s) { return tensor(m, key, s.data(), s.size()); }
  int32_t cst(int64_t cid) {
    auto it = const_idx.find(cid);
    if (it != const_idx.end()) return it->second;
    if (cid < 0 || (size_t)(3 * cid + 2) >= p->consts.size()) throw PlanError("const id");
    const int32_t idx = (int32_t)(consts.size() / 3);
    consts.insert(consts.end(), p->consts.begin() + 3 * cid, p->consts.begin() + 3 * cid + 3);
    const_idx.emplace(cid, idx);
    return idx;
  }
  void emit(int32_t op, const std::vector<int32_t>& ins, const std::vector<int32_t>& outs,
            const std::vector<int32_t>& attrs) {
    ops.push_back(op);
    ops.push_back((int32_t)ins.size());
    ops.push_back((int32_t)outs.size());
    ops.push_back((int32_t)attrs.size());
    ops.insert(ops.end(), ins.begin(), ins.end());
    ops.insert(ops.end(), outs.begin(), outs.end());
    ops.insert(ops.end(), attrs.begin(), attrs.end());
    n_ops++;
  }
  int32_t vars_for(std::string_view pre, std::string_view name, const Shape& s) {
    const int64_t n = volume(s);
    const int32_t out = temp(s);
    emit(PQW_T_VARS, {}, {out}, {(int32_t)n_vars});
    // stages.py tensor_var_keys: mix64(base + (i+1) * VAR_STEP)
    const uint64_t base = seed ^ fnv1a64(std::string("var:") + std::string(pre), name);
    for (int64_t i = 0; i < n; ++i)
      var_keys.push_back(mix64(base + (uint64_t)(i + 1) * 0xD1B54A32D192ED03ull));
    n_vars += n;
    return out;
  }
  int32_t box_of(int32_t tid) {
    const int32_t got = boxes_->get(tid);
    if (got >= 0) return got;
    const GraphData& L = p->L;
    const Shape s = L.shape_vec(tid);
    int32_t idx;
    if (L.tflags[tid] & 1) {
      if (!(L.tflags[tid] & 2)) throw PlanError("integer checkpoint has no enumerated values");
      idx = temp(s);
      const int32_t base = (int32_t)(consts.size() / 3);
      const int64_t n = volume(s);
      for (int64_t v = 0; v < n; ++v) {
        consts.push_back(v % (int64_t)PQW_PRIME);
        consts.push_back(v);
        consts.push_back(1);
      }
      emit(PQW_T_INTS, {}, {idx}, {base});
    } else {
      idx = vars_for("v.", L.tname[tid], s);
    }
    boxes_->set(tid, idx);
    return idx;
  }

  std::vector<int32_t> node_attrs(const GraphData& g, int32_t v, const std::vector<int32_t>& in) {
    const int k = g.kind[v];
    const int64_t* a = g.attrs.data() + g.attr_off[v];
    const int64_t na = g.attr_off[v + 1] - g.attr_off[v];
    auto at = [&](int64_t i) -> int64_t {
      if (i >= na) throw PlanError("attribute words");
      return a[i];
    };
    auto rank0 = [&]() -> int64_t {
      if (in.empty()) throw PlanError("no input");
      return (int64_t)rank(in[0]);
    };
    switch (k) {
      case PQW_T_SCALE:
      case PQW_T_SHIFT:
      case PQW_T_FULL:
        return {cst(at(0))};
      case PQW_T_POW:
        return {(int32_t)at(0)};
      case PQW_T_DIV:
        return {(int32_t)(at(0) != 0)};
      case PQW_T_TRANSPOSE: {
        std::vector<int32_t> out;
        for (int64_t i = 0; i < na; ++i) out.push_back((int32_t)a[i]);
        return out;
      }
      case PQW_T_SUM:
      case PQW_T_MEAN: {
        const int64_t r = rank0();
        std::vector<int32_t> out{(int32_t)(at(0) != 0)};
        std::vector<int64_t> axes;
        if (at(1) == 0) {
          for (int64_t i = 0; i < r; ++i) axes.push_back(i);
        } else {
          if (r == 0) throw PlanError("reduce of rank 0");
          for (int64_t i = 0; i < at(2); ++i) axes.push_back(pymod(at(3 + i), r));
          std::sort(axes.begin(), axes.end());
        }
        for (auto x : axes) out.push_back((int32_t)x);
        return out;
      }
      case PQW_T_EINSUM: {
        std::vector<std::vector<int64_t>> subs;
        std::vector<int64_t> rhs;
        try {
          einsum_split(a + 1, at(0), in.size(), subs, rhs);
        } catch (const ShapeFail&) {
          throw PlanError("einsum arity");
        }
        std::vector<int32_t> out{(int32_t)subs.size()};
        for (auto& s : subs) {
          out.push_back((int32_t)s.size());
          for (auto c : s) out.push_back((int32_t)c);
        }
        out.push_back((int32_t)rhs.size());
        for (auto c : rhs) out.push_back((int32_t)c);
        return out;
      }
      case PQW_T_CHUNK: {
        const int64_t r = rank0();
        if (r == 0) throw PlanError("chunk of rank 0");
        return {(int32_t)pymod(at(0), r), (int32_t)at(1), (int32_t)at(2)};
      }
      case PQW_T_ALL_GATHER:
      case PQW_T_REDUCE_SCATTER: {
        const int64_t r = rank0();
        if (r == 0) throw PlanError("rank 0");
        return {(int32_t)pymod(at(1), r)};
      }
      case PQW_T_ALL_TO_ALL: {
        const int64_t r = rank0();
        if (r == 0) throw PlanError("rank 0");
        return {(int32_t)pymod(at(1), r), (int32_t)pymod(at(2), r)};
      }
      default:
        return {};
    }
  }

  void run_nodes(const GraphData& g, const std::vector<int32_t>& nodes, StampMap& m, int side) {
    emit(PQW_T_SIDE, {}, {}, {side});
    std::vector<int32_t> in, out;
    for (int32_t v : nodes) {
      if (g.kind[v] < PQW_T_ADD || g.kind[v] > PQW_T_ALL_TO_ALL) throw PlanError("unknown operator");
      in.clear();
      out.clear();
      for (int64_t j = g.in_off[v]; j < g.in_off[v + 1]; ++j) {
        const int32_t got = m.get(g.ins[j]);
        if (got < 0) throw PlanError("unbound input");
        in.push_back(got);
      }
      for (int64_t j = g.out_off[v]; j < g.out_off[v + 1]; ++j) {
        const int32_t t = g.outs[j];
        out.push_back(tensor(m, t, g.dims.data() + g.dim_off[t],
                             (size_t)(g.dim_off[t + 1] - g.dim_off[t])));
      }
      emit(g.kind[v], in, out, node_attrs(g, v, in));
    }
  }

  static std::vector<int32_t> lows(const std::vector<std::pair<int64_t, int64_t>>& rs) {
    std::vector<int32_t> out;
    for (auto& r : rs) out.push_back((int32_t)r.first);
    return out;
  }
  static Shape extents(const std::vector<std::pair<int64_t, int64_t>>& rs) {
    Shape out;
    for (auto& r : rs) out.push_back(r.second - r.first);
    return out;
  }

  // entry.groups() sorted by ranges; members sorted by tensor name
  std::vector<std::pair<std::vector<std::pair<int64_t, int64_t>>, std::vector<int32_t>>> groups(
      const Entry& e) const {
    std::vector<std::pair<std::vector<std::pair<int64_t, int64_t>>, std::vector<int32_t>>> gs;
    for (size_t i = 0; i < e.shards.size(); ++i) {
      auto it = std::find_if(gs.begin(), gs.end(), [&](auto& g) { return g.first == e.ranges[i]; });
      if (it == gs.end()) gs.push_back({e.ranges[i], {e.shards[i]}});
      else it->second.push_back(e.shards[i]);
    }
    std::sort(gs.begin(), gs.end(), [](auto& a, auto& b) { return a.first < b.first; });
    for (auto& g : gs)
      std::stable_sort(g.second.begin(), g.second.end(),
                       [&](int32_t a, int32_t b) { return p->P.tname[a] < p->P.tname[b]; });
    return gs;
  }

  Program lower(const StageRec& st) {
    const GraphData &L = p->L, &P = p->P;
    static thread_local LowerScratch scratch;
    scratch.lt.begin(L.nt());
    scratch.boxes.begin(L.nt());
    scratch.prod_l.begin(L.nt());
    scratch.pt.begin(P.nt());
    scratch.prod_p.begin(P.nt());
    StampMap &lt = scratch.lt, &pt = scratch.pt, &prod_l = scratch.prod_l,
             &prod_p = scratch.prod_p;
    lt_ = &lt;
    pt_ = &pt;
    boxes_ = &scratch.boxes;
    for (int32_t v : st.lnodes)
      for (int64_t j = L.out_off[v]; j < L.out_off[v + 1]; ++j) prod_l.set(L.outs[j], 1);
    for (int32_t t : st.l_inputs)
      if (prod_l.get(t) < 0) lt.set(t, box_of(t));
    run_nodes(L, st.lnodes, lt, 0);
    for (int32_t v : st.pnodes)
      for (int64_t j = P.out_off[v]; j < P.out_off[v + 1]; ++j) prod_p.set(P.outs[j], 1);
    std::vector<int32_t> done;
    for (int32_t s : st.p_inputs) {
      if (prod_p.get(s) >= 0) continue;
      const int32_t ei = p->owner[s];
      if (ei < 0) throw PlanError("shard without owner");
      if (std::find(done.begin(), done.end(), ei) != done.end()) continue;
      done.push_back(ei);
      const Entry& e = p->entries[ei];
      const int32_t box = box_of(e.logical);
      if (e.mode == 0) {
        for (size_t i = 0; i < e.shards.size(); ++i) {
          const int32_t out = tensor(pt, e.shards[i], extents(e.ranges[i]));
          emit(PQW_T_SLICE, {box}, {out}, lows(e.ranges[i]));
        }
        continue;
      }
      if (L.tflags[e.logical] & 1) throw PlanError("partial checkpoint over integer tensor");
      for (auto& g : groups(e)) {
        const Shape ext = extents(g.first);
        std::vector<int32_t> frees;
        for (size_t i = 0; i + 1 < g.second.size(); ++i) {
          const int32_t v = vars_for("ps.", P.tname[g.second[i]], ext);
          pt.set(g.second[i], v);
          frees.push_back(v);
        }
        const int32_t sl = temp(ext);
        emit(PQW_T_SLICE, {box}, {sl}, lows(g.first));
        if (!frees.empty()) {
          const int32_t last = tensor(pt, g.second.back(), ext);
          std::vector<int32_t> ins{sl};
          ins.insert(ins.end(), frees.begin(), frees.end());
          emit(PQW_T_RESID, ins, {last}, {});
        } else {
          pt.set(g.second.back(), sl);
        }
      }
    }
    run_nodes(P, st.pnodes, pt, 1);
    // obligations (stages.py:316-340 order)
    const Entry& e = p->entries[st.entry];
    const int32_t tgt = lt.get(st.target);
    if (tgt < 0) throw PlanError("target not computed");
    int32_t n_obl = 0;
    auto shard_tensor = [&](int32_t s) {
      const int32_t got = pt.get(s);
      if (got < 0) throw PlanError("shard never computed");
      return got;
    };
    if (e.mode == 0) {
      for (size_t i = 0; i < e.shards.size(); ++i) {
        const int32_t rhs = shard_tensor(e.shards[i]);
        const Shape ext = extents(e.ranges[i]);
        const int32_t lhs = temp(ext);
        emit(PQW_T_SLICE, {tgt}, {lhs}, lows(e.ranges[i]));
        emit(PQW_T_CHECK, {lhs, rhs}, {}, {n_obl});
        n_obl += (int32_t)volume(ext);
      }
    } else {
      for (auto& g : groups(e)) {
        std::vector<int32_t> rhs;
        for (int32_t s : g.second) rhs.push_back(shard_tensor(s));
        const Shape ext = extents(g.first);
        const int32_t lhs = temp(ext);
        emit(PQW_T_SLICE, {tgt}, {lhs}, lows(g.first));
        std::vector<int32_t> ins{lhs};
        ins.insert(ins.end(), rhs.begin(), rhs.end());
        emit(PQW_T_CHECKSUM, ins, {}, {n_obl});
        n_obl += (int32_t)volume(ext);
      }
    }
    Program out;
    const size_t nts = soff.size() - 1;
    out.ir.reserve(4 + nts + sdims.size() + ops.size());
    out.ir = {IR_MAGIC, (int32_t)nts, n_ops, n_obl};
    for (size_t t = 0; t < nts; ++t) {
      out.ir.push_back((int32_t)(soff[t + 1] - soff[t]));
      for (int32_t i = soff[t]; i < soff[t + 1]; ++i) out.ir.push_back((int32_t)sdims[(size_t)i]);
    }
    out.ir.insert(out.ir.end(), ops.begin(), ops.end());
    out.consts = std::move(consts);
    out.var_keys = std::move(var_keys);
    return out;
  }
};

// A fresh Lowerer per stage (reusing one per thread, buffers kept, measured
// 7 % slower end to end: s3p).
Program lower_stage(const pqw_plan* p, int stage, uint64_t seed) {
  Lowerer lw;
  lw.p = p;
  lw.seed = seed;
  return lw.lower(p->stages[(size_t)stage]);
}

}  // namespace
}  // namespace pqw

using pqw::pfail;

extern "C" {

int pqw_plan_create(const pqw_graph_desc* logical, const pqw_graph_desc* parallel,
                    const pqw_lineage_desc* lineage, const int64_t* consts, size_t n_consts,
                    pqw_plan** out) {
  if (!logical || !parallel || !lineage || !out || (n_consts && !consts))
    return pfail(PQW_EINVAL, "null argument");
  auto* p = new pqw_plan();
  try {
    p->L.load(*logical);
    p->P.load(*parallel);
    p->consts.assign(consts, consts + 3 * n_consts);
    pqw::Col<std::string_view> lnames, snames;
    pqw::Col<char> ls, ss;
    pqw::split_names(lineage->logical_names, lineage->n_entries, ls, lnames);
    int64_t n_sh = 0;
    for (int64_t i = 0; i < lineage->n_entries; ++i) n_sh += lineage->n_shards[i];
    pqw::split_names(lineage->shard_names, n_sh, ss, snames);
    p->entry_of_logical.assign(p->L.nt(), -1);
    p->entries.resize((size_t)lineage->n_entries);
    int64_t k = 0, r = 0;
    for (int64_t i = 0; i < lineage->n_entries; ++i) {
      auto& e = p->entries[(size_t)i];
      e.logical = p->L.find(lnames[(size_t)i]);
      e.mode = lineage->mode[i];
      if (e.logical < 0 || e.mode > 1) p->lineage_ok = false;
      else p->entry_of_logical[e.logical] = (int32_t)i;
      for (int32_t j = 0; j < lineage->n_shards[i]; ++j, ++k) {
        const int32_t s = p->P.find(snames[(size_t)k]);
        if (s < 0) p->lineage_ok = false;
        e.shards.push_back(s);
        std::vector<std::pair<int64_t, int64_t>> rs;
        for (int32_t a = 0; a < lineage->shard_ndim[k]; ++a, ++r)
          rs.push_back({lineage->ranges[2 * r], lineage->ranges[2 * r + 1]});
        e.ranges.push_back(std::move(rs));
      }
    }
  } catch (const std::exception& ex) {
    delete p;
    return pfail(PQW_EINVAL, std::string("plan load: ") + ex.what());
  }
  *out = p;
  return PQW_OK;
}

void pqw_plan_destroy(pqw_plan* p) { delete p; }

int pqw_plan_validate(pqw_plan* p) {
  if (!p) return pfail(PQW_EINVAL, "null plan");
  std::string why;
  if (!pqw::validate_graph(p->L, why)) return pfail(PQW_EPLAN, "logical graph: " + why);
  if (!pqw::validate_graph(p->P, why)) return pfail(PQW_EPLAN, "parallel graph: " + why);
  p->validated = true;
  return PQW_OK;
}

int pqw_plan_check_lineage(pqw_plan* p, int64_t out[2]) {
  if (!p || !out) return pfail(PQW_EINVAL, "null argument");
  int64_t hard = 0, tiling = 0;
  for (const auto& e : p->entries) {
    if (e.logical < 0) {
      hard++;
      continue;
    }
    if (e.mode > 1) hard++;
    const auto shape = p->L.shape_vec(e.logical);
    for (size_t i = 0; i < e.shards.size(); ++i) {
      if (e.shards[i] < 0) {
        hard++;
        continue;
      }
      const auto ps = p->P.shape_vec(e.shards[i]);
      bool same = ps.size() == e.ranges[i].size();
      for (size_t a = 0; same && a < ps.size(); ++a)
        same = ps[a] == e.ranges[i][a].second - e.ranges[i][a].first;
      if (!same) hard++;
    }
    // graph.py entry_tiles_exactly: distinct boxes in bounds, disjoint, covering
    std::vector<const std::vector<std::pair<int64_t, int64_t>>*> boxes;
    for (const auto& r : e.ranges) {
      bool seen = false;
      for (auto* b : boxes) seen = seen || *b == r;
      if (!seen) boxes.push_back(&r);
    }
    bool ok = true;
    int64_t vol = 0, total = 1;
    for (int64_t d : shape) total *= d;
    for (auto* b : boxes) {
      if (b->size() != shape.size()) {
        ok = false;
        break;
      }
      int64_t v = 1;
      for (size_t a = 0; a < shape.size(); ++a) {
        const auto& [lo, hi] = (*b)[a];
        if (!(0 <= lo && lo < hi && hi <= shape[a])) ok = false;
        v *= hi - lo;
      }
      vol += v;
    }
    if (ok && vol != total) ok = false;
    for (size_t i = 0; ok && i < boxes.size(); ++i)
      for (size_t j = i + 1; ok && j < boxes.size(); ++j) {
        bool overlap = true;
        for (size_t a = 0; a < shape.size(); ++a)
          overlap = overlap && (*boxes[i])[a].first < (*boxes[j])[a].second &&
                    (*boxes[j])[a].first < (*boxes[i])[a].second;
        if (overlap) ok = false;
      }
    if (!ok) tiling++;
  }
  out[0] = hard;
  out[1] = tiling;
  return PQW_OK;
}

int pqw_plan_build_stages(pqw_plan* p, int64_t out[3]) {
  if (!p || !out) return pfail(PQW_EINVAL, "null argument");
  if (!p->L.resolved || !p->P.resolved || !p->lineage_ok || !p->L.unique_producers ||
      !p->P.unique_producers)
    return pfail(PQW_EPLAN, "lineage or producers not well formed");
  try {
    pqw::build(p);
  } catch (const std::exception& ex) {
    p->stages.clear();
    return pfail(PQW_EPLAN, std::string("build_stages: ") + ex.what());
  }
  p->built = true;
  out[0] = (int64_t)p->stages.size();
  out[1] = (int64_t)p->uncovered[0].size();
  out[2] = (int64_t)p->uncovered[1].size();
  return PQW_OK;
}

int pqw_plan_stage_target(pqw_plan* p, int stage) {
  if (!p || !p->built || stage < 0 || (size_t)stage >= p->stages.size())
    return pfail(PQW_EINVAL, "bad stage");
  return p->stages[(size_t)stage].target;
}

long pqw_plan_stage_nodes(pqw_plan* p, int stage, int side, int32_t* out, size_t cap) {
  if (!p || !p->built || stage < 0 || (size_t)stage >= p->stages.size())
    return pfail(PQW_EINVAL, "bad stage");
  const auto& st = p->stages[(size_t)stage];
  const auto& v = side == 0 ? st.lnodes : side == 1 ? st.pnodes : side == 2 ? st.l_inputs
                                                                              : st.p_inputs;
  if (out) std::memcpy(out, v.data(), std::min(cap, v.size()) * sizeof(int32_t));
  return (long)v.size();
}

long pqw_plan_uncovered(pqw_plan* p, int side, int32_t* out, size_t cap) {
  if (!p || !p->built) return pfail(PQW_ESTATE, "stages not built");
  const auto& v = p->uncovered[side ? 1 : 0];
  if (out) std::memcpy(out, v.data(), std::min(cap, v.size()) * sizeof(int32_t));
  return (long)v.size();
}

int pqw_plan_add_stages(pqw_plan* p, pqw_engine* e, uint64_t seed, const int32_t* stages, size_t n,
                        int32_t* out_index) {
  if (!p || !e || !out_index) return pfail(PQW_EINVAL, "null argument");
  if (!p->built) return pfail(PQW_ESTATE, "stages not built");
  std::vector<int32_t> list;
  if (stages) list.assign(stages, stages + n);
  else {
    n = p->stages.size();
    for (size_t i = 0; i < n; ++i) list.push_back((int32_t)i);
  }
  for (int32_t s : list)
    if (s < 0 || (size_t)s >= p->stages.size()) return pfail(PQW_EINVAL, "bad stage index");
  static const bool timing = getenv("PQW_TIMING") != nullptr;
  auto lap = [t = std::chrono::steady_clock::now()](const char* what) mutable {
    const auto now = std::chrono::steady_clock::now();
    if (timing)
      fprintf(stderr, "PQW_TIMING add_stages %s %.1f ms\n", what,
              std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  };
  // Lower every stage and hash its program on host threads; group equal
  // hashes in order (the representative: the engine's cached program, else
  // the batch's first); confirm equal texts on host threads; then queue in
  // order, passing the verified duplicate so the engine neither hashes nor
  // compares again. Only representatives' texts are kept.
  std::vector<pqw::Program> progs(n);
  std::vector<uint64_t> hash(n, 0);
  std::vector<char> bad(n, 0);
  std::atomic<uint64_t> t_lower{0}, t_hash{0}, words{0};
  pqw::parallel_for(n, [&](size_t i, unsigned) {
    try {
      const auto t0 = std::chrono::steady_clock::now();
      progs[i] = pqw::lower_stage(p, list[i], seed);
      const auto t1 = std::chrono::steady_clock::now();
      const auto& pg = progs[i];
      hash[i] = pqw::program_hash(pg.ir.data(), pg.ir.size(), pg.consts.data(),
                                  pg.consts.size() / 3, pg.var_keys.size());
      if (timing) {
        const auto t2 = std::chrono::steady_clock::now();
        t_lower += (uint64_t)std::chrono::duration_cast<std::chrono::microseconds>(t1 - t0).count();
        t_hash += (uint64_t)std::chrono::duration_cast<std::chrono::microseconds>(t2 - t1).count();
        words += pg.ir.size();
      }
    } catch (const std::exception&) {
      bad[i] = 1;
    }
  });
  if (timing)
    fprintf(stderr, "PQW_TIMING add_stages (thread-ms) lower %.1f hash %.1f; program words %llu\n",
            t_lower.load() / 1e3, t_hash.load() / 1e3, (unsigned long long)words.load());
  lap("lower+hash");
  // rep[i]: -1 none (first of its hash), >= 0 batch index, <= -2 engine stage -(s + 2)
  std::vector<int64_t> rep(n, -1);
  {
    std::unordered_map<uint64_t, int64_t> first;
    first.reserve(n);
    for (size_t i = 0; i < n; ++i) {
      if (bad[i]) continue;
      auto it = first.find(hash[i]);
      if (it != first.end()) {
        rep[i] = it->second;
        continue;
      }
      const std::vector<int32_t>* cir;
      const std::vector<int64_t>* cco;
      int st;
      if (pqw::cached_program(e, hash[i], &cir, &cco, &st)) {
        rep[i] = -(int64_t)st - 2;
        first.emplace(hash[i], rep[i]);
      } else {
        first.emplace(hash[i], (int64_t)i);
      }
    }
  }
  std::vector<char> same(n, 0);
  pqw::parallel_for(n, [&](size_t i, unsigned) {
    if (rep[i] == -1) return;
    const std::vector<int32_t>* rir;
    const std::vector<int64_t>* rco;
    if (rep[i] >= 0) {
      rir = &progs[(size_t)rep[i]].ir;
      rco = &progs[(size_t)rep[i]].consts;
    } else {
      int st;
      pqw::cached_program(e, hash[i], &rir, &rco, &st);
    }
    same[i] = *rir == progs[i].ir && *rco == progs[i].consts;
  });
  pqw::parallel_for(n, [&](size_t i, unsigned) {  // duplicates' texts are not needed
    if (same[i] && rep[i] != -1) {
      std::vector<int32_t>().swap(progs[i].ir);
      std::vector<int64_t>().swap(progs[i].consts);
    }
  });
  lap("dedup");
  std::vector<int> eidx(n, -1);
  int64_t status[16];
  for (size_t i = 0; i < n; ++i) {
    if (bad[i]) {
      out_index[i] = PQW_EPLAN;
      continue;
    }
    auto& pg = progs[i];
    int s_same = -1;
    if (same[i]) s_same = rep[i] >= 0 ? eidx[(size_t)rep[i]] : (int)(-rep[i] - 2);
    const int idx = pqw::stage_add_hashed(e, pg.ir.data(), pg.ir.size(), pg.consts.data(),
                                          pg.consts.size() / 3, pg.var_keys.data(),
                                          pg.var_keys.size(), hash[i], s_same, &pg.ir,
                                          &pg.consts, status);
    if (idx < 0) return idx;
    out_index[i] = idx;
    eidx[i] = idx;
  }
  lap("queue");
  return PQW_OK;
}

int pqw_plan_stage_program(pqw_plan* p, int stage, uint64_t seed, int32_t* ir, size_t ir_cap,
                           int64_t* consts, size_t consts_cap, uint64_t* var_keys, size_t vk_cap,
                           int64_t lens[3]) {
  if (!p || !lens) return pfail(PQW_EINVAL, "null argument");
  if (!p->built || stage < 0 || (size_t)stage >= p->stages.size())
    return pfail(PQW_EINVAL, "bad stage");
  pqw::Program pg;
  try {
    pg = pqw::lower_stage(p, stage, seed);
  } catch (const std::exception& ex) {
    return pfail(PQW_EPLAN, std::string("lower: ") + ex.what());
  }
  lens[0] = (int64_t)pg.ir.size();
  lens[1] = (int64_t)pg.consts.size() / 3;
  lens[2] = (int64_t)pg.var_keys.size();
  if (ir) std::memcpy(ir, pg.ir.data(), std::min(ir_cap, pg.ir.size()) * 4);
  if (consts) std::memcpy(consts, pg.consts.data(), std::min(consts_cap * 3, pg.consts.size()) * 8);
  if (var_keys)
    std::memcpy(var_keys, pg.var_keys.data(), std::min(vk_cap, pg.var_keys.size()) * 8);
  return PQW_OK;
}

}  // extern "C"

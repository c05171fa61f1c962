// schedule.cpp -- back end of the stage compiler: value DAG -> v4 program.
//
// 1. List scheduling. Units are taken in priority order (the depth-first order
//    of the obligation cones, which keeps the live set that of a sequential
//    evaluation) by NW simulated warps. The warp that frees up first takes the
//    highest-priority ready unit it can start now -- a unit whose operands a
//    different warp produced is penalised by the cross-warp latency -- and
//    bundles with it further ready units of the same kind (same op, function,
//    arity) from a bounded look-ahead window, up to `bmax`. Every bundle gets a
//    timestamp (start time, warp); every warp's stream is in timestamp order.
// 2. Slot allocation. A value lives from its defining bundle to its last
//    reading bundle; a slot is reused only by a bundle that starts strictly
//    after the previous occupant's last read. Linear scan chooses values to
//    keep in global memory when the shared file is too small ("spill
//    everywhere": the defining bundle writes a temporary that a SPILL bundle
//    stores right after it; every reading bundle is preceded by a FILL into a
//    temporary); then all intervals are coloured exactly.
// 3. Synchronisation. A bundle WAITs for the producer of every operand on
//    another warp (read after write) and for the readers of the previous
//    occupant of every slot it writes (write after read); waits implied by
//    earlier ones (vector clocks) are dropped. All waits point to bundles with
//    smaller timestamps, which makes the program deadlock-free. Producers
//    SIGNAL after exactly the bundles someone waits on.
#include "schedule.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <deque>
#include <memory>
#include <queue>
#include <set>
#include <stdexcept>
#include <thread>
#include <unordered_map>

namespace pqw {
namespace {

[[noreturn]] void fail(const char* m) { throw std::runtime_error(m); }

constexpr uint64_t INF = ~0ull;

// cost model (issue slots of one warp)
uint32_t op_cost(const DagUnit& u) {
  switch (u.op) {
    case I_DOT: return u.k == 1 ? 9 : 5 + 4 * u.k;
    case I_SUM: return u.k == 2 ? 8 : 4 + 3 * u.k;
    case I_SUB: return 9;
    case I_NEG: return 6;
    case I_HASH: return 30;
    case I_INV: return u.guarded ? 22 : 260;
    case I_VAR: return 36;
    case I_CONST: return 3;
    case I_CHK: return 7;
    case I_DEN: return 4;
    default: return 4;
  }
}
thread_local uint64_t g_bundle_base = 10;  // cost-model constant per bundle (dispatch + latency)
uint64_t bundle_cost(const DagUnit& h, size_t n) {
  return g_bundle_base + n * op_cost(h) + (h.op == I_INV && h.guarded ? 250 : 0);
}

// Set of unit ids in [0, n) as a bit vector: ordered iteration from any id
// by word scans (the list scheduler walks its ready sets in priority order).
struct IdSet {
  std::vector<uint64_t> w;
  uint32_t n = 0;
  explicit IdSet(uint32_t n_ = 0) : w((n_ + 63) / 64, 0), n(n_) {}
  void insert(uint32_t i) { w[i >> 6] |= 1ull << (i & 63); }
  void erase(uint32_t i) { w[i >> 6] &= ~(1ull << (i & 63)); }
  // first member >= i, or n
  uint32_t next(uint32_t i) const {
    if (i >= n) return n;
    size_t k = i >> 6;
    uint64_t m = w[k] & (~0ull << (i & 63));
    while (!m) {
      if (++k == w.size()) return n;
      m = w[k];
    }
    return (uint32_t)(k * 64 + __builtin_ctzll(m));
  }
};

struct Exec {             // one instruction bundle of a warp stream
  uint32_t warp;
  uint64_t ts;
  uint8_t kind;           // 0 main, 1 fill, 2 spill
  uint32_t main;          // main bundle index
  uint32_t seq = 0;       // position in the warp's stream
};

// Reader list of an interval: almost every interval has one to three readers
// (a fill temporary exactly one), so they live inline; longer lists spill to
// the heap. Tens of thousands of intervals per large program made the
// per-interval std::vector allocations a visible part of the back end.
struct Readers {
  static constexpr uint32_t INL = 3;
  uint32_t n = 0, cap = INL;
  uint32_t inl[INL];
  std::unique_ptr<uint32_t[]> heap;
  Readers() = default;
  Readers(std::initializer_list<uint32_t> l) {
    for (uint32_t x : l) push_back(x);
  }
  Readers(Readers&& o) noexcept : n(o.n), cap(o.cap), heap(std::move(o.heap)) {
    std::copy(o.inl, o.inl + INL, inl);
    o.n = 0;
    o.cap = INL;
  }
  Readers& operator=(Readers&& o) noexcept {
    n = o.n;
    cap = o.cap;
    heap = std::move(o.heap);
    std::copy(o.inl, o.inl + INL, inl);
    o.n = 0;
    o.cap = INL;
    return *this;
  }
  uint32_t* data() { return heap ? heap.get() : inl; }
  const uint32_t* data() const { return heap ? heap.get() : inl; }
  void push_back(uint32_t x) {
    if (n == cap) {
      std::unique_ptr<uint32_t[]> h(new uint32_t[2 * cap]);
      std::copy(data(), data() + n, h.get());
      heap = std::move(h);
      cap *= 2;
    }
    data()[n++] = x;
  }
  bool empty() const { return n == 0; }
  uint32_t size() const { return n; }
  uint32_t operator[](uint32_t i) const { return data()[i]; }
  const uint32_t* begin() const { return data(); }
  const uint32_t* end() const { return data() + n; }
};

struct Interval {
  uint64_t start, end;
  uint32_t writer;        // exec id
  Readers readers;        // exec ids
  uint32_t slot = 0;
};

// Exact colouring of intervals (a slot is free for `start` once its occupant's
// end < start). Returns the number of slots; fills slot and, per interval, the
// previous occupant of its slot (or -1). Among free slots a writer prefers one
// whose previous occupant was only touched by its own warp (`owner`: the warp
// of all of an interval's readers, or -1 when several), so the slot reuse needs
// no cross-warp write-after-read wait; the slot count is optimal either way.
uint32_t colour(std::vector<Interval>& iv, std::vector<int32_t>& prev,
                const std::vector<int32_t>& owner, const std::vector<uint32_t>& writer_warp,
                uint32_t NW) {
  std::vector<uint32_t> order(iv.size());
  for (uint32_t i = 0; i < iv.size(); ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
    return iv[a].start != iv[b].start ? iv[a].start < iv[b].start : a < b;
  });
  using E = std::pair<uint64_t, uint32_t>;  // (end, interval)
  std::priority_queue<E, std::vector<E>, std::greater<E>> busy;
  // free slots per owning warp (index NW: shared by several warps), in release
  // order: the own warp's list is used LIFO (no wait either way), the others
  // oldest-first (the longer ago a slot was released, the likelier its readers
  // are done and the wait is free)
  std::vector<std::deque<std::pair<uint64_t, uint32_t>>> free_s(NW + 1);
  std::vector<int32_t> last_of_slot;
  prev.assign(iv.size(), -1);
  uint32_t n = 0;
  for (uint32_t i : order) {
    while (!busy.empty() && busy.top().first < iv[i].start) {
      const uint32_t j = busy.top().second;
      busy.pop();
      free_s[owner[j] >= 0 ? (uint32_t)owner[j] : NW].push_back({iv[j].end, iv[j].slot});
    }
    const uint32_t w = writer_warp[i];
    uint32_t s = UINT32_MAX;
    if (!free_s[w].empty()) {
      s = free_s[w].back().second;
      free_s[w].pop_back();
    } else {
      int32_t best = -1;
      for (uint32_t k = 0; k <= NW; ++k)
        if (!free_s[k].empty() &&
            (best < 0 || free_s[k].front().first < free_s[best].front().first))
          best = (int32_t)k;
      if (best >= 0) {
        s = free_s[best].front().second;
        free_s[best].pop_front();
      }
    }
    if (s == UINT32_MAX) {
      s = n++;
      last_of_slot.push_back(-1);
    }
    iv[i].slot = s;
    prev[i] = last_of_slot[s];
    last_of_slot[s] = (int32_t)i;
    busy.push({iv[i].end, i});
  }
  return n;
}

}  // namespace

Program schedule_program(const Dag& dag, const SchedOptions& opt) {
  const auto& U = dag.units;
  const uint32_t N = (uint32_t)U.size();
  const uint32_t NW = opt.n_warps;
  if (NW < 1 || NW > 32) fail("n_warps must be in [1, 32]");
  const uint64_t X = opt.xlat;
  g_bundle_base = opt.bundle_base;

  // ---- producers / consumers ------------------------------------------------
  std::vector<uint32_t> pred_off(N + 1, 0), preds;
  std::vector<uint32_t> ncons(N, 0);
  {
    std::vector<uint32_t> tmp, stamp(N, UINT32_MAX);
    for (uint32_t u = 0; u < N; ++u) {
      const DagUnit& d = U[u];
      if ((uint64_t)d.arg0 + d.nargs > dag.pool.size()) fail("operand list out of range");
      tmp.clear();  // distinct operands (dedup by stamp, then sort the few left)
      for (uint32_t i = 0; i < d.nargs; ++i) {
        const uint32_t p = dag.pool[d.arg0 + i];
        if (p >= u) fail("operand defined after its use");
        if (stamp[p] != u) {
          stamp[p] = u;
          tmp.push_back(p);
        }
      }
      std::sort(tmp.begin(), tmp.end());
      for (uint32_t p : tmp) {
        if (!U[p].defines()) fail("operand is not a value");
        preds.push_back(p);
        ncons[p]++;
      }
      pred_off[u + 1] = (uint32_t)preds.size();
    }
  }
  std::vector<uint32_t> cons_off(N + 1, 0), cons(preds.size());
  for (uint32_t u = 0; u < N; ++u) cons_off[u + 1] = cons_off[u] + ncons[u];
  {
    std::vector<uint32_t> fillp(cons_off.begin(), cons_off.end() - 1);
    for (uint32_t u = 0; u < N; ++u)
      for (uint32_t i = pred_off[u]; i < pred_off[u + 1]; ++i) cons[fillp[preds[i]]++] = u;
  }

  // bundle classes: units of one class may share a bundle
  std::vector<uint32_t> cls(N);
  uint32_t n_cls = 0;
  {
    std::unordered_map<uint64_t, uint32_t> ids;
    for (uint32_t u = 0; u < N; ++u) {
      const DagUnit& d = U[u];
      const uint64_t key = (uint64_t)d.op | ((uint64_t)d.fn << 8) | ((uint64_t)d.k << 16) |
                           ((uint64_t)(d.op == I_INV && !d.guarded) << 40);
      auto it = ids.find(key);
      if (it == ids.end()) it = ids.emplace(key, n_cls++).first;
      cls[u] = it->second;
    }
  }

  // bottom level: the cost-model length of the longest path from a unit to
  // the end of the program (critical-path priority among eligible units)
  std::vector<uint64_t> blevel(N, 0);
  for (uint32_t u = N; u-- > 0;) {
    uint64_t m = 0;
    for (uint32_t i = cons_off[u]; i < cons_off[u + 1]; ++i) m = std::max(m, blevel[cons[i]]);
    blevel[u] = m + op_cost(U[u]);
  }

  // One scheduling attempt with look-ahead window o.window and bundle width
  // o.bmax; false if the value file cannot hold even its temporaries.
  static const uint32_t leaf_window =
      getenv("PQW_LEAF_WINDOW") ? (uint32_t)atoi(getenv("PQW_LEAF_WINDOW")) : 0;
  static const bool timing = getenv("PQW_TIMING") != nullptr && getenv("PQW_TIMING_BACKEND") != nullptr;
  auto try_once = [&](const SchedOptions& o, Program& prog) -> bool {
    auto tb0 = std::chrono::steady_clock::now();
    auto blap = [&](const char* what) {
      if (!timing || N < 10000) return;
      const auto t = std::chrono::steady_clock::now();
      fprintf(stderr, "PQW_TIMING back end %u units: %s %.1f ms\n", N, what,
              std::chrono::duration<double, std::milli>(t - tb0).count());
      tb0 = t;
    };
    // ---- 1. list scheduling -------------------------------------------------
    std::vector<uint64_t> fin(N, 0), F1(N, 0), F2(N, 0);
    std::vector<int32_t> wof(N, -1), W1(N, -1);
    std::vector<uint8_t> has2(N, 0), done(N, 0);
    std::vector<uint32_t> npred(N), bundle_of(N, 0);
    for (uint32_t u = 0; u < N; ++u) npred[u] = pred_off[u + 1] - pred_off[u];
    IdSet ready(N);
    std::vector<IdSet> ready_cls(n_cls, IdSet(N));  // the ready units of each class
    auto make_ready = [&](uint32_t u) {
      uint64_t f1 = 0;
      int32_t w1 = -1;
      for (uint32_t i = pred_off[u]; i < pred_off[u + 1]; ++i) {
        const uint32_t p = preds[i];
        if (w1 < 0 || fin[p] > f1) {
          f1 = fin[p];
          w1 = wof[p];
        }
      }
      uint64_t f2 = 0;
      bool h2 = false;
      for (uint32_t i = pred_off[u]; i < pred_off[u + 1]; ++i) {
        const uint32_t p = preds[i];
        if (wof[p] != w1) {
          f2 = std::max(f2, fin[p]);
          h2 = true;
        }
      }
      F1[u] = f1;
      W1[u] = w1;
      F2[u] = f2;
      has2[u] = h2;
      ready.insert(u);
      ready_cls[cls[u]].insert(u);
    };
    auto est = [&](uint32_t u, uint32_t w) -> uint64_t {
      if (W1[u] < 0) return 0;
      if ((int32_t)w == W1[u]) return has2[u] ? std::max(F1[u], F2[u] + X) : F1[u];
      return F1[u] + X;
    };
    for (uint32_t u = 0; u < N; ++u)
      if (npred[u] == 0) make_ready(u);

    struct Bundle {
      uint32_t warp;
      uint64_t start, finish;
      std::vector<uint32_t> units;
    };
    std::vector<Bundle> bundles;
    std::vector<uint64_t> T(NW, 0);
    uint32_t frontier = 0, n_done = 0;
    std::vector<uint32_t> cand;
    uint64_t makespan = 0;
    while (n_done < N) {
      uint32_t w = 0;
      for (uint32_t i = 1; i < std::min(NW, o.active_warps); ++i)
        if (T[i] < T[w]) w = i;
      const uint64_t t = T[w];
      // unit ids below lim are in the window (every ready unit is >= frontier)
      const uint32_t lim = (uint32_t)std::min<uint64_t>((uint64_t)frontier + o.window, N);
      uint32_t head = ready.next(frontier);
      uint64_t tnext = INF;
      for (; head < lim; head = ready.next(head + 1)) {
        const uint64_t e = est(head, w);
        if (e <= t) break;
        tnext = std::min(tnext, e);
      }
      if (head >= lim) {
        T[w] = tnext == INF ? t + 1 : std::max(t + 1, tnext);
        continue;
      }
      if (o.pick_scan) {
        // among the next few eligible units, the one on the longest remaining path
        uint32_t seen = 0;
        const uint32_t first = head;
        for (uint32_t j = ready.next(first + 1); j < lim && seen < o.pick_scan; j = ready.next(j + 1))
          if (est(j, w) <= t) {
            ++seen;
            if (blevel[j] > blevel[head]) head = j;
          }
      }
      const DagUnit& H = U[head];
      cand.clear();
      cand.push_back(head);
      if (!(H.op == I_INV && !H.guarded)) {
        const IdSet& rc = ready_cls[cls[head]];
        // leaves (VAR, CONST) are ready from the start: bundling them from the
        // whole window would load witness values long before their readers
        // and hold slots meanwhile; they join a bundle only from near the head
        uint32_t blim = lim;
        if ((H.op == I_VAR || H.op == I_CONST) && leaf_window)
          blim = (uint32_t)std::min<uint64_t>(lim, (uint64_t)head + leaf_window);
        for (uint32_t j = rc.next(frontier); j < blim && cand.size() < o.bmax; j = rc.next(j + 1))
          if (j != head && est(j, w) <= t) cand.push_back(j);
      }
      const uint64_t cost = bundle_cost(H, cand.size());
      const uint32_t bid = (uint32_t)bundles.size();
      bundles.push_back({w, t, t + cost, cand});
      for (uint32_t u : cand) {
        ready.erase(u);
        ready_cls[cls[u]].erase(u);
        done[u] = 1;
        fin[u] = t + cost;
        wof[u] = (int32_t)w;
        bundle_of[u] = bid;
        n_done++;
      }
      for (uint32_t u : cand)
        for (uint32_t i = cons_off[u]; i < cons_off[u + 1]; ++i)
          if (--npred[cons[i]] == 0) make_ready(cons[i]);
      T[w] = t + cost;
      makespan = std::max(makespan, T[w]);
      while (frontier < N && done[frontier]) frontier++;
    }
    const uint32_t NB = (uint32_t)bundles.size();
    std::vector<uint64_t> bts(NB);
    for (uint32_t b = 0; b < NB; ++b)
      bts[b] = ((bundles[b].start * NW) + bundles[b].warp) * 4 + 1;
    // a bundle's reads are over once it finishes: any bundle that starts at or
    // after that time (timestamp > rend) may overwrite what it read
    auto rend = [&](uint32_t b) -> uint64_t { return bundles[b].finish * NW * 4; };

    // value intervals in timestamp space
    std::vector<uint64_t> vdef(N, 0), vend(N, 0);
    std::vector<uint32_t> values;
    for (uint32_t u = 0; u < N; ++u) {
      if (!U[u].defines()) continue;
      values.push_back(u);
      vdef[u] = bts[bundle_of[u]];
      uint64_t e = rend(bundle_of[u]);
      for (uint32_t i = cons_off[u]; i < cons_off[u + 1]; ++i)
        e = std::max(e, rend(bundle_of[cons[i]]));
      vend[u] = e;
    }
    std::sort(values.begin(), values.end(), [&](uint32_t a, uint32_t b) {
      return vdef[a] != vdef[b] ? vdef[a] < vdef[b] : a < b;
    });

    blap("list scheduling");
    // ---- 2. allocation: choose spills, then colour exactly -------------------
    const uint32_t K = o.smem_slots;
    // the distinct bundles reading each value (CSR)
    std::vector<uint32_t> rdb_off(N + 1, 0), rdb;
    {
      std::vector<uint32_t> rd, seen(bundles.size(), UINT32_MAX);
      for (uint32_t u = 0; u < N; ++u) {
        rd.clear();
        for (uint32_t i = cons_off[u]; i < cons_off[u + 1]; ++i) {
          const uint32_t b = bundle_of[cons[i]];
          if (seen[b] != u) {
            seen[b] = u;
            rd.push_back(b);
          }
        }
        std::sort(rd.begin(), rd.end());
        rdb.insert(rdb.end(), rd.begin(), rd.end());
        rdb_off[u + 1] = (uint32_t)rdb.size();
      }
    }
    // A spilled CONST is rematerialised instead of going through global memory:
    // its residue is written into a temporary before every reading bundle, it
    // is never stored, and its defining bundle drops it. (Rematerialising
    // spilled VARs the same way -- key load plus hash per reader -- measured
    // slower than filling them: the keys miss the L1 the value file leaves.)
    const bool remat_var = getenv("PQW_REMAT_VAR") != nullptr;
    auto remat_ok = [&](uint32_t v) {
      return U[v].op == I_CONST || (remat_var && U[v].op == I_VAR);
    };
    // slots the exact colouring below will need for a spill choice: the most
    // shared-memory intervals alive at once (a slot frees strictly after its
    // interval's end), without building the intervals themselves. Every
    // interval endpoint is 4 Z + r, r in {0, 1}, with Z a bundle's start
    // (start * NW + warp) or finish (finish * NW) key; numbering the distinct
    // Z keeps the order, so a difference array over 2 * |Z| points replaces
    // sorting the endpoints (same count: an interval [a, b] covers a..b).
    std::vector<uint64_t> zkey;
    zkey.reserve(2 * NB);
    for (uint32_t b = 0; b < NB; ++b) {
      zkey.push_back(bundles[b].start * NW + bundles[b].warp);
      zkey.push_back(bundles[b].finish * NW);
    }
    std::sort(zkey.begin(), zkey.end());
    zkey.erase(std::unique(zkey.begin(), zkey.end()), zkey.end());
    auto zrank = [&](uint64_t z) {
      return (uint32_t)(std::lower_bound(zkey.begin(), zkey.end(), z) - zkey.begin());
    };
    std::vector<uint32_t> p_start(NB), p_fin(NB);  // point index of bts(b) - 1 and of rend(b)
    for (uint32_t b = 0; b < NB; ++b) {
      p_start[b] = 2 * zrank(bundles[b].start * NW + bundles[b].warp);
      p_fin[b] = 2 * zrank(bundles[b].finish * NW);
    }
    std::vector<uint32_t> p_vend(N, 0);  // point of vend: the latest reader's rend
    for (uint32_t v : values) {
      uint32_t best = p_fin[bundle_of[v]];
      for (uint32_t i = cons_off[v]; i < cons_off[v + 1]; ++i) best = std::max(best, p_fin[bundle_of[cons[i]]]);
      p_vend[v] = best;
    }
    std::vector<int32_t> cover(2 * zkey.size() + 2);
    auto slots_needed = [&](const std::vector<uint8_t>& spilled) -> uint32_t {
      std::fill(cover.begin(), cover.end(), 0);
      auto add = [&](uint32_t a, uint32_t b) {  // points a..b
        cover[a]++;
        cover[b + 1]--;
      };
      for (uint32_t v : values) {
        const uint32_t bdef = bundle_of[v];
        if (!spilled[v]) {
          add(p_start[bdef] + 1, p_vend[v]);  // [vdef, vend]
        } else {
          if (!remat_ok(v)) add(p_start[bdef] + 1, p_fin[bdef] + 1);  // [vdef, rend(bdef) + 1]
          for (uint32_t i = rdb_off[v]; i < rdb_off[v + 1]; ++i)
            add(p_start[rdb[i]], p_fin[rdb[i]]);  // [bts - 1, rend]
        }
      }
      int32_t live = 0, most = 0;
      for (int32_t c : cover) {
        live += c;
        most = std::max(most, live);
      }
      return (uint32_t)most;
    };
    // spill choice for `keff` resident values: sweep in definition order
    // keeping at most keff values resident; when full, the resident value (or
    // the new one) that ends last is spilled. Two heaps over (end, value) with
    // lazy deletion: the earliest end expires, the latest end is evicted.
    // default: evict the value whose live length per squared read count is
    // largest (rarely read, long-lived values go to global memory first);
    // PQW_SPILL_MODE=0 restores the latest-ending rule (fewest spilled values)
    static const int spill_mode = getenv("PQW_SPILL_MODE") ? atoi(getenv("PQW_SPILL_MODE")) : 3;
    auto evict_key = [&](uint32_t v) -> uint64_t {
      if (spill_mode == 0) return vend[v];
      const uint64_t reads = rdb_off[v + 1] - rdb_off[v];
      if (spill_mode == 1) return (vend[v] - vdef[v]) / (reads + 1);
      if (spill_mode == 3) return (vend[v] - vdef[v]) / ((reads + 1) * (reads + 1));
      if (spill_mode == 4) return (vend[v] - vdef[v]) * 4 / (reads + 4);
      return vend[v] / (reads + 1);
    };
    auto select = [&](uint32_t keff, std::vector<uint8_t>& spilled) {
      spilled.assign(N, 0);
      using E = std::pair<uint64_t, uint32_t>;
      std::priority_queue<E, std::vector<E>, std::greater<E>> by_first;
      std::priority_queue<E> by_last;
      std::vector<uint8_t> gone(N, 0);  // expired or evicted
      uint32_t n_active = 0;
      for (uint32_t v : values) {
        while (!by_first.empty() && by_first.top().first < vdef[v]) {
          const uint32_t x = by_first.top().second;
          by_first.pop();
          if (!gone[x]) {
            gone[x] = 1;
            n_active--;
          }
        }
        while (!by_last.empty() && gone[by_last.top().second]) by_last.pop();
        if (n_active < keff) {
          by_first.push({vend[v], v});
          by_last.push({evict_key(v), v});
          n_active++;
        } else if (by_last.top().first > evict_key(v)) {
          const uint32_t x = by_last.top().second;
          by_last.pop();
          gone[x] = 1;
          spilled[x] = 1;
          by_first.push({vend[v], v});
          by_last.push({evict_key(v), v});
        } else {
          spilled[v] = 1;
        }
      }
    };
    // the reserve for FILL/SPILL temporaries grows until the spill choice for
    // K - reserve resident values fits the value file with its temporaries
    uint32_t overshoot = 0, tries = 0, last_fail = 0, prev_n = 0;
    for (uint32_t reserve = 0;; ++tries) {
      std::vector<uint8_t> spilled;
      select(K - reserve, spilled);
      uint32_t n_sm = slots_needed(spilled);
      if (n_sm > K) {  // more temporaries than the reserve: spill more
        overshoot = n_sm - K;
        if (reserve + 1 >= K) break;  // give up on this schedule: re-schedule narrower
        // past half the value file, a step that won back less than the
        // remaining overshoot means the temporaries of this schedule's bundles
        // alone nearly fill it: give up early as well
        if (tries >= 2 && reserve > K / 2 && (uint64_t)n_sm + overshoot > prev_n) break;
        prev_n = n_sm;
        // step by the overshoot (each step spills about what the last one
        // overshot; the slot count is not monotone in the reserve, so small
        // steps land closer to the least reserve that fits); double after a
        // few steps to bound the search
        const uint32_t step = 2 * overshoot + 16;
        last_fail = reserve;
        reserve = std::min(K - 1, tries < 4 ? reserve + step : std::max(reserve * 2, reserve + step));
        continue;
      }
      // a step can overshoot the least reserve that fits by far (every
      // reserved slot is a value spilled); bisect back towards the last
      // failing reserve while the value file is left well under-used
      if (tries > 0) {
        std::vector<uint8_t> cand;
        for (int r = 0; r < 2 && reserve - last_fail > 32 && K - n_sm > 32; ++r) {
          const uint32_t mid = last_fail + (reserve - last_fail) / 2;
          select(K - mid, cand);
          const uint32_t n = slots_needed(cand);
          if (n <= K) {
            reserve = mid;
            n_sm = n;
            spilled.swap(cand);
          } else {
            last_fail = mid;
          }
        }
      }
      if (timing && N >= 10000) fprintf(stderr, "PQW_TIMING back end %u units: reserve search %u tries\n", N, tries + 1);
      blap("reserve search");
      // exec bundles: [FILL] main [SPILL] per main bundle
      std::vector<Exec> ex;
      std::vector<int32_t> fill_of(NB, -1), spill_of(NB, -1), main_exec(NB, -1);
      std::vector<uint8_t> needs_fill(NB, 0), needs_spill(NB, 0);
      for (uint32_t v : values) {
        if (!spilled[v]) continue;
        if (!remat_ok(v)) needs_spill[bundle_of[v]] = 1;
        for (uint32_t i = cons_off[v]; i < cons_off[v + 1]; ++i) needs_fill[bundle_of[cons[i]]] = 1;
      }
      for (uint32_t b = 0; b < NB; ++b) {
        if (needs_fill[b]) {
          fill_of[b] = (int32_t)ex.size();
          ex.push_back({bundles[b].warp, bts[b] - 1, 1, b});
        }
        main_exec[b] = (int32_t)ex.size();
        ex.push_back({bundles[b].warp, bts[b], 0, b});
        if (needs_spill[b]) {
          spill_of[b] = (int32_t)ex.size();
          ex.push_back({bundles[b].warp, bts[b] + 1, 2, b});
        }
      }
      // intervals
      std::vector<Interval> sm, gm;
      std::vector<uint32_t> v_iv(N, ~0u), v_giv(N, ~0u);
      std::unordered_map<uint64_t, uint32_t> fill_iv;  // (bundle << 32 | value) -> interval
      for (uint32_t v : values) {
        const uint32_t bdef = bundle_of[v];
        const uint32_t* rd0 = rdb.data() + rdb_off[v];
        const uint32_t* rd1 = rdb.data() + rdb_off[v + 1];
        if (!spilled[v]) {
          Interval I{vdef[v], vend[v], (uint32_t)main_exec[bdef], {}};
          for (const uint32_t* b = rd0; b != rd1; ++b) I.readers.push_back((uint32_t)main_exec[*b]);
          v_iv[v] = (uint32_t)sm.size();
          sm.push_back(std::move(I));
        } else if (remat_ok(v)) {
          for (const uint32_t* pb = rd0; pb != rd1; ++pb) {
            const uint32_t b = *pb;
            Interval Fi{bts[b] - 1, rend(b), (uint32_t)fill_of[b], {(uint32_t)main_exec[b]}};
            fill_iv[((uint64_t)b << 32) | v] = (uint32_t)sm.size();
            sm.push_back(std::move(Fi));
          }
        } else {
          Interval T1{vdef[v], rend(bdef) + 1, (uint32_t)main_exec[bdef], {(uint32_t)spill_of[bdef]}};
          v_iv[v] = (uint32_t)sm.size();
          sm.push_back(std::move(T1));
          Interval G{vdef[v] + 1, rend(bdef) + 1, (uint32_t)spill_of[bdef], {}};
          for (const uint32_t* pb = rd0; pb != rd1; ++pb) {
            const uint32_t b = *pb;
            G.end = std::max(G.end, bts[b]);
            G.readers.push_back((uint32_t)fill_of[b]);
            Interval Fi{bts[b] - 1, rend(b), (uint32_t)fill_of[b], {(uint32_t)main_exec[b]}};
            fill_iv[((uint64_t)b << 32) | v] = (uint32_t)sm.size();
            sm.push_back(std::move(Fi));
          }
          v_giv[v] = (uint32_t)gm.size();
          gm.push_back(std::move(G));
        }
      }
      std::vector<int32_t> sprev, gprev;
      auto owners = [&](const std::vector<Interval>& iv, std::vector<int32_t>& own,
                        std::vector<uint32_t>& wr) {
        own.assign(iv.size(), -1);
        wr.resize(iv.size());
        for (uint32_t i = 0; i < iv.size(); ++i) {
          wr[i] = ex[iv[i].writer].warp;
          int32_t o = (int32_t)ex[iv[i].writer].warp;  // no readers: the writer's warp
          if (!iv[i].readers.empty()) {
            o = (int32_t)ex[iv[i].readers[0]].warp;
            for (uint32_t r : iv[i].readers)
              if ((int32_t)ex[r].warp != o) o = -1;
          }
          own[i] = o < 0 ? -1 : o;
        }
      };
      std::vector<int32_t> s_own, g_own;
      std::vector<uint32_t> s_wr, g_wr;
      owners(sm, s_own, s_wr);
      n_sm = colour(sm, sprev, s_own, s_wr, NW);
      if (n_sm > K) fail("internal: colouring needs more slots than the interval count");
      owners(gm, g_own, g_wr);
      const uint32_t n_gm = colour(gm, gprev, g_own, g_wr, NW);
      blap("intervals + colouring");
      if (getenv("PQW_DEBUG_QUAD")) {
        // slot-time of shared intervals whose writer and readers share a quadrant
        uint64_t tot = 0, loc = 0, nloc = 0, same_warp = 0;
        for (const auto& I : sm) {
          const uint64_t len = I.end - I.start;
          tot += len;
          const uint32_t q = ex[I.writer].warp % 4;
          bool l = true, sw = true;
          for (uint32_t r : I.readers) {
            l = l && ex[r].warp % 4 == q;
            sw = sw && ex[r].warp == ex[I.writer].warp;
          }
          if (l) { loc += len; nloc++; }
          if (sw) same_warp += len;
        }
        uint64_t by_op[I_NUM_OPS] = {};
        for (const auto& I : sm) {
          const auto& E = ex[I.writer];
          const uint32_t op = E.kind == 0 ? U[bundles[E.main].units[0]].op : (E.kind == 1 ? I_FILL : I_SPILL);
          by_op[op] += I.end - I.start;
        }
        fprintf(stderr, "QUADDBG intervals=%zu slots=%u quad-local slot-time %.1f%% (n=%llu) same-warp %.1f%% | by def op:",
                sm.size(), n_sm, 100.0 * loc / std::max<uint64_t>(tot, 1), (unsigned long long)nloc,
                100.0 * same_warp / std::max<uint64_t>(tot, 1));
        for (int i = 0; i < I_NUM_OPS; ++i)
          if (by_op[i]) fprintf(stderr, " op%d=%.1f%%", i, 100.0 * by_op[i] / std::max<uint64_t>(tot, 1));
        fprintf(stderr, "\n");
        uint64_t sv = 0, sv_loc = 0, fl = 0, fl_loc = 0;
        for (uint32_t v : values) {
          if (!spilled[v] || remat_ok(v)) continue;
          const uint32_t q = bundles[bundle_of[v]].warp % 4;
          bool l = true;
          uint64_t nr = 0;
          for (uint32_t i = rdb_off[v]; i < rdb_off[v + 1]; ++i, ++nr) l = l && bundles[rdb[i]].warp % 4 == q;
          sv++; fl += nr;
          if (l) { sv_loc++; fl_loc += nr; }
        }
        fprintf(stderr, "TMEMDBG spilled=%llu local=%llu fills=%llu local_fills=%llu gm_slots=%u\n",
                (unsigned long long)sv, (unsigned long long)sv_loc, (unsigned long long)fl,
                (unsigned long long)fl_loc, n_gm);
      }

      blap("allocation");
      // ---- 3. synchronisation -------------------------------------------------
      const uint32_t NE = (uint32_t)ex.size();
      std::vector<std::vector<uint32_t>> stream(NW);
      {
        std::vector<uint32_t> order(NE);
        for (uint32_t i = 0; i < NE; ++i) order[i] = i;
        std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return ex[a].ts < ex[b].ts; });
        for (uint32_t e : order) {
          ex[e].seq = (uint32_t)stream[ex[e].warp].size();
          stream[ex[e].warp].push_back(e);
        }
      }
      // requirements per exec: (warp, count) with count = producer seq + 1
      std::vector<std::vector<std::pair<uint32_t, uint32_t>>> req(NE);
      auto need = [&](uint32_t e, uint32_t producer) {
        if (ex[producer].warp == ex[e].warp) return;
        req[e].push_back({ex[producer].warp, ex[producer].seq + 1});
      };
      for (uint32_t v : values) {
        const uint32_t bdef = bundle_of[v];
        if (!spilled[v]) {
          for (uint32_t r : sm[v_iv[v]].readers) need(r, (uint32_t)main_exec[bdef]);
        } else if (!remat_ok(v)) {
          for (uint32_t r : gm[v_giv[v]].readers) need(r, (uint32_t)spill_of[bdef]);
        }
      }
      auto war = [&](std::vector<Interval>& iv, const std::vector<int32_t>& prv) {
        for (uint32_t i = 0; i < iv.size(); ++i) {
          if (prv[i] < 0) continue;
          const Interval& P = iv[prv[i]];
          if (P.readers.empty()) need(iv[i].writer, P.writer);
          for (uint32_t r : P.readers) need(iv[i].writer, r);
        }
      };
      war(sm, sprev);
      war(gm, gprev);
      // vector clocks in timestamp order
      std::vector<uint32_t> snap((size_t)NE * NW, 0);
      std::vector<std::vector<uint32_t>> vc(NW, std::vector<uint32_t>(NW, 0));
      std::vector<std::vector<std::pair<uint32_t, uint32_t>>> waits(NE);
      std::vector<uint8_t> signal_after(NE, 0);
      {
        std::vector<uint32_t> order(NE);
        for (uint32_t i = 0; i < NE; ++i) order[i] = i;
        std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return ex[a].ts < ex[b].ts; });
        for (uint32_t e : order) {
          const uint32_t w = ex[e].warp;
          auto& rq = req[e];
          std::sort(rq.begin(), rq.end(), [](auto& a, auto& b) {
            return a.first != b.first ? a.first < b.first : a.second > b.second;
          });
          for (size_t i = 0; i < rq.size(); ++i) {
            if (i && rq[i].first == rq[i - 1].first) continue;  // max count per warp first
            const uint32_t pw = rq[i].first, c = rq[i].second;
            if (vc[w][pw] >= c) continue;
            waits[e].push_back({pw, c});
            const uint32_t pe = stream[pw][c - 1];
            signal_after[pe] = 1;
            const uint32_t* s = &snap[(size_t)pe * NW];
            for (uint32_t j = 0; j < NW; ++j) vc[w][j] = std::max(vc[w][j], s[j]);
            vc[w][pw] = std::max(vc[w][pw], c);
          }
          vc[w][w] = ex[e].seq + 1;
          std::copy(vc[w].begin(), vc[w].end(), &snap[(size_t)e * NW]);
        }
      }

      blap("synchronisation");
      // ---- 4. emission ------------------------------------------------------------
      prog = Program{};
      auto& code = prog.code;
      const uint32_t table = (NW + 3) / 4;
      code.assign(table, pqw_ins{0, 0, 0, 0});
      std::vector<uint32_t> fields;
      auto put_bundle = [&](uint32_t op, uint32_t fn, uint32_t k, uint32_t n, uint32_t aux,
                            const std::vector<uint32_t>& f, uint32_t nf) {
        // f: nf fields per op, op-major (f[i * nf + j])
        code.push_back(pqw_ins{isa_header(op, fn, k), n, aux, 0});
        // the last group is padded with copies of the bundle's last op (a
        // repeated op rewrites the same value, a repeated check re-checks), so
        // the device runs whole groups without per-op predicates; INV (whose
        // destinations hold running products) is the one op that counts
        for (uint32_t g = 0; g < n; g += GROUP)
          for (uint32_t j = 0; j < nf; ++j) {
            uint32_t v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (uint32_t i = 0; i < GROUP; ++i) {
              const uint32_t src = g + i < n ? g + i : n - 1;
              if (g + i < n || op != I_INV) v[i] = f[(size_t)src * nf + j];
            }
            code.push_back(pqw_ins{v[0], v[1], v[2], v[3]});
            code.push_back(pqw_ins{v[4], v[5], v[6], v[7]});
          }
        prog.op_hist[op] += n;
      };
      auto soff = [&](uint32_t iv) { return sm[iv].slot * SLOT_BYTES; };
      for (uint32_t w = 0; w < NW; ++w) {
        reinterpret_cast<uint32_t*>(code.data())[w] = (uint32_t)code.size();
        for (uint32_t e : stream[w]) {
          const Exec& E = ex[e];
          // all but the last wait become WAIT instructions, three per instruction;
          // the last one rides in the bundle header: each (warp + 1) << 24 | count
          const size_t nwait = waits[e].size();
          auto enc = [](const std::pair<uint32_t, uint32_t>& wt) -> uint32_t {
            if (wt.second >= (1u << 24)) fail("stream too long for a folded wait");
            return ((wt.first + 1) << 24) | wt.second;
          };
          // the second-to-last wait also rides in the header (y >> 13) when its
          // count fits 13 bits (and the bundle's n fits the low 13)
          const bool fold2 = nwait >= 2 && waits[e][nwait - 2].second < (1u << 13);
          const size_t n_instr_waits = nwait - (nwait ? 1 : 0) - (fold2 ? 1 : 0);
          for (size_t i = 0; i < n_instr_waits; i += 3) {
            const uint32_t second = i + 1 < n_instr_waits ? enc(waits[e][i + 1]) : 0u;
            const uint32_t third = i + 2 < n_instr_waits ? enc(waits[e][i + 2]) : 0u;
            code.push_back(pqw_ins{isa_header(I_WAIT, 0, 0), third, enc(waits[e][i]), second});
            prog.op_hist[I_WAIT]++;
          }
          prog.n_waits += (uint32_t)nwait;
          const size_t hdr = code.size();  // header of this exec's (first) instruction
          size_t last_hdr = hdr;            // header that publishes the exec's progress
          const auto& B = bundles[E.main];
          if (E.kind == 1 || E.kind == 2) {
            fields.clear();
            uint32_t n = 0;
            if (E.kind == 1) {
              // global fills, then rematerialised VARs, then CONSTs (one exec:
              // the wait rides on the first header, the signal on the last)
              std::vector<uint32_t> seen, fvar, fcst;
              uint32_t nv = 0, nc = 0;
              for (uint32_t u : B.units)
                for (uint32_t a = 0; a < U[u].nargs; ++a) {
                  const uint32_t v = dag.pool[U[u].arg0 + a];
                  if (!spilled[v] || std::find(seen.begin(), seen.end(), v) != seen.end()) continue;
                  seen.push_back(v);
                  const uint32_t dst = soff(fill_iv.at(((uint64_t)E.main << 32) | v));
                  if (U[v].op == I_VAR && remat_ok(v)) {
                    fvar.push_back(dst);
                    fvar.push_back(U[v].aux);
                    nv++;
                  } else if (U[v].op == I_CONST && remat_ok(v)) {
                    fcst.push_back(dst);
                    fcst.push_back(U[v].aux);
                    nc++;
                  } else {
                    fields.push_back(dst);
                    fields.push_back(gm[v_giv[v]].slot * SLOT_BYTES);
                    n++;
                  }
                }
              if (n) {
                last_hdr = code.size();
                put_bundle(I_FILL, 0, 0, n, 0, fields, 2);
              }
              if (nv) {
                last_hdr = code.size();
                put_bundle(I_VAR, 0, 0, nv, 0, fvar, 2);
                prog.n_remat += nv;
              }
              if (nc) {
                last_hdr = code.size();
                put_bundle(I_CONST, 0, 0, nc, 0, fcst, 2);
                prog.n_remat += nc;
              }
            } else {
              for (uint32_t u : B.units)
                if (U[u].defines() && spilled[u] && !remat_ok(u)) {
                  fields.push_back(gm[v_giv[u]].slot * SLOT_BYTES);
                  fields.push_back(soff(v_iv[u]));
                  n++;
                }
              put_bundle(I_SPILL, 0, 0, n, 0, fields, 2);
            }
          } else {
            const DagUnit& H = U[B.units[0]];
            auto opnd = [&](uint32_t v) -> uint32_t {
              if (!spilled[v]) return soff(v_iv[v]);
              return soff(fill_iv.at(((uint64_t)E.main << 32) | v));
            };
            fields.clear();
            uint32_t nf = isa_fields(H.op, H.k);
            for (uint32_t u : B.units) {
              const DagUnit& d = U[u];
              const uint32_t* a = &dag.pool[d.arg0];
              switch (d.op) {
                case I_CHK:
                  fields.push_back(d.aux);
                  fields.push_back(opnd(a[0]));
                  fields.push_back(opnd(a[1]));
                  break;
                case I_DEN:
                  fields.push_back(opnd(a[0]));
                  break;
                case I_VAR:
                case I_CONST:
                  if (spilled[u] && remat_ok(u)) break;  // rematerialised at every reader
                  fields.push_back(soff(v_iv[u]));
                  fields.push_back(d.aux);
                  break;
                default:
                  fields.push_back(soff(v_iv[u]));
                  for (uint32_t i = 0; i < d.nargs; ++i) fields.push_back(opnd(a[i]));
              }
              if (fields.size() % nf) fail("internal: operand count does not match the op");
              // field ops per witness
              switch (d.op) {
                case I_DOT: prog.cls[0] += d.k; prog.cls[1] += d.k - 1; break;
                case I_SUM: prog.cls[1] += d.k - 1; break;
                case I_SUB: case I_NEG: prog.cls[1] += 1; break;
                case I_HASH: case I_VAR: prog.cls[2] += 1; break;  // remat copies not counted
                case I_CHK: case I_DEN: prog.cls[4] += 1; break;
                default: break;
              }
            }
            if (H.op == I_INV) {
              const uint64_t n = B.units.size();
              if (n > 1 && !H.guarded) fail("internal: unguarded inversions bundled");
              prog.cls[0] += 3 * (n - 1);
              prog.cls[3] += 1;
            }
            put_bundle(H.op, H.fn, H.k, (uint32_t)(fields.size() / nf), 0, fields, nf);
          }
          if (nwait) {
            const auto& pr = waits[e][nwait - 1];
            if (pr.second >= (1u << 24)) fail("stream too long for a folded wait");
            code[hdr].a = ((pr.first + 1) << 24) | pr.second;
          }
          if (fold2) {
            const auto& pr = waits[e][nwait - 2];
            if (code[hdr].dst < (1u << 13)) {
              code[hdr].dst |= (((pr.first + 1) << 13) | pr.second) << 13;
            } else {  // n too large to share the word: a WAIT instruction after all
              code.insert(code.begin() + (ptrdiff_t)hdr,
                          pqw_ins{isa_header(I_WAIT, 0, 0), 0, enc(pr), 0});
              prog.op_hist[I_WAIT]++;
              ++last_hdr;
            }
          }
          if (signal_after[e]) {
            code[last_hdr].b = E.seq + 1;  // header.w: publish progress after this exec
            prog.op_hist[I_SIGNAL]++;
          }
        }
        code.push_back(pqw_ins{I_END, 0, 0, 0});
      }
      blap("emission");
      prog.n_slots = n_sm;
      prog.n_spill = n_gm;
      prog.n_bundles = NB;
      prog.makespan = makespan;
      for (uint32_t v : values) prog.n_spilled_values += spilled[v];
      if (getenv("PQW_DEBUG_SPILL")) {
        uint64_t by[I_NUM_OPS] = {}, fills[I_NUM_OPS] = {};
        for (uint32_t v : values)
          if (spilled[v]) {
            by[U[v].op]++;
            fills[U[v].op] += rdb_off[v + 1] - rdb_off[v];
          }
        uint64_t var_vals = 0, var_reads = 0;
        for (uint32_t v : values)
          if (U[v].op == I_VAR) {
            var_vals++;
            var_reads += rdb_off[v + 1] - rdb_off[v];
          }
        fprintf(stderr, "SPILLDBG values=%zu vars=%llu var-reading-bundles=%llu bundles=%u spilled:", values.size(),
                (unsigned long long)var_vals, (unsigned long long)var_reads, NB);
        for (int i = 0; i < I_NUM_OPS; ++i)
          if (by[i]) fprintf(stderr, " op%d=%llu(fills %llu)", i, (unsigned long long)by[i], (unsigned long long)fills[i]);
        fprintf(stderr, "\n");
      }
      return true;
    }
    return false;
  };

  // A wide look-ahead window exposes the most parallelism (and the widest
  // bundles) but holds more values live; narrower windows trade parallelism
  // for fewer spills. Take the best modelled time: makespan plus the
  // FILL/SPILL traffic spread over the warps.
  std::vector<uint32_t> windows;
  if (opt.window) {
    windows.push_back(opt.window);
  } else {
    for (uint32_t w : {N + 1, 4096u, 1024u, 384u, 64u, 8u, 1u})
      if (windows.empty() || w < windows.back()) windows.push_back(std::max<uint32_t>(w, 1));
  }
  Program best;
  bool have = false;
  uint64_t best_score = INF;
  auto attempt = [&](uint32_t win, Program& cand) -> bool {
    g_bundle_base = opt.bundle_base;  // thread_local: attempts may run on worker threads
    SchedOptions o = opt;
    o.window = win;
    for (uint32_t bm = opt.bmax;; bm /= 2) {
      o.bmax = std::max<uint32_t>(bm, 1);
      if (try_once(o, cand)) return true;
      if (bm <= 1) return false;
    }
  };
  auto consider = [&](Program& cand) {
    const uint64_t traffic = cand.op_hist[I_FILL] + cand.op_hist[I_SPILL];
    const uint64_t score = cand.makespan + traffic * opt.spill_cost / NW;
    if (score < best_score) {
      best_score = score;
      best = std::move(cand);
      have = true;
    }
  };
  // the widest window first; only when it spills are the narrower ones tried
  // The widest window wins the cost comparison on every program of the
  // BASELINE workloads (its extra spills cost less than the parallelism the
  // narrower windows give up, confirmed on the GPU), so narrower windows are
  // tried only when it does not fit the value file at all.
  for (uint32_t win : windows) {
    if (have) break;
    Program cand;
    if (attempt(win, cand)) consider(cand);
  }
  if (!have) {
    // last resort: one warp, one op per bundle (a sequential evaluation)
    SchedOptions o = opt;
    o.window = 1;
    o.bmax = 1;
    o.active_warps = 1;
    if (!try_once(o, best)) fail("stage does not fit the shared value file");
  }
  return best;
}

}  // namespace pqw

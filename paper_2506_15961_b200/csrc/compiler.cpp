// compiler.cpp -- stage compiler: tensor-op program -> straight-line F_p bytecode.
//
// What the reference does per stage with hash-consed symbolic expressions
// (pkg/src/planeq/ops.py:66-77 generic execute, ops.py:923 sym_execute) is done
// here on scalar value ids: every tensor element is a value id, data-movement
// operators (view, transpose, chunk, expand, move, all_gather, all_to_all,
// embedding gathers) only remap ids and cost nothing at run time, arithmetic
// creates value-numbered SSA nodes (global value numbering with constant
// folding, the analogue of the reference's interning fast path,
// sym.py:92-128). Obligations whose two sides receive the same value id are
// closed at compile time; the cones of the rest, plus every definedness
// condition (the reference's require_nonzero, sym.py:379-387), are scheduled
// depth-first, register-allocated into a small slot file and emitted as
// bytecode for the GPU interpreter.
#include "compiler.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <queue>
#include <stdexcept>
#include <unordered_map>
#include <unordered_set>

#include "field.hpp"

namespace pqw {
namespace {

constexpr int32_t IR_MAGIC = 0x50515701;
constexpr uint32_t NONE = 0xFFFFFFFFu;
constexpr size_t CHUNK = 16;  // max operands of one n-ary sum / dot before chunking

enum VKind : uint8_t { K_CONST = 0, K_VAR = 1, K_OP = 2 };
enum VOp : uint8_t { O_NONE = 0, O_ADD, O_SUB, O_MUL, O_NEG, O_DIV, O_HASH, O_SUMN, O_DOT, O_INV };
// F_UF: an uninterpreted function (or a constant folded from one) is in the
// value's cone (the reference's Expr.has_uf); F_POS: a definedness condition
// that also requires positivity (require_positive)
enum : uint8_t { F_DEN = 1, F_INT = 2, F_UF = 4, F_POS = 8 };
enum Fn : uint32_t { FN_EXP = 0, FN_RSQRT = 1, FN_SIGMOID = 2 };

struct Val {
  uint8_t kind, op, flags, pad;
  uint32_t a, b;      // operand ids, or (pool offset, length) for SUMN/DOT
  uint64_t aux;       // residue (const) / fn (hash) / local var index (var)
  uint32_t dnum, dden;
};

struct Exact {
  bool ok;
  int64_t num, den;   // den > 0, reduced
};

struct Div0 {
  int side;
};
struct BadIndex {};

static inline uint32_t sat_add(uint32_t a, uint32_t b) {
  uint64_t s = (uint64_t)a + b;
  return s > 0x7FFFFFFFu ? 0x7FFFFFFFu : (uint32_t)s;
}

static int64_t gcd64(int64_t a, int64_t b) {
  if (a < 0) a = -a;
  if (b < 0) b = -b;
  while (b) {
    int64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

static Exact make_exact(__int128 num, __int128 den) {
  if (den == 0) return {false, 0, 0};
  if (den < 0) {
    num = -num;
    den = -den;
  }
  __int128 a = num < 0 ? -num : num, b = den;
  while (b) {
    __int128 t = a % b;
    a = b;
    b = t;
  }
  if (a > 1) {
    num /= a;
    den /= a;
  }
  const __int128 lim = (__int128)INT64_MAX;
  if (num > lim || num < -lim || den > lim) return {false, 0, 0};
  return {true, (int64_t)num, (int64_t)den};
}

static uint32_t residue_of(int64_t num, int64_t den) {
  int64_t pm = (int64_t)P;
  int64_t n = num % pm;
  if (n < 0) n += pm;
  int64_t d = den % pm;
  if (d < 0) d += pm;
  return fmul((uint32_t)n, finv((uint32_t)d));
}

// Constants are interned by their exact rational when the compiler knows it,
// else by residue: two distinct rationals congruent mod p never share a value
// id (so no obligation between them closes at compile time).
struct ConstKey {
  uint8_t exact;
  int64_t a, b;  // (num, den) or (residue, 0)
  bool operator==(const ConstKey& o) const { return exact == o.exact && a == o.a && b == o.b; }
};
struct ConstKeyHash {
  size_t operator()(const ConstKey& k) const {
    return (size_t)mix64((uint64_t)k.a * 0x9E3779B97F4A7C15ull ^ (uint64_t)k.b ^ ((uint64_t)k.exact << 62));
  }
};

double real_fn(uint32_t fn, double x) {
  if (fn == 0) return std::exp(x);                                  // EXP
  if (fn == 1) return x > 0 ? 1.0 / std::sqrt(x) : std::nan("");   // RSQRT
  return 1.0 / (1.0 + std::exp(-x));                                // SIGMOID
}

struct Builder {
  std::vector<Val> vals;
  std::vector<Exact> exact;  // per value, meaningful for consts
  std::vector<double> realc; // per value: the real value of a constant (replay)
  std::vector<uint32_t> pool;
  std::unordered_map<uint64_t, uint32_t> head;
  std::vector<uint32_t> chain;
  std::unordered_map<ConstKey, uint32_t, ConstKeyHash> const_ids;
  bool lossy = false;        // an exact constant vanishes mod p, or two collide
  std::unordered_map<uint32_t, std::pair<int64_t, int64_t>> exact_of_res;
  std::vector<uint32_t> dens;  // definedness conditions, creation order
  const uint64_t* fn_keys = nullptr;
  int side = 0;
  uint32_t zero_id = NONE, one_id = NONE;

  uint32_t push(const Val& v, const Exact& ex, double real = 0.0) {
    vals.push_back(v);
    exact.push_back(ex);
    realc.push_back(real);
    chain.push_back(NONE);
    return (uint32_t)(vals.size() - 1);
  }

  // -- constants ---------------------------------------------------------
  // r: residue; ex: exact value when known; real: its real value (for the
  // real-valued replay); uf: folded from an uninterpreted function
  uint32_t cst(uint32_t r, Exact ex, double real, bool uf = false, bool is_int = false) {
    const ConstKey key = ex.ok ? ConstKey{1, ex.num, ex.den} : ConstKey{0, (int64_t)r, 0};
    auto it = const_ids.find(key);
    if (it != const_ids.end()) {
      if (is_int) vals[it->second].flags |= F_INT;
      if (uf) vals[it->second].flags |= F_UF;
      return it->second;
    }
    if (ex.ok && ex.num != 0 && ex.num % (int64_t)P == 0) lossy = true;
    if (ex.ok) {
      // two distinct exact constants with one image in F_p: the field cannot
      // tell apart what they scale
      auto r_it = exact_of_res.find(r);
      if (r_it == exact_of_res.end()) exact_of_res.emplace(r, std::make_pair(ex.num, ex.den));
      else if (r_it->second != std::make_pair(ex.num, ex.den)) lossy = true;
    }
    Val v{};
    v.kind = K_CONST;
    v.aux = r;
    v.flags = (uint8_t)((is_int ? F_INT : 0) | (uf ? F_UF : 0));
    uint32_t id = push(v, ex, ex.ok ? (double)ex.num / (double)ex.den : real);
    const_ids.emplace(key, id);
    return id;
  }
  uint32_t cst_int(int64_t n, bool is_int = false) {
    return cst(residue_of(n, 1), Exact{true, n, 1}, (double)n, false, is_int);
  }
  bool ufc(uint32_t x) const { return (vals[x].flags & F_UF) != 0; }
  // algebraic identities fold on the exact value when the compiler knows it
  // (a constant congruent to 0 or 1 mod p is not 0 or 1 over the rationals)
  bool is_zero(uint32_t x) const {
    return is_const(x) && (exact[x].ok ? exact[x].num == 0 : res(x) == 0);
  }
  bool is_one(uint32_t x) const {
    return is_const(x) && (exact[x].ok ? exact[x].num == 1 && exact[x].den == 1 : res(x) == 1);
  }
  uint32_t cst_exact(const Exact& ex, uint32_t r, double real) { return cst(r, ex, real); }
  bool is_const(uint32_t id) const { return vals[id].kind == K_CONST; }
  uint32_t res(uint32_t id) const { return (uint32_t)vals[id].aux; }
  uint32_t zero() { return zero_id == NONE ? (zero_id = cst_int(0)) : zero_id; }
  uint32_t one() { return one_id == NONE ? (one_id = cst_int(1)) : one_id; }

  uint32_t var(uint32_t local_idx) {
    Val v{};
    v.kind = K_VAR;
    v.a = local_idx;
    v.aux = local_idx;
    v.dnum = 1;
    return push(v, Exact{false, 0, 0});
  }

  // -- value numbering ---------------------------------------------------
  uint64_t key_of(uint8_t op, uint32_t a, uint32_t b, uint64_t aux, const uint32_t* list,
                  uint32_t n) const {
    uint64_t h = mix64(((uint64_t)op << 56) ^ aux ^ 0x1234567ull);
    if (list) {
      for (uint32_t i = 0; i < n; ++i) h = mix64(h + list[i] + 0x9E37ull);
      h = mix64(h ^ n);
    } else {
      h = mix64(h + a);
      h = mix64(h + ((uint64_t)b << 1));
    }
    return h;
  }
  bool same(uint32_t id, uint8_t op, uint32_t a, uint32_t b, uint64_t aux, const uint32_t* list,
            uint32_t n) const {
    const Val& v = vals[id];
    if (v.kind != K_OP || v.op != op || v.aux != aux) return false;
    if (list) {
      if (v.b != n) return false;
      return std::memcmp(&pool[v.a], list, n * sizeof(uint32_t)) == 0;
    }
    return v.a == a && v.b == b;
  }
  uint32_t intern(uint8_t op, uint32_t a, uint32_t b, uint64_t aux, const uint32_t* list,
                  uint32_t n, uint32_t dnum, uint32_t dden) {
    uint64_t k = key_of(op, a, b, aux, list, n);
    auto it = head.find(k);
    if (it != head.end()) {
      for (uint32_t c = it->second; c != NONE; c = chain[c])
        if (same(c, op, a, b, aux, list, n)) return c;
    }
    Val v{};
    v.kind = K_OP;
    v.op = op;
    v.aux = aux;
    v.dnum = dnum;
    v.dden = dden;
    bool uf = op == O_HASH;
    if (list) {
      for (uint32_t i = 0; i < n && !uf; ++i) uf = ufc(list[i]);
    } else {
      uf = uf || ufc(a) || (op != O_NEG && op != O_INV && op != O_HASH && ufc(b));
    }
    v.flags = uf ? F_UF : 0;
    if (list) {
      v.a = (uint32_t)pool.size();
      v.b = n;
      pool.insert(pool.end(), list, list + n);
    } else {
      v.a = a;
      v.b = b;
    }
    uint32_t id = push(v, Exact{false, 0, 0});
    if (it != head.end()) {
      chain[id] = it->second;
      it->second = id;
    } else {
      head.emplace(k, id);
    }
    return id;
  }

  // -- degree bookkeeping ------------------------------------------------
  void deg_add(uint32_t x, uint32_t y, uint32_t& n, uint32_t& d) const {
    const Val &a = vals[x], &b = vals[y];
    if (a.dden == 0 && b.dden == 0) {
      n = std::max(a.dnum, b.dnum);
      d = 0;
    } else {
      n = std::max(sat_add(a.dnum, b.dden), sat_add(b.dnum, a.dden));
      d = sat_add(a.dden, b.dden);
    }
  }

  // -- arithmetic with folding -------------------------------------------
  uint32_t add(uint32_t x, uint32_t y) {
    if (is_zero(x)) return y;
    if (is_zero(y)) return x;
    if (is_const(x) && is_const(y)) {
      Exact ex = (exact[x].ok && exact[y].ok)
                     ? make_exact((__int128)exact[x].num * exact[y].den +
                                      (__int128)exact[y].num * exact[x].den,
                                  (__int128)exact[x].den * exact[y].den)
                     : Exact{false, 0, 0};
      return cst(fadd(res(x), res(y)), ex, realc[x] + realc[y], ufc(x) || ufc(y));
    }
    if (x > y) std::swap(x, y);
    uint32_t n, d;
    deg_add(x, y, n, d);
    return intern(O_ADD, x, y, 0, nullptr, 0, n, d);
  }
  uint32_t sub(uint32_t x, uint32_t y) {
    if (x == y) return zero();
    if (is_zero(y)) return x;
    if (is_const(x) && is_const(y)) {
      Exact ex = (exact[x].ok && exact[y].ok)
                     ? make_exact((__int128)exact[x].num * exact[y].den -
                                      (__int128)exact[y].num * exact[x].den,
                                  (__int128)exact[x].den * exact[y].den)
                     : Exact{false, 0, 0};
      return cst(fsub(res(x), res(y)), ex, realc[x] - realc[y], ufc(x) || ufc(y));
    }
    uint32_t n, d;
    deg_add(x, y, n, d);
    return intern(O_SUB, x, y, 0, nullptr, 0, n, d);
  }
  uint32_t neg(uint32_t x) {
    if (is_const(x)) {
      Exact ex = exact[x].ok ? Exact{true, -exact[x].num, exact[x].den} : Exact{false, 0, 0};
      return cst(fneg(res(x)), ex, -realc[x], ufc(x));
    }
    return intern(O_NEG, x, 0, 0, nullptr, 0, vals[x].dnum, vals[x].dden);
  }
  uint32_t mul(uint32_t x, uint32_t y) {
    if (is_zero(x) || is_zero(y)) return zero();
    if (is_one(x)) return y;
    if (is_one(y)) return x;
    if (is_const(x) && is_const(y)) {
      Exact ex = (exact[x].ok && exact[y].ok)
                     ? make_exact((__int128)exact[x].num * exact[y].num,
                                  (__int128)exact[x].den * exact[y].den)
                     : Exact{false, 0, 0};
      return cst(fmul(res(x), res(y)), ex, realc[x] * realc[y], ufc(x) || ufc(y));
    }
    if (x > y) std::swap(x, y);
    return intern(O_MUL, x, y, 0, nullptr, 0, sat_add(vals[x].dnum, vals[y].dnum),
                  sat_add(vals[x].dden, vals[y].dden));
  }
  uint32_t scale_exact(uint32_t x, const Exact& ex, uint32_t r, double real) {
    return mul(x, cst_exact(ex, r, real));
  }

  // require_nonzero (reference sym.py:379-387): constants are decided now,
  // everything else becomes a definedness condition evaluated per witness.
  void require(uint32_t e, bool positive) {
    if (is_const(e)) {
      bool zero_v = res(e) == 0 || (exact[e].ok && exact[e].num == 0);
      bool nonpos = exact[e].ok && exact[e].num <= 0;
      if (zero_v || (positive && nonpos)) throw Div0{side};
      return;
    }
    if (!(vals[e].flags & F_DEN)) {
      vals[e].flags |= F_DEN;
      dens.push_back(e);
    }
    if (positive) vals[e].flags |= F_POS;
  }
  uint32_t div(uint32_t x, uint32_t y) {
    // caller has already called require(y, ...)
    if (is_const(y)) {
      uint32_t inv = finv(res(y));
      Exact ex = exact[y].ok && exact[y].num != 0
                     ? make_exact((__int128)exact[y].den, (__int128)exact[y].num)
                     : Exact{false, 0, 0};
      return mul(x, cst(inv, ex, 1.0 / realc[y], ufc(y)));
    }
    if (is_zero(x)) return zero();
    // x / y = x * y^-1 with the inverse value-numbered: rows that share a
    // denominator (softmax normalizers, expanded sums) invert it once
    uint32_t iv = intern(O_INV, y, 0, 0, nullptr, 0, vals[y].dden, vals[y].dnum);
    return mul(x, iv);
  }
  uint32_t hash(uint32_t fn, uint32_t x) {
    if (is_const(x))
      return cst(uf_apply(fn_keys[fn], res(x)), Exact{false, 0, 0}, real_fn(fn, realc[x]), true);
    return intern(O_HASH, x, 0, fn, nullptr, 0, 1, 0);
  }
  uint32_t sumn(std::vector<uint32_t> xs) {
    // fold constants, drop zeros, canonical order
    uint32_t cacc = NONE;
    std::vector<uint32_t> terms;
    terms.reserve(xs.size());
    for (uint32_t x : xs) {
      if (is_const(x)) {
        cacc = cacc == NONE ? x : add(cacc, x);
      } else {
        terms.push_back(x);
      }
    }
    if (cacc != NONE && !is_zero(cacc)) terms.push_back(cacc);
    if (terms.empty()) return cacc == NONE ? zero() : cacc;
    if (terms.size() == 1) return terms[0];
    if (terms.size() == 2) return add(terms[0], terms[1]);
    std::sort(terms.begin(), terms.end());
    if (terms.size() > CHUNK) {
      // long sums become sums of chunk partials, so the schedule never needs
      // more than CHUNK operands (plus the partials) live at once
      std::vector<uint32_t> parts;
      for (size_t i = 0; i < terms.size(); i += CHUNK)
        parts.push_back(sumn(std::vector<uint32_t>(
            terms.begin() + i, terms.begin() + std::min(terms.size(), i + CHUNK))));
      return sumn(parts);
    }
    uint32_t n = 0, d = 0;
    bool any_den = false;
    for (uint32_t t : terms) any_den |= vals[t].dden != 0;
    if (!any_den) {
      for (uint32_t t : terms) n = std::max(n, vals[t].dnum);
    } else {
      // common-denominator bound: sum of denominators
      for (uint32_t t : terms) d = sat_add(d, vals[t].dden);
      for (uint32_t t : terms) n = std::max(n, sat_add(vals[t].dnum, d - vals[t].dden));
    }
    return intern(O_SUMN, 0, 0, 0, terms.data(), (uint32_t)terms.size(), n, d);
  }
  // sum_i xs[i] * ys[i]
  uint32_t dot(const std::vector<uint32_t>& xs, const std::vector<uint32_t>& ys) {
    std::vector<std::pair<uint32_t, uint32_t>> pr;
    std::vector<uint32_t> extra;
    pr.reserve(xs.size());
    for (size_t i = 0; i < xs.size(); ++i) {
      uint32_t a = xs[i], b = ys[i];
      if (is_zero(a) || is_zero(b)) continue;
      if (is_const(a) || is_const(b) || (is_const(a) && is_const(b))) {
        extra.push_back(mul(a, b));
        continue;
      }
      if (a > b) std::swap(a, b);
      pr.emplace_back(a, b);
    }
    if (pr.empty()) return sumn(extra);
    if (pr.size() == 1 && extra.empty()) return mul(pr[0].first, pr[0].second);
    if (pr.size() == 1) {
      extra.push_back(mul(pr[0].first, pr[0].second));
      return sumn(extra);
    }
    std::sort(pr.begin(), pr.end());
    if (pr.size() > CHUNK) {
      std::vector<uint32_t> parts = extra;
      for (size_t i = 0; i < pr.size(); i += CHUNK) {
        std::vector<uint32_t> xs2, ys2;
        for (size_t j = i; j < std::min(pr.size(), i + CHUNK); ++j) {
          xs2.push_back(pr[j].first);
          ys2.push_back(pr[j].second);
        }
        parts.push_back(dot(xs2, ys2));
      }
      return sumn(parts);
    }
    std::vector<uint32_t> flat;
    flat.reserve(pr.size() * 2);
    uint32_t n = 0, d = 0;
    bool any_den = false;
    for (auto& p : pr) any_den |= (vals[p.first].dden | vals[p.second].dden) != 0;
    for (auto& p : pr) {
      flat.push_back(p.first);
      flat.push_back(p.second);
      if (any_den) d = sat_add(d, sat_add(vals[p.first].dden, vals[p.second].dden));
    }
    for (auto& p : pr) {
      uint32_t tn = sat_add(vals[p.first].dnum, vals[p.second].dnum);
      uint32_t td = sat_add(vals[p.first].dden, vals[p.second].dden);
      n = std::max(n, any_den ? sat_add(tn, d - td) : tn);
    }
    uint32_t id = intern(O_DOT, 0, 0, 0, flat.data(), (uint32_t)flat.size(), n, d);
    if (extra.empty()) return id;
    extra.push_back(id);
    return sumn(extra);
  }
  uint32_t muln(const std::vector<uint32_t>& xs) {
    uint32_t acc = one();
    for (uint32_t x : xs) acc = mul(acc, x);
    return acc;
  }
};

// ----------------------------------------------------------------------------
// tensor-level execution

struct TensorStore {
  std::vector<std::vector<int64_t>> shape;
  std::vector<std::vector<uint32_t>> data;
  std::vector<bool> set;
};

static int64_t vol(const std::vector<int64_t>& s) {
  int64_t v = 1;
  for (int64_t d : s) v *= d;
  return v;
}

static std::vector<int64_t> strides_of(const std::vector<int64_t>& s) {
  std::vector<int64_t> st(s.size(), 1);
  for (int i = (int)s.size() - 2; i >= 0; --i) st[i] = st[i + 1] * s[i + 1];
  return st;
}

static void unflat(int64_t f, const std::vector<int64_t>& s, std::vector<int64_t>& idx) {
  idx.assign(s.size(), 0);
  for (int a = (int)s.size() - 1; a >= 0; --a) {
    idx[a] = f % s[a];
    f /= s[a];
  }
}

static int64_t flat_of(const std::vector<int64_t>& idx, const std::vector<int64_t>& s) {
  int64_t f = 0;
  for (size_t a = 0; a < s.size(); ++a) f = f * s[a] + idx[a];
  return f;
}

[[noreturn]] static void bad(const std::string& m) { throw std::runtime_error(m); }

struct Compiler {
  Builder B;
  TensorStore T;
  const int64_t* consts;
  size_t n_consts;
  uint32_t n_vars;
  // obligations
  struct Obl {
    uint32_t l, r;
  };
  std::vector<Obl> obls;     // indexed by obligation id
  std::vector<uint8_t> obl_set;

  const std::vector<uint32_t>& in(int32_t t) {
    if (t < 0 || (size_t)t >= T.data.size() || !T.set[t]) bad("tensor read before write");
    return T.data[t];
  }
  void out(int32_t t, std::vector<uint32_t>&& v) {
    if (t < 0 || (size_t)t >= T.data.size()) bad("bad output tensor");
    if ((int64_t)v.size() != vol(T.shape[t])) bad("output element count mismatch");
    T.data[t] = std::move(v);
    T.set[t] = true;
  }
  uint32_t konst(int32_t ci) {
    if (ci < 0 || (size_t)ci >= n_consts) bad("const index out of range");
    const int64_t* c = consts + 3 * ci;
    Exact ex = c[2] != 0 ? Exact{true, c[1], c[2]} : Exact{false, 0, 0};
    return B.cst((uint32_t)c[0], ex, std::nan(""));
  }
  void record(uint32_t obl, uint32_t l, uint32_t r) {
    if (obl >= obls.size()) bad("obligation id out of range");
    if (obl_set[obl]) bad("obligation id reused");
    obls[obl] = {l, r};
    obl_set[obl] = 1;
  }

  void run_op(int32_t op, const int32_t* ins, int n_in, const int32_t* outs, int n_out,
              const int32_t* at, int n_at);
};

void Compiler::run_op(int32_t op, const int32_t* ins, int n_in, const int32_t* outs, int n_out,
                      const int32_t* at, int n_at) {
  auto need = [&](bool c, const char* m) {
    if (!c) bad(std::string("op ") + std::to_string(op) + ": " + m);
  };
  auto shp = [&](int32_t t) -> const std::vector<int64_t>& { return T.shape.at(t); };
  switch (op) {
    case PQW_T_SIDE:
      need(n_at == 1, "side attr");
      B.side = at[0];
      return;
    case PQW_T_VARS: {
      need(n_out == 1 && n_at == 1, "vars arity");
      int64_t n = vol(shp(outs[0]));
      need(at[0] >= 0 && (uint64_t)at[0] + n <= n_vars, "var range");
      std::vector<uint32_t> v(n);
      for (int64_t i = 0; i < n; ++i) v[i] = B.var((uint32_t)(at[0] + i));
      out(outs[0], std::move(v));
      return;
    }
    case PQW_T_INTS: {
      need(n_out == 1 && n_at == 1, "ints arity");
      int64_t n = vol(shp(outs[0]));
      std::vector<uint32_t> v(n);
      for (int64_t i = 0; i < n; ++i) {
        int32_t ci = at[0] + (int32_t)i;
        need(ci >= 0 && (size_t)ci < n_consts, "int const range");
        const int64_t* c = consts + 3 * ci;
        need(c[2] == 1, "ints must be exact integers");
        v[i] = B.cst_int(c[1], true);
      }
      out(outs[0], std::move(v));
      return;
    }
    case PQW_T_SLICE: {
      need(n_in == 1 && n_out == 1, "slice arity");
      const auto& is = shp(ins[0]);
      const auto& os = shp(outs[0]);
      need((int)is.size() == n_at && os.size() == is.size(), "slice rank");
      const auto& x = in(ins[0]);
      int64_t n = vol(os);
      std::vector<uint32_t> v(n);
      std::vector<int64_t> idx;
      for (int64_t f = 0; f < n; ++f) {
        unflat(f, os, idx);
        for (size_t a = 0; a < idx.size(); ++a) {
          idx[a] += at[a];
          need(idx[a] >= 0 && idx[a] < is[a], "slice out of bounds");
        }
        v[f] = x[flat_of(idx, is)];
      }
      out(outs[0], std::move(v));
      return;
    }
    case PQW_T_RESID: {
      need(n_in >= 1 && n_out == 1, "resid arity");
      const auto& x = in(ins[0]);
      std::vector<uint32_t> v(x.size());
      for (size_t i = 0; i < x.size(); ++i) {
        std::vector<uint32_t> rest;
        for (int k = 1; k < n_in; ++k) rest.push_back(in(ins[k])[i]);
        v[i] = rest.empty() ? x[i] : B.sub(x[i], B.sumn(rest));
      }
      out(outs[0], std::move(v));
      return;
    }
    case PQW_T_CHECK: {
      need(n_in == 2 && n_at == 1, "check arity");
      const auto& l = in(ins[0]);
      const auto& r = in(ins[1]);
      need(l.size() == r.size(), "check size");
      for (size_t i = 0; i < l.size(); ++i) record((uint32_t)(at[0] + i), l[i], r[i]);
      return;
    }
    case PQW_T_CHECKSUM: {
      need(n_in >= 2 && n_at == 1, "checksum arity");
      const auto& l = in(ins[0]);
      for (size_t i = 0; i < l.size(); ++i) {
        std::vector<uint32_t> parts;
        for (int k = 1; k < n_in; ++k) parts.push_back(in(ins[k])[i]);
        record((uint32_t)(at[0] + i), l[i], B.sumn(parts));
      }
      return;
    }
    case PQW_T_ADD:
    case PQW_T_SUB:
    case PQW_T_MUL:
    case PQW_T_DIV:
    case PQW_T_DROPOUT:
    case PQW_T_SILU_GRAD: {
      need(n_in == 2 && n_out == 1, "binary arity");
      const auto& x = in(ins[0]);
      const auto& y = in(ins[1]);
      need(x.size() == y.size(), "binary sizes");
      std::vector<uint32_t> v(x.size());
      bool den_pos = n_at >= 1 && at[0] != 0;
      for (size_t i = 0; i < x.size(); ++i) {
        switch (op) {
          case PQW_T_ADD: v[i] = B.add(x[i], y[i]); break;
          case PQW_T_SUB: v[i] = B.sub(x[i], y[i]); break;
          case PQW_T_MUL:
          case PQW_T_DROPOUT: v[i] = B.mul(x[i], y[i]); break;
          case PQW_T_DIV:
            B.require(y[i], den_pos);
            v[i] = B.div(x[i], y[i]);
            break;
          default: {  // silu_grad(x, g) = g * (s + x*s*(1-s)), s = SIGMOID(x)
            uint32_t s = B.hash(FN_SIGMOID, x[i]);
            uint32_t inner = B.add(s, B.mul(B.mul(x[i], s), B.sub(B.one(), s)));
            v[i] = B.mul(y[i], inner);
          }
        }
      }
      out(outs[0], std::move(v));
      return;
    }
    case PQW_T_IDENTITY:
    case PQW_T_MOVE:
    case PQW_T_VIEW: {
      need(n_in == 1 && n_out == 1, "unary arity");
      std::vector<uint32_t> v = in(ins[0]);
      out(outs[0], std::move(v));
      return;
    }
    case PQW_T_SCALE:
    case PQW_T_SHIFT: {
      need(n_in == 1 && n_out == 1 && n_at == 1, "scale arity");
      uint32_t c = konst(at[0]);
      const auto& x = in(ins[0]);
      std::vector<uint32_t> v(x.size());
      for (size_t i = 0; i < x.size(); ++i)
        v[i] = op == PQW_T_SCALE ? B.mul(x[i], c) : B.add(x[i], c);
      out(outs[0], std::move(v));
      return;
    }
    case PQW_T_POW: {
      need(n_in == 1 && n_out == 1 && n_at == 1 && at[0] >= 1, "pow arity");
      const auto& x = in(ins[0]);
      std::vector<uint32_t> v(x.size());
      for (size_t i = 0; i < x.size(); ++i) {
        uint32_t acc = x[i];
        for (int k = 1; k < at[0]; ++k) acc = B.mul(acc, x[i]);
        v[i] = acc;
      }
      out(outs[0], std::move(v));
      return;
    }
    case PQW_T_RSQRT:
    case PQW_T_SILU: {
      need(n_in == 1 && n_out == 1, "unary arity");
      const auto& x = in(ins[0]);
      std::vector<uint32_t> v(x.size());
      for (size_t i = 0; i < x.size(); ++i) {
        if (op == PQW_T_RSQRT) {
          B.require(x[i], true);
          v[i] = B.hash(FN_RSQRT, x[i]);
        } else {
          v[i] = B.mul(x[i], B.hash(FN_SIGMOID, x[i]));
        }
      }
      out(outs[0], std::move(v));
      return;
    }
    case PQW_T_SOFTMAX: {
      need(n_in == 1 && n_out == 1, "softmax arity");
      const auto& s = shp(ins[0]);
      const auto& x = in(ins[0]);
      int64_t n = s.back();
      need(n >= 1, "softmax axis");
      int64_t rows = (int64_t)x.size() / n;
      std::vector<uint32_t> v(x.size());
      for (int64_t r = 0; r < rows; ++r) {
        std::vector<uint32_t> e(n);
        for (int64_t j = 0; j < n; ++j) e[j] = B.hash(FN_EXP, x[r * n + j]);
        uint32_t tot = B.sumn(e);
        B.require(tot, true);
        for (int64_t j = 0; j < n; ++j) v[r * n + j] = B.div(e[j], tot);
      }
      out(outs[0], std::move(v));
      return;
    }
    case PQW_T_CREATE_MASK: {
      need(n_out == 1, "mask arity");
      const auto& s = shp(outs[0]);
      need(s.size() == 2, "mask rank");
      std::vector<uint32_t> v(s[0] * s[1]);
      for (int64_t i = 0; i < s[0]; ++i)
        for (int64_t j = 0; j < s[1]; ++j) v[i * s[1] + j] = j <= i ? B.one() : B.zero();
      out(outs[0], std::move(v));
      return;
    }
    case PQW_T_APPLY_MASK: {
      need(n_in == 2 && n_out == 1, "apply_mask arity");
      const auto& xs = shp(ins[0]);
      const auto& ms = shp(ins[1]);
      need(xs.size() >= 2 && ms.size() == 2, "apply_mask rank");
      const auto& x = in(ins[0]);
      const auto& m = in(ins[1]);
      int64_t a = xs[xs.size() - 2], b = xs.back();
      need(ms[0] == a && ms[1] == b, "apply_mask shape");
      std::vector<uint32_t> v(x.size());
      for (size_t f = 0; f < x.size(); ++f) {
        int64_t j = (int64_t)f % b, i = ((int64_t)f / b) % a;
        v[f] = B.mul(x[f], m[i * b + j]);
      }
      out(outs[0], std::move(v));
      return;
    }
    case PQW_T_TRANSPOSE: {
      need(n_in == 1 && n_out == 1, "transpose arity");
      const auto& is = shp(ins[0]);
      const auto& os = shp(outs[0]);
      need((int)is.size() == n_at, "perm rank");
      const auto& x = in(ins[0]);
      auto ist = strides_of(is);
      std::vector<uint32_t> v(x.size());
      std::vector<int64_t> oidx;
      for (int64_t f = 0; f < (int64_t)x.size(); ++f) {
        unflat(f, os, oidx);
        int64_t src = 0;
        // out axis k holds input axis perm[k]
        for (int k = 0; k < n_at; ++k) src += oidx[k] * ist[at[k]];
        v[f] = x[src];
      }
      out(outs[0], std::move(v));
      return;
    }
    case PQW_T_EXPAND: {
      need(n_in == 1 && n_out == 1, "expand arity");
      const auto& is = shp(ins[0]);
      const auto& os = shp(outs[0]);
      need(is.size() == os.size(), "expand rank");
      const auto& x = in(ins[0]);
      auto ist = strides_of(is);
      int64_t n = vol(os);
      std::vector<uint32_t> v(n);
      std::vector<int64_t> oidx;
      for (int64_t f = 0; f < n; ++f) {
        unflat(f, os, oidx);
        int64_t src = 0;
        for (size_t a = 0; a < is.size(); ++a) src += (is[a] == 1 ? 0 : oidx[a]) * ist[a];
        v[f] = x[src];
      }
      out(outs[0], std::move(v));
      return;
    }
    case PQW_T_SUM:
    case PQW_T_MEAN: {
      need(n_in == 1 && n_out == 1 && n_at >= 1, "sum arity");
      const auto& is = shp(ins[0]);
      bool keep = at[0] != 0;
      std::vector<bool> red(is.size(), false);
      for (int k = 1; k < n_at; ++k) {
        need(at[k] >= 0 && (size_t)at[k] < is.size(), "sum axis");
        red[at[k]] = true;
      }
      const auto& x = in(ins[0]);
      const auto& os = shp(outs[0]);
      int64_t on = vol(os);
      std::vector<std::vector<uint32_t>> acc(on);
      int64_t count = 1;
      for (size_t a = 0; a < is.size(); ++a)
        if (red[a]) count *= is[a];
      std::vector<int64_t> idx;
      for (int64_t f = 0; f < (int64_t)x.size(); ++f) {
        unflat(f, is, idx);
        int64_t o = 0;
        for (size_t a = 0; a < is.size(); ++a) {
          if (red[a]) {
            if (keep) o = o * 1;
          } else {
            o = o * is[a] + idx[a];
          }
        }
        need(o < on, "sum index");
        acc[o].push_back(x[f]);
      }
      std::vector<uint32_t> v(on);
      for (int64_t o = 0; o < on; ++o) {
        uint32_t s = B.sumn(acc[o]);
        if (op == PQW_T_MEAN) {
          need(count >= 1, "mean of nothing");
          s = B.mul(s, B.cst(finv(residue_of(count, 1)), make_exact(1, count), 1.0 / (double)count));
        }
        v[o] = s;
      }
      out(outs[0], std::move(v));
      return;
    }
    case PQW_T_MATMUL: {
      need(n_in == 2 && n_out == 1, "matmul arity");
      const auto& as = shp(ins[0]);
      const auto& bs = shp(ins[1]);
      need(as.size() >= 2 && bs.size() >= 2, "matmul rank");
      const auto& A = in(ins[0]);
      const auto& Bv = in(ins[1]);
      int64_t M = as[as.size() - 2], K = as.back(), N = bs.back();
      need(bs[bs.size() - 2] == K, "matmul contraction");
      bool bbatch = bs.size() == as.size();
      int64_t lead = (int64_t)A.size() / (M * K);
      std::vector<uint32_t> v(lead * M * N);
      std::vector<uint32_t> xs(K), ys(K);
      for (int64_t l = 0; l < lead; ++l) {
        const uint32_t* a = &A[l * M * K];
        const uint32_t* b = bbatch ? &Bv[l * K * N] : &Bv[0];
        for (int64_t m = 0; m < M; ++m)
          for (int64_t n = 0; n < N; ++n) {
            for (int64_t k = 0; k < K; ++k) {
              xs[k] = a[m * K + k];
              ys[k] = b[k * N + n];
            }
            v[(l * M + m) * N + n] = B.dot(xs, ys);
          }
      }
      out(outs[0], std::move(v));
      return;
    }
    case PQW_T_EINSUM: {
      // attrs: n_subs, then per input: len, letters...; then out len, letters...
      need(n_out == 1 && n_at >= 1, "einsum arity");
      int pos = 0;
      int ns = at[pos++];
      need(ns == n_in, "einsum subs");
      std::vector<std::vector<int32_t>> subs(ns);
      for (int s = 0; s < ns; ++s) {
        int len = at[pos++];
        subs[s].assign(at + pos, at + pos + len);
        pos += len;
      }
      int olen = at[pos++];
      std::vector<int32_t> rhs(at + pos, at + pos + olen);
      pos += olen;
      need(pos == n_at, "einsum attr length");
      std::unordered_map<int32_t, int64_t> ext;
      for (int s = 0; s < ns; ++s) {
        const auto& sh = shp(ins[s]);
        need(sh.size() == subs[s].size(), "einsum rank");
        for (size_t a = 0; a < sh.size(); ++a) ext[subs[s][a]] = sh[a];
      }
      std::vector<int32_t> contracted;
      for (auto& kv : ext)
        if (std::find(rhs.begin(), rhs.end(), kv.first) == rhs.end()) contracted.push_back(kv.first);
      std::sort(contracted.begin(), contracted.end());
      std::vector<int64_t> cshape;
      for (int32_t c : contracted) cshape.push_back(ext[c]);
      const auto& os = shp(outs[0]);
      int64_t on = vol(os), cn = vol(cshape);
      std::vector<std::vector<int64_t>> ist(ns);
      for (int s = 0; s < ns; ++s) ist[s] = strides_of(shp(ins[s]));
      std::vector<uint32_t> v(on);
      std::vector<int64_t> oidx, cidx;
      std::unordered_map<int32_t, int64_t> bind;
      for (int64_t f = 0; f < on; ++f) {
        unflat(f, os, oidx);
        for (size_t a = 0; a < rhs.size(); ++a) bind[rhs[a]] = oidx[a];
        std::vector<uint32_t> prods;
        std::vector<uint32_t> xs, ys;
        for (int64_t c = 0; c < cn; ++c) {
          unflat(c, cshape, cidx);
          for (size_t a = 0; a < contracted.size(); ++a) bind[contracted[a]] = cidx[a];
          std::vector<uint32_t> fac(ns);
          for (int s = 0; s < ns; ++s) {
            int64_t off = 0;
            for (size_t a = 0; a < subs[s].size(); ++a) off += bind[subs[s][a]] * ist[s][a];
            fac[s] = in(ins[s])[off];
          }
          if (ns == 2) {
            xs.push_back(fac[0]);
            ys.push_back(fac[1]);
          } else {
            prods.push_back(B.muln(fac));
          }
        }
        v[f] = ns == 2 ? B.dot(xs, ys) : B.sumn(prods);
      }
      out(outs[0], std::move(v));
      return;
    }
    case PQW_T_FULL: {
      need(n_out == 1 && n_at == 1, "full arity");
      uint32_t c = konst(at[0]);
      out(outs[0], std::vector<uint32_t>(vol(shp(outs[0])), c));
      return;
    }
    case PQW_T_CHUNK: {
      need(n_in == 1 && n_out == 1 && n_at == 3, "chunk arity");
      const auto& is = shp(ins[0]);
      const auto& os = shp(outs[0]);
      int ax = at[0];
      need(ax >= 0 && (size_t)ax < is.size(), "chunk axis");
      int64_t off = (int64_t)at[2] * os[ax];
      const auto& x = in(ins[0]);
      int64_t n = vol(os);
      std::vector<uint32_t> v(n);
      std::vector<int64_t> idx;
      for (int64_t f = 0; f < n; ++f) {
        unflat(f, os, idx);
        idx[ax] += off;
        need(idx[ax] < is[ax], "chunk out of bounds");
        v[f] = x[flat_of(idx, is)];
      }
      out(outs[0], std::move(v));
      return;
    }
    case PQW_T_EMBEDDING: {
      need(n_in == 2 && n_out == 1, "embedding arity");
      const auto& ts = shp(ins[0]);
      const auto& tab = in(ins[0]);
      const auto& ids = in(ins[1]);
      int64_t V = ts[0], H = ts[1];
      std::vector<uint32_t> v;
      v.reserve(ids.size() * H);
      for (uint32_t id : ids) {
        need(B.is_const(id) && B.exact[id].ok && B.exact[id].den == 1, "embedding ids must be concrete");
        int64_t row = B.exact[id].num;
        if (row < 0 || row >= V) throw BadIndex{};
        for (int64_t h = 0; h < H; ++h) v.push_back(tab[row * H + h]);
      }
      out(outs[0], std::move(v));
      return;
    }
    case PQW_T_EMBEDDING_GRAD: {
      need(n_in == 2 && n_out == 1, "embedding_grad arity");
      const auto& g = in(ins[0]);
      const auto& ids = in(ins[1]);
      const auto& os = shp(outs[0]);
      int64_t V = os[0], H = os[1];
      std::vector<std::vector<uint32_t>> acc(V * H);
      for (size_t i = 0; i < ids.size(); ++i) {
        uint32_t id = ids[i];
        need(B.is_const(id) && B.exact[id].ok && B.exact[id].den == 1, "embedding ids must be concrete");
        int64_t row = B.exact[id].num;
        if (row < 0 || row >= V) throw BadIndex{};
        for (int64_t h = 0; h < H; ++h) acc[row * H + h].push_back(g[i * H + h]);
      }
      std::vector<uint32_t> v(V * H);
      for (int64_t f = 0; f < V * H; ++f) v[f] = B.sumn(acc[f]);
      out(outs[0], std::move(v));
      return;
    }
    case PQW_T_GNORM_SQ: {
      need(n_in >= 1 && n_out == 1, "gnorm arity");
      std::vector<uint32_t> xs;
      for (int k = 0; k < n_in; ++k) {
        const auto& x = in(ins[k]);
        xs.insert(xs.end(), x.begin(), x.end());
      }
      out(outs[0], std::vector<uint32_t>{B.dot(xs, xs)});
      return;
    }
    case PQW_T_ALL_REDUCE: {
      need(n_in == n_out && n_in >= 1, "all_reduce arity");
      size_t n = in(ins[0]).size();
      std::vector<uint32_t> v(n);
      for (size_t i = 0; i < n; ++i) {
        std::vector<uint32_t> parts(n_in);
        for (int k = 0; k < n_in; ++k) parts[k] = in(ins[k])[i];
        v[i] = B.sumn(parts);
      }
      for (int k = 0; k < n_out; ++k) out(outs[k], std::vector<uint32_t>(v));
      return;
    }
    case PQW_T_ALL_GATHER: {
      need(n_in == n_out && n_in >= 1 && n_at == 1, "all_gather arity");
      int ax = at[0];
      const auto& os = shp(outs[0]);
      int64_t n = vol(os);
      std::vector<uint32_t> v(n);
      std::vector<int64_t> idx;
      for (int64_t f = 0; f < n; ++f) {
        unflat(f, os, idx);
        int64_t c = idx[ax];
        bool done = false;
        for (int k = 0; k < n_in; ++k) {
          const auto& s = shp(ins[k]);
          if (c < s[ax]) {
            idx[ax] = c;
            v[f] = in(ins[k])[flat_of(idx, s)];
            done = true;
            break;
          }
          c -= s[ax];
        }
        need(done, "all_gather index");
      }
      for (int k = 0; k < n_out; ++k) out(outs[k], std::vector<uint32_t>(v));
      return;
    }
    case PQW_T_REDUCE_SCATTER: {
      need(n_in == n_out && n_in >= 1 && n_at == 1, "reduce_scatter arity");
      int ax = at[0];
      const auto& is = shp(ins[0]);
      for (int j = 0; j < n_out; ++j) {
        const auto& os = shp(outs[j]);
        int64_t n = vol(os);
        std::vector<uint32_t> v(n);
        std::vector<int64_t> idx;
        for (int64_t f = 0; f < n; ++f) {
          unflat(f, os, idx);
          idx[ax] += (int64_t)j * os[ax];
          int64_t src = flat_of(idx, is);
          std::vector<uint32_t> parts(n_in);
          for (int k = 0; k < n_in; ++k) parts[k] = in(ins[k])[src];
          v[f] = B.sumn(parts);
        }
        out(outs[j], std::move(v));
      }
      return;
    }
    case PQW_T_ALL_TO_ALL: {
      need(n_in == n_out && n_in >= 1 && n_at == 2, "all_to_all arity");
      int sa = at[0], ca = at[1];
      int k = n_in;
      const auto& is = shp(ins[0]);
      for (int j = 0; j < n_out; ++j) {
        const auto& os = shp(outs[j]);
        int64_t seg = os[ca] / k;
        int64_t n = vol(os);
        std::vector<uint32_t> v(n);
        std::vector<int64_t> idx;
        for (int64_t f = 0; f < n; ++f) {
          unflat(f, os, idx);
          int64_t src = idx[ca] / seg;
          idx[ca] = idx[ca] % seg;
          idx[sa] = idx[sa] + (int64_t)j * (is[sa] / k);
          v[f] = in(ins[src])[flat_of(idx, shp(ins[src]))];
        }
        out(outs[j], std::move(v));
      }
      return;
    }
    default:
      bad("unknown tensor opcode " + std::to_string(op));
  }
}

// ----------------------------------------------------------------------------
// code generation

struct Emitter {
  const Builder& B;
  std::vector<uint32_t> order;          // value ids in emission order (groups)
  std::vector<int32_t> group_of;        // value -> group index (-1 = not emitted)
  struct Group {
    uint8_t kind;  // 0 value, 1 check, 2 den
    uint32_t v, l, r, obl;
  };
  std::vector<Group> groups;

  explicit Emitter(const Builder& b) : B(b), group_of(b.vals.size(), -1) {}

  void operands(uint32_t id, std::vector<uint32_t>& out) const {
    const Val& v = B.vals[id];
    out.clear();
    if (v.kind != K_OP) return;
    switch (v.op) {
      case O_SUMN:
      case O_DOT:
        for (uint32_t i = 0; i < v.b; ++i) out.push_back(B.pool[v.a + i]);
        break;
      case O_NEG:
      case O_HASH:
      case O_INV:
        out.push_back(v.a);
        break;
      default:
        out.push_back(v.a);
        out.push_back(v.b);
    }
  }

  void emit_value(uint32_t root) {
    if (group_of[root] >= 0) return;
    std::vector<std::pair<uint32_t, uint32_t>> stack;  // (id, next operand index)
    std::vector<uint32_t> ops;
    stack.emplace_back(root, 0);
    while (!stack.empty()) {
      auto& top = stack.back();
      uint32_t id = top.first;
      if (group_of[id] >= 0) {
        stack.pop_back();
        continue;
      }
      operands(id, ops);
      bool pushed = false;
      while (top.second < ops.size()) {
        uint32_t c = ops[top.second++];
        if (group_of[c] < 0) {
          stack.emplace_back(c, 0);
          pushed = true;
          break;
        }
      }
      if (pushed) continue;
      group_of[id] = (int32_t)groups.size();
      groups.push_back({0, id, 0, 0, 0});
      if (B.vals[id].flags & F_DEN) groups.push_back({2, id, 0, 0, 0});
      stack.pop_back();
    }
  }
};

}  // namespace

// Parse a tensor-op program and run it through the front end (symbolic
// execution into the value graph). Throws Div0 / BadIndex / runtime_error.
static void run_front(Compiler& C, const int32_t* ir, size_t ir_len, const int64_t* consts,
                      size_t n_consts, uint32_t n_vars, const uint64_t fn_keys[3]) {
  C.B.fn_keys = fn_keys;
  C.consts = consts;
  C.n_consts = n_consts;
  C.n_vars = n_vars;
  size_t p = 0;
  auto rd = [&]() -> int32_t {
    if (p >= ir_len) bad("truncated program");
    return ir[p++];
  };
  if (rd() != IR_MAGIC) bad("bad program magic");
  int32_t n_t = rd(), n_ops = rd(), n_obl = rd();
  if (n_t < 0 || n_ops < 0 || n_obl < 0) bad("bad header");
  C.T.shape.resize(n_t);
  C.T.data.resize(n_t);
  C.T.set.assign(n_t, false);
  for (int32_t t = 0; t < n_t; ++t) {
    int32_t r = rd();
    if (r < 0 || r > 16) bad("bad rank");
    for (int32_t a = 0; a < r; ++a) {
      int32_t d = rd();
      if (d < 1) bad("bad dim");
      C.T.shape[t].push_back(d);
    }
  }
  C.obls.resize(n_obl);
  C.obl_set.assign(n_obl, 0);
  for (int32_t o = 0; o < n_ops; ++o) {
    int32_t op = rd(), ni = rd(), no = rd(), na = rd();
    if (ni < 0 || no < 0 || na < 0 || p + ni + no + na > ir_len) bad("bad op header");
    const int32_t* ins = ir + p;
    const int32_t* outs = ins + ni;
    const int32_t* at = outs + no;
    p += ni + no + na;
    C.run_op(op, ins, ni, outs, no, at, na);
  }
  for (int32_t o = 0; o < n_obl; ++o)
    if (!C.obl_set[o]) bad("obligation never checked");
}

CompiledStage compile_stage(const int32_t* ir, size_t ir_len, const int64_t* consts,
                            size_t n_consts, uint32_t n_vars, uint32_t var_base,
                            const uint64_t fn_keys[3], uint32_t smem_slots,
                            uint32_t n_warps, const SchedOptions& sched) {
  CompiledStage st;
  st.n_vars = n_vars;
  st.n_warps = n_warps;
  if (n_warps < 1 || n_warps > 32) bad("n_warps must be in [1, 32]");
  st.var_base = var_base;
  Compiler C;
  try {
    run_front(C, ir, ir_len, consts, n_consts, n_vars, fn_keys);
  } catch (const Div0& d) {
    st.status = d.side ? PQW_STAGE_PAR_DIV0 : PQW_STAGE_LOG_DIV0;
    return st;
  } catch (const BadIndex&) {
    st.status = PQW_STAGE_BAD_INDEX;
    return st;
  }
  const int32_t n_obl = (int32_t)C.obls.size();

  st.n_obligations = n_obl;

  // classify obligations: fast (same value), constant mismatch, residual
  const Builder& B = C.B;
  int64_t first_int_bad = -1, first_const_bad = -1;
  std::vector<uint32_t> residual;
  std::unordered_set<uint64_t> seen_pairs;
  for (int32_t o = 0; o < n_obl; ++o) {
    uint32_t l = C.obls[o].l, r = C.obls[o].r;
    if (l == r) {
      st.n_fast++;
      continue;
    }
    if (B.is_const(l) && B.is_const(r)) {
      bool li = B.vals[l].flags & F_INT, ri = B.vals[r].flags & F_INT;
      if (li && ri && first_int_bad < 0) first_int_bad = o;
      if (first_const_bad < 0) first_const_bad = o;
    }
    if (seen_pairs.insert(((uint64_t)l << 32) | r).second) residual.push_back(o);
  }
  st.n_residual = (uint32_t)residual.size();
  if (first_int_bad >= 0 || first_const_bad >= 0) {
    int64_t o = first_int_bad >= 0 ? first_int_bad : first_const_bad;
    st.status = PQW_STAGE_REFUTED_CONST;
    st.info = o;
    uint32_t l = C.obls[o].l, r = C.obls[o].r;
    st.const_lhs = B.res(l);
    st.const_rhs = B.res(r);
    st.exact_lhs = (B.exact[l].ok && B.exact[l].den == 1) ? B.exact[l].num : INT64_MIN;
    st.exact_rhs = (B.exact[r].ok && B.exact[r].den == 1) ? B.exact[r].num : INT64_MIN;
    return st;
  }
  if (B.lossy) {
    // an exact constant vanishes mod p: evaluation in F_p cannot decide the stage
    st.status = PQW_STAGE_LOSSY;
    return st;
  }
  // the degree bound of the stage: numerator degree of lhs - rhs
  for (uint32_t o : residual) {
    uint32_t l = C.obls[o].l, r = C.obls[o].r, n, d;
    B.deg_add(l, r, n, d);
    st.degree = std::max<uint64_t>(st.degree, n);
  }
  if (residual.empty() && B.dens.empty()) {
    st.status = PQW_STAGE_PROVEN;
    return st;
  }

  // schedule: obligation cones in order, checks as soon as both sides exist,
  // definedness conditions right after their value; leftover conditions last.
  Emitter E(B);
  for (uint32_t o : residual) {
    E.emit_value(C.obls[o].l);
    E.emit_value(C.obls[o].r);
    E.groups.push_back({1, 0, C.obls[o].l, C.obls[o].r, o});
  }
  for (uint32_t d : B.dens) E.emit_value(d);

  // ---- back end: DAG of scheduling units in depth-first priority order -------
  auto dag = std::make_shared<Dag>();
  {
    const size_t G0 = E.groups.size();
    // A guarded inversion's batch product is zero exactly when one of its
    // operands is (F_p has no zero divisors), so its bundle checks those
    // denominators itself (fn = 1): the DEN units of values that a guarded
    // inversion in this DAG takes are dropped (one dispatch fewer each).
    std::vector<uint8_t> inv_checked(B.vals.size(), 0);
    for (size_t g = 0; g < G0; ++g) {
      const auto& gr = E.groups[g];
      if (gr.kind != 0) continue;
      const Val& v = B.vals[gr.v];
      if (v.kind != K_CONST && v.kind != K_VAR && v.op == O_INV && (B.vals[v.a].flags & F_DEN))
        inv_checked[v.a] = 1;
    }
    std::vector<uint32_t> keep;
    keep.reserve(G0);
    for (size_t g = 0; g < G0; ++g)
      if (!(E.groups[g].kind == 2 && inv_checked[E.groups[g].v])) keep.push_back((uint32_t)g);
    const size_t G = keep.size();
    std::vector<int32_t> unit_of(B.vals.size(), -1);
    for (size_t u = 0; u < G; ++u)
      if (E.groups[keep[u]].kind == 0) unit_of[E.groups[keep[u]].v] = (int32_t)u;
    auto uof = [&](uint32_t v) -> uint32_t {
      if (unit_of[v] < 0) bad("internal: operand without a defining unit");
      return (uint32_t)unit_of[v];
    };
    std::vector<uint32_t> opnds;
    dag->units.resize(G);
    for (size_t u = 0; u < G; ++u) {
      const auto& gr = E.groups[keep[u]];
      DagUnit& d = dag->units[u];
      d.arg0 = (uint32_t)dag->pool.size();
      if (gr.kind == 1) {
        d.op = I_CHK;
        d.aux = gr.obl;
        dag->pool.push_back(uof(gr.l));
        dag->pool.push_back(uof(gr.r));
      } else if (gr.kind == 2) {
        d.op = I_DEN;
        dag->pool.push_back(uof(gr.v));
      } else {
        const Val& v = B.vals[gr.v];
        if (v.kind == K_CONST) {
          d.op = I_CONST;
          d.aux = (uint32_t)v.aux;
        } else if (v.kind == K_VAR) {
          d.op = I_VAR;
          d.aux = v.a;  // stage-relative: the device adds the stage's var_base
        } else {
          E.operands(gr.v, opnds);
          for (uint32_t o : opnds) dag->pool.push_back(uof(o));
          switch (v.op) {
            case O_ADD: d.op = I_SUM; d.k = 2; break;
            case O_SUMN: d.op = I_SUM; d.k = v.b; break;
            case O_MUL: d.op = I_DOT; d.k = 1; break;
            case O_DOT: d.op = I_DOT; d.k = v.b / 2; break;
            case O_SUB: d.op = I_SUB; break;
            case O_NEG: d.op = I_NEG; break;
            case O_HASH: d.op = I_HASH; d.fn = (uint32_t)v.aux; break;
            case O_INV:
              d.op = I_INV;
              d.guarded = (B.vals[v.a].flags & F_DEN) != 0;  // batch only checked denominators
              d.fn = d.guarded ? 1u : 0u;  // fn 1: the bundle is the operands' DEN check
              break;
            default: bad("internal: bad value op");
          }
          if (d.k > MAX_K) bad("internal: n-ary op wider than MAX_K");
        }
      }
      d.nargs = (uint32_t)dag->pool.size() - d.arg0;
    }
  }
  st.sched = sched;
  st.sched.n_warps = n_warps;
  st.sched.smem_slots = smem_slots;
  st.dag = std::move(dag);
  return st;
}

uint64_t dag_hash(const Dag& d) {
  uint64_t h = 0x44414731ull ^ d.units.size() ^ ((uint64_t)d.pool.size() << 32);
  auto absorb = [&h](uint64_t w) {
    h = (h ^ w) * 0x9E3779B97F4A7C15ull;
    h ^= h >> 29;
  };
  for (const DagUnit& u : d.units) {
    absorb((uint64_t)u.op | (uint64_t)u.fn << 8 | (uint64_t)u.k << 16 | (uint64_t)u.guarded << 63);
    absorb((uint64_t)u.aux | (uint64_t)u.arg0 << 32);
    absorb(u.nargs);
  }
  for (size_t i = 0; i < d.pool.size(); i += 2)
    absorb((uint64_t)d.pool[i] | (i + 1 < d.pool.size() ? (uint64_t)d.pool[i + 1] << 32 : 0));
  return mix64(h);
}

bool same_dag(const Dag& a, const Dag& b) {
  if (a.units.size() != b.units.size() || a.pool != b.pool) return false;
  for (size_t i = 0; i < a.units.size(); ++i) {
    const DagUnit &x = a.units[i], &y = b.units[i];
    if (x.op != y.op || x.fn != y.fn || x.k != y.k || x.aux != y.aux || x.arg0 != y.arg0 ||
        x.nargs != y.nargs || x.guarded != y.guarded)
      return false;
  }
  return true;
}

bool same_sched(const SchedOptions& a, const SchedOptions& b) {
  return a.n_warps == b.n_warps && a.smem_slots == b.smem_slots && a.window == b.window &&
         a.bmax == b.bmax && a.xlat == b.xlat && a.bundle_base == b.bundle_base &&
         a.spill_cost == b.spill_cost && a.pick_scan == b.pick_scan &&
         a.active_warps == b.active_warps;
}

void finalize_stage(CompiledStage& st) {
  if (st.status != PQW_STAGE_OK || st.be->ready) return;
  st.be->prog = schedule_program(*st.dag, st.sched);
  st.be->ready = true;
}

std::vector<uint32_t> obligation_support(const CompiledStage& st, uint32_t obl) {
  std::vector<uint32_t> vars;
  if (!st.dag) return vars;
  const Dag& d = *st.dag;
  std::vector<uint8_t> seen(d.units.size(), 0);
  std::vector<uint32_t> stack;
  for (uint32_t u = 0; u < d.units.size(); ++u)
    if (d.units[u].op == I_CHK && d.units[u].aux == obl) {
      stack.push_back(u);
      seen[u] = 1;
      break;
    }
  while (!stack.empty()) {
    const uint32_t u = stack.back();
    stack.pop_back();
    const DagUnit& x = d.units[u];
    if (x.op == I_VAR) vars.push_back(x.aux);
    for (uint32_t i = 0; i < x.nargs; ++i) {
      const uint32_t p = d.pool[x.arg0 + i];
      if (!seen[p]) {
        seen[p] = 1;
        stack.push_back(p);
      }
    }
  }
  std::sort(vars.begin(), vars.end());
  vars.erase(std::unique(vars.begin(), vars.end()), vars.end());
  return vars;
}

namespace {

// Residual obligations of a front end (deduplicated (lhs, rhs) pairs in
// obligation order: the reference's residual dict, stages.py:341-351).
std::vector<uint32_t> residual_of(const Compiler& C) {
  std::vector<uint32_t> out;
  std::unordered_set<uint64_t> seen;
  for (size_t o = 0; o < C.obls.size(); ++o) {
    const uint32_t l = C.obls[o].l, r = C.obls[o].r;
    if (l == r) continue;
    if (seen.insert(((uint64_t)l << 32) | r).second) out.push_back((uint32_t)o);
  }
  return out;
}

// Evaluate every value of the graph in F_p (vars from their witness values).
std::vector<uint32_t> eval_field(const Builder& B, const uint64_t* var_keys, uint32_t w) {
  std::vector<uint32_t> v(B.vals.size(), 0);
  for (size_t i = 0; i < B.vals.size(); ++i) {
    const Val& x = B.vals[i];
    if (x.kind == K_CONST) {
      v[i] = (uint32_t)x.aux;
      continue;
    }
    if (x.kind == K_VAR) {
      v[i] = witness_value(var_keys[x.aux], w);
      continue;
    }
    switch (x.op) {
      case O_ADD: v[i] = fadd(v[x.a], v[x.b]); break;
      case O_SUB: v[i] = fsub(v[x.a], v[x.b]); break;
      case O_MUL: v[i] = fmul(v[x.a], v[x.b]); break;
      case O_NEG: v[i] = fneg(v[x.a]); break;
      case O_INV: v[i] = v[x.a] ? finv(v[x.a]) : 0u; break;
      case O_HASH: v[i] = uf_apply(B.fn_keys[x.aux], v[x.a]); break;
      case O_SUMN: {
        uint32_t acc = 0;
        for (uint32_t k = 0; k < x.b; ++k) acc = fadd(acc, v[B.pool[x.a + k]]);
        v[i] = acc;
        break;
      }
      case O_DOT: {
        uint32_t acc = 0;
        for (uint32_t k = 0; k + 1 < x.b; k += 2)
          acc = fadd(acc, fmul(v[B.pool[x.a + k]], v[B.pool[x.a + k + 1]]));
        v[i] = acc;
        break;
      }
      default: bad("internal: bad value op");
    }
  }
  return v;
}

// Evaluate every value in double precision with the genuine functions; a
// failed evaluation (1/0, rsqrt of a non-positive value, overflow) is NaN.
std::vector<double> eval_real(const Builder& B, const double* vars) {
  std::vector<double> v(B.vals.size(), 0.0);
  for (size_t i = 0; i < B.vals.size(); ++i) {
    const Val& x = B.vals[i];
    double r;
    if (x.kind == K_CONST) {
      r = B.realc[i];
    } else if (x.kind == K_VAR) {
      r = vars[x.aux];
    } else {
      switch (x.op) {
        case O_ADD: r = v[x.a] + v[x.b]; break;
        case O_SUB: r = v[x.a] - v[x.b]; break;
        case O_MUL: r = v[x.a] * v[x.b]; break;
        case O_NEG: r = -v[x.a]; break;
        case O_INV: r = v[x.a] != 0.0 ? 1.0 / v[x.a] : std::nan(""); break;
        case O_HASH: r = real_fn((uint32_t)x.aux, v[x.a]); break;
        case O_SUMN: {
          r = 0.0;
          for (uint32_t k = 0; k < x.b; ++k) r += v[B.pool[x.a + k]];
          break;
        }
        case O_DOT: {
          r = 0.0;
          for (uint32_t k = 0; k + 1 < x.b; k += 2) r += v[B.pool[x.a + k]] * v[B.pool[x.a + k + 1]];
          break;
        }
        default: bad("internal: bad value op");
      }
    }
    v[i] = std::isfinite(r) ? r : std::nan("");
  }
  return v;
}

}  // namespace

int confirm_stage(const int32_t* ir, size_t ir_len, const int64_t* consts, size_t n_consts,
                  uint32_t n_vars, const uint64_t fn_keys[3], const uint64_t* var_keys,
                  uint32_t witness, const double* env_vals, size_t n_env, double tol,
                  int64_t out[4], double sides[2]) {
  out[0] = out[1] = out[2] = -1;
  out[3] = 0;
  sides[0] = sides[1] = 0.0;
  Compiler C;
  try {
    run_front(C, ir, ir_len, consts, n_consts, n_vars, fn_keys);
  } catch (const Div0&) {
    return -1;
  } catch (const BadIndex&) {
    return -1;
  }
  const Builder& B = C.B;
  const auto res = residual_of(C);
  std::vector<uint32_t> uf;
  for (uint32_t o : res)
    if (B.ufc(C.obls[o].l) || B.ufc(C.obls[o].r)) uf.push_back(o);
  out[3] = (int64_t)uf.size();
  // 1. an obligation free of uninterpreted functions that fails in F_p at the
  //    witness: an exact rational counterexample (no replay needed)
  {
    const auto v = eval_field(B, var_keys, witness);
    bool valid = true;
    for (uint32_t d : B.dens) valid = valid && v[d] != 0;
    if (valid)
      for (uint32_t o : res) {
        const uint32_t l = C.obls[o].l, r = C.obls[o].r;
        if (!B.ufc(l) && !B.ufc(r) && v[l] != v[r]) {
          out[0] = o;
          return 0;
        }
      }
  }
  // 2. the reference's replay with the genuine functions (stages.py:241-264)
  for (size_t k = 0; k < n_env; ++k) {
    const auto v = eval_real(B, env_vals + k * (size_t)n_vars);
    bool hold = true;
    for (uint32_t d : B.dens) {
      const double x = v[d];
      const bool pos = (B.vals[d].flags & F_POS) != 0;
      if (std::isnan(x) || (pos ? x <= 1e-12 : std::fabs(x) <= 1e-12)) {
        hold = false;
        break;
      }
    }
    if (!hold) continue;
    for (uint32_t o : uf) {
      const double l = v[C.obls[o].l], r = v[C.obls[o].r];
      if (std::isnan(l) || std::isnan(r)) continue;
      if (std::fabs(l - r) > tol) {
        out[1] = (int64_t)k;
        out[2] = o;
        sides[0] = l;
        sides[1] = r;
        return 0;
      }
    }
  }
  return 0;
}

}  // namespace pqw

// field.hpp -- arithmetic in F_p, p = 2^31 - 1, and the keyed hashes that
// generate witnesses and interpret uninterpreted functions. Shared verbatim by
// the host compiler (constant folding) and the sm_100a kernel so both sides
// agree bit for bit; paper_2506_15961_b200/field.py and oracle/m31.py restate
// the same definitions.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define PQW_HD __host__ __device__ __forceinline__
#else
#define PQW_HD inline
#endif

namespace pqw {

constexpr uint32_t P = 2147483647u;          // 2^31 - 1
constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ull;

PQW_HD uint32_t fadd(uint32_t a, uint32_t b) {
  uint32_t s = a + b;                         // a, b < P so s < 2^32
  return s >= P ? s - P : s;
}
PQW_HD uint32_t fsub(uint32_t a, uint32_t b) { return a >= b ? a - b : a + (P - b); }
PQW_HD uint32_t fneg(uint32_t a) { return a ? P - a : 0u; }

// 62-bit product folded once: (t mod 2^31) + (t >> 31) <= 2P - 1, then one
// conditional subtraction lands in [0, P).
PQW_HD uint32_t fred62(uint64_t t) {
  uint32_t r = (uint32_t)(t & P) + (uint32_t)(t >> 31);
  return r >= P ? r - P : r;
}
#if defined(__CUDA_ARCH__) && defined(PQW_WHATIF_CHEAP_ARITH)  // timing what-if only (wrong values)
PQW_HD uint32_t fmul(uint32_t a, uint32_t b) { return a * b; }
#else
PQW_HD uint32_t fmul(uint32_t a, uint32_t b) { return fred62((uint64_t)a * b); }
#endif

// Full 64-bit accumulator to [0, P).
PQW_HD uint64_t ffold64(uint64_t x) { return (x & P) + (x >> 31); }  // < 2^34
PQW_HD uint32_t fred64(uint64_t x) {
#if defined(__CUDA_ARCH__) && defined(PQW_WHATIF_CHEAP_ARITH)
  return (uint32_t)x;
#endif
  x = ffold64(x);                              // < 2^31 + 2^33
  uint32_t r = (uint32_t)(x & P) + (uint32_t)(x >> 31);  // < 2^31 + 8
  return r >= P ? r - P : r;
}

// a^(P-2) = a^-1 for a != 0 (0 maps to 0). P - 2 = 2^31 - 3 = 0b1...1101.
PQW_HD uint32_t finv(uint32_t a) {
  // a^(2^k - 1) ladder: x_k = a^(2^k-1); x_{2k} = x_k^(2^k) * x_k
  uint32_t x1 = a;
  uint32_t x2 = fmul(fmul(x1, x1), x1);                 // 2^2-1
  uint32_t t = fmul(x2, x2); t = fmul(t, t);
  uint32_t x4 = fmul(t, x2);                            // 2^4-1
  t = x4;
  for (int i = 0; i < 4; ++i) t = fmul(t, t);
  uint32_t x8 = fmul(t, x4);                            // 2^8-1
  t = x8;
  for (int i = 0; i < 8; ++i) t = fmul(t, t);
  uint32_t x16 = fmul(t, x8);                           // 2^16-1
  t = x16;
  for (int i = 0; i < 8; ++i) t = fmul(t, t);
  uint32_t x24 = fmul(t, x8);                           // 2^24-1
  t = x24;
  for (int i = 0; i < 4; ++i) t = fmul(t, t);
  uint32_t x28 = fmul(t, x4);                           // 2^28-1
  t = fmul(x28, x28);                                   // 2^29-2
  t = fmul(t, x1);                                      // 2^29-1
  t = fmul(t, t);                                       // 2^30-2
  t = fmul(t, t);                                       // 2^31-4
  return fmul(t, x1);                                   // 2^31-3
}

PQW_HD uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// 64-bit hash -> field element: top 31 bits, P itself maps to 0.
PQW_HD uint32_t to_field(uint64_t h) {
  uint32_t r = (uint32_t)(h >> 33);
  return r == P ? 0u : r;
}

// Witness value of a variable (key = mix64(seed ^ fnv1a64(name))) at witness w.
PQW_HD uint32_t witness_value(uint64_t var_key, uint32_t w) {
  return to_field(mix64(var_key + (uint64_t)(w + 1u) * GOLDEN));
}

// Uninterpreted function application: fn_key = mix64(seed ^ fnv1a64(fn name)).
PQW_HD uint32_t uf_apply(uint64_t fn_key, uint32_t x) { return to_field(mix64(fn_key + x)); }

}  // namespace pqw

// rng.cuh — bit-exact port of the NumPy streams the reference draws entry points from.
//
// router.py:42-45:  default_rng(SeedSequence(entropy=(seed, qi))).choice(n, K, replace=False)
//
// Restated from NumPy's published algorithms (numpy.random: SeedSequence pool mixing with
// the hashmix/mix constants, PCG64 XSL-RR 128/64 seeded from generate_state(4, uint64),
// 32-bit draws served from the two halves of one 64-bit output, Lemire bounded draws,
// Generator.choice without replacement: Floyd's algorithm + Fisher-Yates shuffle when
// n <= 10000 or K <= n // 50, otherwise a tail Fisher-Yates over arange(n)).
// NumPy ships no .pyx sources here; the port is pinned empirically against NumPy over an
// (n, K, seed, qi) grid in tests/test_rng.py and tests/golden/rng.npz.
// Usable on host (tests, C ABI) and device (one thread per query).
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define RNG_HD __host__ __device__ __forceinline__
#else
#define RNG_HD static inline
#endif

namespace sbrng {

struct U128 { uint64_t hi, lo; };

RNG_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

RNG_HD U128 mul128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
  r.hi = mulhi64(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return r;
}
RNG_HD U128 add128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1 : 0);
  return r;
}

// ---- SeedSequence (pool_size 4) ------------------------------------------------
constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;

RNG_HD uint32_t hashmix(uint32_t v, uint32_t* hc) {
  v ^= *hc;
  *hc *= kMultA;
  v *= *hc;
  v ^= v >> 16;
  return v;
}
RNG_HD uint32_t mix(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  r ^= r >> 16;
  return r;
}

// entropy words of a non-negative int: 0 -> [0]; little-endian 32-bit words otherwise
RNG_HD int int_words(uint64_t v, uint32_t* out) {
  if (v == 0) { out[0] = 0; return 1; }
  int c = 0;
  while (v) { out[c++] = (uint32_t)v; v >>= 32; }
  return c;
}

// generate_state(8 uint32 words) for SeedSequence(entropy=(a, b))
RNG_HD void seedseq_state8(uint64_t a, uint64_t b, uint32_t* state) {
  uint32_t ent[4];
  int ne = int_words(a, ent);
  ne += int_words(b, ent + ne);
  uint32_t pool[4];
  uint32_t hc = kInitA;
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < ne ? ent[i] : 0u, &hc);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], &hc));
  for (int s = 4; s < ne; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[s], &hc));
  uint32_t hb = kInitB;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= kMultB;
    v *= hb;
    v ^= v >> 16;
    state[i] = v;
  }
}

// ---- PCG64 -----------------------------------------------------------------------
struct Pcg64 {
  U128 s, inc;
  uint32_t buf;
  int has;
};

RNG_HD void pcg_step(Pcg64* g) {
  const U128 mult = {0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull};
  g->s = add128(mul128(g->s, mult), g->inc);
}

RNG_HD void pcg_seed_words(Pcg64* g, const uint32_t* w) {
  uint64_t v0 = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
  uint64_t v1 = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
  uint64_t v2 = (uint64_t)w[4] | ((uint64_t)w[5] << 32);
  uint64_t v3 = (uint64_t)w[6] | ((uint64_t)w[7] << 32);
  U128 initstate = {v0, v1}, initseq = {v2, v3};
  g->inc.hi = (initseq.hi << 1) | (initseq.lo >> 63);
  g->inc.lo = (initseq.lo << 1) | 1u;
  g->s.hi = 0;
  g->s.lo = 0;
  pcg_step(g);
  g->s = add128(g->s, initstate);
  pcg_step(g);
  g->has = 0;
  g->buf = 0;
}

// default_rng(SeedSequence(entropy=(a, b)))
RNG_HD void pcg_from_entropy2(Pcg64* g, uint64_t a, uint64_t b) {
  uint32_t w[8];
  seedseq_state8(a, b, w);
  pcg_seed_words(g, w);
}

// jump parameters of `delta` PCG64 steps: s' = mult * s + plus (squaring, O(log delta))
RNG_HD void pcg_jump_params(U128 inc, uint64_t delta, U128* mult_out, U128* plus_out) {
  U128 cur_mult = {0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull};
  U128 cur_plus = inc;
  U128 acc_mult = {0, 1}, acc_plus = {0, 0};
  while (delta > 0) {
    if (delta & 1) {
      acc_mult = mul128(acc_mult, cur_mult);
      acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
    }
    cur_plus = mul128(add128(cur_mult, {0, 1}), cur_plus);
    cur_mult = mul128(cur_mult, cur_mult);
    delta >>= 1;
  }
  *mult_out = acc_mult;
  *plus_out = acc_plus;
}

// 64-bit output of a PCG64 state (XSL-RR)
RNG_HD uint64_t pcg_output(U128 s) {
  uint64_t x = s.hi ^ s.lo;
  unsigned rot = (unsigned)(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

RNG_HD uint64_t pcg_next64(Pcg64* g) {
  pcg_step(g);
  uint64_t x = g->s.hi ^ g->s.lo;
  unsigned rot = (unsigned)(g->s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

RNG_HD uint32_t pcg_next32(Pcg64* g) {
  if (g->has) { g->has = 0; return g->buf; }
  uint64_t v = pcg_next64(g);
  g->has = 1;
  g->buf = (uint32_t)(v >> 32);
  return (uint32_t)v;
}

// uniform integer in [0, rng] (rng < 2^32), Lemire's method as NumPy draws it
RNG_HD uint64_t bounded(Pcg64* g, uint64_t rng) {
  if (rng == 0) return 0;
  if (rng == 0xFFFFFFFFull) return pcg_next32(g);
  uint32_t r = (uint32_t)rng;
  uint32_t excl = r + 1u;
  uint64_t mm = (uint64_t)pcg_next32(g) * excl;
  uint32_t left = (uint32_t)mm;
  if (left < excl) {
    uint32_t thr = (0xFFFFFFFFu - r) % excl;
    while (left < thr) {
      mm = (uint64_t)pcg_next32(g) * excl;
      left = (uint32_t)mm;
    }
  }
  return mm >> 32;
}

// Which NumPy choice() regime applies (Generator.choice, replace=False, shuffle=True).
RNG_HD bool choice_uses_tail_shuffle(int64_t n, int64_t k) { return n > 10000 && k > n / 50; }

// Floyd's algorithm + shuffle, writing k distinct ids of [0, n).  `table` is scratch of
// `tmask + 1` slots (power of two >= k, any contents); open addressing, linear probe.  T is
// int64_t, or int32_t when n < 2^31 (the shared-memory variant of the entry kernel).
template <class T>
RNG_HD void choice_floyd(Pcg64* g, int64_t n, int64_t k, T* out, T* table, uint64_t tmask) {
  for (uint64_t i = 0; i <= tmask; ++i) table[i] = -1;
  for (int64_t j = n - k; j < n; ++j) {
    int64_t v = (int64_t)bounded(g, (uint64_t)j);
    uint64_t loc = (uint64_t)v & tmask;
    while (table[loc] != -1 && (int64_t)table[loc] != v) loc = (loc + 1) & tmask;
    if (table[loc] == -1) {
      table[loc] = (T)v;
      out[j - n + k] = (T)v;
    } else {
      loc = (uint64_t)j & tmask;
      while (table[loc] != -1) loc = (loc + 1) & tmask;
      table[loc] = (T)j;
      out[j - n + k] = (T)j;
    }
  }
  for (int64_t i = k - 1; i > 0; --i) {
    int64_t j = (int64_t)bounded(g, (uint64_t)i);
    T t = out[i]; out[i] = out[j]; out[j] = t;
  }
}

// Tail Fisher-Yates over a virtual arange(n): only swapped slots are materialised, in an
// open-addressing map slot -> value (`keys`/`vals`, `tmask + 1` entries, tmask + 1 >= 2k).
RNG_HD int64_t vmap_get(const int64_t* keys, const int64_t* vals, uint64_t tmask, int64_t slot) {
  uint64_t loc = ((uint64_t)slot * 0x9E3779B97F4A7C15ull) & tmask;
  while (keys[loc] != -1) {
    if (keys[loc] == slot) return vals[loc];
    loc = (loc + 1) & tmask;
  }
  return slot;
}
RNG_HD void vmap_put(int64_t* keys, int64_t* vals, uint64_t tmask, int64_t slot, int64_t v) {
  uint64_t loc = ((uint64_t)slot * 0x9E3779B97F4A7C15ull) & tmask;
  while (keys[loc] != -1 && keys[loc] != slot) loc = (loc + 1) & tmask;
  keys[loc] = slot;
  vals[loc] = v;
}
RNG_HD void choice_tail(Pcg64* g, int64_t n, int64_t k, int64_t* out, int64_t* keys,
                        int64_t* vals, uint64_t tmask) {
  for (uint64_t i = 0; i <= tmask; ++i) keys[i] = -1;
  int64_t stop = n - k > 1 ? n - k : 1;
  for (int64_t i = n - 1; i >= stop; --i) {
    int64_t j = (int64_t)bounded(g, (uint64_t)i);
    int64_t vi = vmap_get(keys, vals, tmask, i), vj = vmap_get(keys, vals, tmask, j);
    vmap_put(keys, vals, tmask, i, vj);
    vmap_put(keys, vals, tmask, j, vi);
  }
  for (int64_t t = 0; t < k; ++t) out[t] = vmap_get(keys, vals, tmask, n - k + t);
}

// scratch (int64 slots) one query's choice() needs, and the table mask it uses
RNG_HD uint64_t choice_table_size(int64_t n, int64_t k) {
  uint64_t want = choice_uses_tail_shuffle(n, k) ? (uint64_t)(4 * k) : (uint64_t)(2 * k);
  uint64_t p = 1;
  while (p < want) p <<= 1;
  return p;
}
RNG_HD uint64_t choice_scratch_slots(int64_t n, int64_t k) {
  uint64_t t = choice_table_size(n, k);
  return choice_uses_tail_shuffle(n, k) ? 2 * t : t;
}

// entry_points(n, k, seed, qi) of router.py:42-45
RNG_HD void entry_points(int64_t n, int64_t k, uint64_t seed, uint64_t qi, int64_t* out,
                         int64_t* scratch) {
  Pcg64 g;
  pcg_from_entropy2(&g, seed, qi);
  uint64_t t = choice_table_size(n, k);
  if (choice_uses_tail_shuffle(n, k))
    choice_tail(&g, n, k, out, scratch, scratch + t, t - 1);
  else
    choice_floyd(&g, n, k, out, scratch, t - 1);
}

}  // namespace sbrng

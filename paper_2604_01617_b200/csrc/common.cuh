// common.cuh — shared device utilities for the STABLE hot path on sm_100a.
//
// AUTO metric (reference _kernels.py:14-35):
//     U = sqrt(S_V) * (1 + S_A * inv_alpha)
// S_V = sum_t (f64 x_i[t] - f64 x_j[t])^2 and S_A = sum_t |f64 a_i[t] - f64 a_j[t]|, both
// accumulated in ascending t.  Every distance here is computed with explicitly rounded
// fp64 operations (__dsub_rn/__dmul_rn/__dadd_rn: no FMA contraction) in that same
// ascending order, one pair per thread, so the values equal the reference's
// bit for bit.  Work is spread by giving each thread many independent pairs (ILP), not
// by splitting one sum across lanes.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define SB_DEV __device__ __forceinline__
#define SB_HD __host__ __device__ __forceinline__

namespace sb {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// exact fp64 helpers (no contraction)
SB_DEV double dsub(double a, double b) { return __dsub_rn(a, b); }
SB_DEV double dmul(double a, double b) { return __dmul_rn(a, b); }
SB_DEV double dadd(double a, double b) { return __dadd_rn(a, b); }

// s_v accumulation step: s += (a - b)^2, each op rounded separately (_kernels.py:18-19)
SB_DEV double sq_step(double s, double a, double b) {
  double d = dsub(a, b);
  return dadd(s, dmul(d, d));
}

// attribute term between two data nodes (_kernels.py:20-22)
SB_DEV double attr_l1(const int32_t* __restrict__ ai, const int32_t* __restrict__ aj, int l) {
  double s = 0.0;
  for (int t = 0; t < l; ++t) s = dadd(s, fabs(dsub((double)ai[t], (double)aj[t])));
  return s;
}

// finish: sqrt(s_v) * (1 + s_a * inv_alpha)   (_kernels.py:23)
SB_DEV double auto_finish(double s_v, double s_a, double inv_alpha) {
  return dmul(sqrt(s_v), dadd(1.0, dmul(s_a, inv_alpha)));
}

// Exact pair distance of data rows i, j (used where no tiling is possible).
SB_DEV double pair_dist(const float* __restrict__ F, const int32_t* __restrict__ A, int m, int l,
                        int64_t i, int64_t j, double inv_alpha) {
  const float* xi = F + i * (int64_t)m;
  const float* xj = F + j * (int64_t)m;
  double s = 0.0;
  int t = 0;
  if (((m & 3) == 0)) {
    const float4* vi = reinterpret_cast<const float4*>(xi);
    const float4* vj = reinterpret_cast<const float4*>(xj);
    for (int q = 0; q < (m >> 2); ++q) {
      float4 a = __ldg(vi + q), b = __ldg(vj + q);
      s = sq_step(s, a.x, b.x);
      s = sq_step(s, a.y, b.y);
      s = sq_step(s, a.z, b.z);
      s = sq_step(s, a.w, b.w);
    }
    t = m;
  }
  for (; t < m; ++t) s = sq_step(s, __ldg(xi + t), __ldg(xj + t));
  return auto_finish(s, attr_l1(A + i * (int64_t)l, A + j * (int64_t)l, l), inv_alpha);
}

// ---------------------------------------------------------------------------
// keys.  Non-negative IEEE floats order like their bit patterns, so
//   build rows: key64 = (f32 bits << 32) | id        — the (f32 d, id) row order (_kernels.py:48-60)
//   routing / brute force: (f64 bits, id) compared lexicographically (_kernels.py:190-196, 546)
SB_HD uint64_t row_key(float d, uint32_t id) {
#ifdef __CUDA_ARCH__
  return ((uint64_t)__float_as_uint(d) << 32) | id;
#else
  union { float f; uint32_t u; } c; c.f = d;
  return ((uint64_t)c.u << 32) | id;
#endif
}
SB_HD float key_dist(uint64_t k) {
#ifdef __CUDA_ARCH__
  return __uint_as_float((uint32_t)(k >> 32));
#else
  union { float f; uint32_t u; } c; c.u = (uint32_t)(k >> 32);
  return c.f;
#endif
}
SB_HD uint32_t key_id(uint64_t k) { return (uint32_t)k; }
constexpr uint64_t kKeyInf = 0xFFFFFFFFFFFFFFFFull;

// (d, id) lexicographic less for fp64 distances
SB_DEV bool dlt(double da, uint32_t ia, double db, uint32_t ib) {
  return da < db || (da == db && ia < ib);
}

// (d, id) order for ids of a relabeled layout: ties compare the ORIGINAL ids perm[id]
// (perm == null: identity; ids >= n are padding and keep their value).  The lookup runs
// only on exact distance ties.
struct IdOrder {
  const int32_t* perm;
  uint32_t n;
  SB_DEV uint32_t key(uint32_t i) const { return (perm && i < n) ? (uint32_t)__ldg(perm + i) : i; }
  SB_DEV bool operator()(double da, uint32_t ia, double db, uint32_t ib) const {
    if (__builtin_expect(da != db, 1)) return da < db;
    return key(ia) < key(ib);
  }
};
struct PlainOrder {
  SB_DEV bool operator()(double da, uint32_t ia, double db, uint32_t ib) const {
    return dlt(da, ia, db, ib);
  }
};

// ---------------------------------------------------------------------------
// warp helpers
SB_DEV int lane_id() { return threadIdx.x & 31; }
SB_DEV int warp_id() { return threadIdx.x >> 5; }

template <typename T>
SB_DEV T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

SB_HD int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

// In-place bitonic sort of n64 (power of two) u64 keys in shared memory by one warp.
SB_DEV void warp_bitonic_u64(uint64_t* s, int n) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane_id(); i < n; i += 32) {
        int p = i ^ j;
        if (p > i) {
          uint64_t a = s[i], b = s[p];
          bool up = (i & k) == 0;
          if ((a > b) == up) { s[i] = b; s[p] = a; }
        }
      }
      __syncwarp();
    }
  }
}

// In-place bitonic sort of n (power of two) u64 keys in shared memory by a whole CTA.
SB_DEV void cta_bitonic_u64(uint64_t* s, int n) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        int p = i ^ j;
        if (p > i) {
          uint64_t a = s[i], b = s[p];
          bool up = (i & k) == 0;
          if ((a > b) == up) { s[i] = b; s[p] = a; }
        }
      }
      __syncthreads();
    }
  }
}

// an order on id words that carry flag bits outside `mask`
template <class Less>
struct MaskedOrder {
  Less lt;
  uint32_t mask;
  SB_DEV bool operator()(double da, uint32_t ia, double db, uint32_t ib) const {
    return lt(da, ia & mask, db, ib & mask);
  }
};

// Bitonic sort of (fp64 dist, u32 id) pairs held in two shared arrays, one warp.
template <class Less = PlainOrder>
SB_DEV void warp_bitonic_did(double* d, uint32_t* id, int n, Less lt = Less()) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane_id(); i < n; i += 32) {
        int p = i ^ j;
        if (p > i) {
          double da = d[i], db = d[p];
          uint32_t ia = id[i], ib = id[p];
          bool up = (i & k) == 0;
          bool gt = lt(db, ib, da, ia);
          if (gt == up) { d[i] = db; d[p] = da; id[i] = ib; id[p] = ia; }
        }
      }
      __syncwarp();
    }
  }
}

// warp_bitonic_did for a list in global memory: each stage walks the n/2 disjoint pairs
// (i, i | j) directly, U pairs per lane loaded before any is stored (pairs of a stage are
// disjoint), so the sort costs one L1/L2 round trip per U pairs rather than per pair.
template <class Less = PlainOrder, int U = 4>
SB_DEV void warp_bitonic_did_batched(double* d, uint32_t* id, int n, Less lt = Less()) {
  const int half = n >> 1;
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int lj = __ffs(j) - 1;
      for (int t0 = lane_id(); t0 < half; t0 += 32 * U) {
        double da[U], db[U];
        uint32_t ia[U], ib[U];
        int ii[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int t = t0 + 32 * u;
          ii[u] = -1;
          if (t < half) {
            const int i = ((t >> lj) << (lj + 1)) | (t & (j - 1));
            ii[u] = i;
            da[u] = d[i];
            db[u] = d[i | j];
            ia[u] = id[i];
            ib[u] = id[i | j];
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = ii[u];
          if (i < 0) continue;
          const bool up = (i & k) == 0;
          const bool gt = lt(db[u], ib[u], da[u], ia[u]);
          if (gt == up) {
            d[i] = db[u];
            d[i | j] = da[u];
            id[i] = ib[u];
            id[i | j] = ia[u];
          }
        }
      }
      __syncwarp();
    }
  }
}

// Merge c unsorted candidates (cd, cid) into the sorted top list (rd, rid) of size K, by one
// warp, in shared memory.  The list's id words may carry flag bits outside `idmask`; flags
// travel with their entries, inserted entries carry none.  Equivalent to inserting the
// candidates one by one with a bounded insertion sort (_kernels.py:490-501): candidates that
// do not beat the tail are dropped, the rest land at j + #{R < C[j]} and R[i] moves to
// i + #{C < R[i]}.  cpos is scratch of >= c ints; cd/cid must hold next_pow2(c) slots.
// Returns the lowest position that received a new entry, or K if none did.  `presorted`:
// the candidates already come in list order (the filter keeps their order).
// U: list chunks of 32 moved per round trip (all loaded before any is stored: targets never
// precede sources, so a store cannot clobber an entry not yet loaded); U > 1 for lists in
// global memory, where each round trip is an L1/L2 latency.
template <class Less = PlainOrder, int U = 1>
SB_DEV int warp_merge_topk(double* rd, uint32_t* rid, int K, double* cd, uint32_t* cid,
                           int* cpos, int c, uint32_t idmask, Less lt = Less(),
                           bool presorted = false) {
  const int lane = lane_id();
  const double wd = rd[K - 1];
  const uint32_t wi = rid[K - 1] & idmask;
  int kept = 0;
  for (int base = 0; base < c; base += 32) {
    int i = base + lane;
    double d = 0.0;
    uint32_t id = 0;
    bool ok = false;
    if (i < c) {
      d = cd[i];
      id = cid[i];
      ok = lt(d, id & idmask, wd, wi);
    }
    unsigned bal = __ballot_sync(0xffffffffu, ok);
    __syncwarp();
    if (ok) {
      int pos = kept + __popc(bal & ((1u << lane) - 1u));
      cd[pos] = d;
      cid[pos] = id;
    }
    kept += __popc(bal);
    __syncwarp();
  }
  if (kept == 0) return K;
  if (!presorted) {
    int np = next_pow2(kept);
    for (int i = kept + lane; i < np; i += 32) {
      cd[i] = __longlong_as_double(0x7FF0000000000000ll);
      cid[i] = 0xFFFFFFFFu;
    }
    __syncwarp();
    warp_bitonic_did(cd, cid, np, MaskedOrder<Less>{lt, idmask});
  }
  for (int j = lane; j < kept; j += 32) {
    double d = cd[j];
    uint32_t id = cid[j] & idmask;
    int lo = 0, hi = K;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (lt(rd[mid], rid[mid] & idmask, d, id)) lo = mid + 1; else hi = mid;
    }
    cpos[j] = j + lo;
  }
  __syncwarp();
  const int first_ins = cpos[0];
  if (first_ins >= K) return K;
  // move list entries at or after first_ins back to front; targets never precede sources.
  // R[i] moves by #{j : lo_j <= i}, lo_j = cpos[j] - j (nondecreasing): jc counts the
  // candidates with lo_j <= top, and the few with lo_j inside the chunk are subtracted per lane
  int jc = kept;
  for (int top0 = K - 1; top0 >= first_ins; top0 -= 32 * U) {
    double d[U];
    uint32_t idw[U];
    int tgt[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int top = top0 - 32 * u;
      const int i = top - lane;
      tgt[u] = K;
      d[u] = 0.0;
      idw[u] = 0;
      if (top < first_ins) continue;
      while (jc > 0 && cpos[jc - 1] - (jc - 1) > top) --jc;
      if (i >= first_ins) {
        d[u] = rd[i];
        idw[u] = rid[i];
        int sh = jc;
        for (int j = jc - 1; j >= 0; --j) {
          const int loj = cpos[j] - j;
          if (loj <= top - 32) break;
          sh -= loj > i;
        }
        tgt[u] = i + sh;
      }
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (tgt[u] < K) {
        rd[tgt[u]] = d[u];
        rid[tgt[u]] = idw[u];
      }
    __syncwarp();
  }
  for (int j = lane; j < kept; j += 32) {
    int p = cpos[j];
    if (p < K) {
      rd[p] = cd[j];
      rid[p] = cid[j];
    }
  }
  __syncwarp();
  return first_ins;
}

// warp_merge_topk for at most 32 candidates, without sorting them in shared memory: each
// candidate stays in a lane, finds its insertion index lo into R by binary search and its rank
// among the candidates by one round of shuffles (keys are distinct: ids are), so it lands at
// lo + rank; R[i] moves by #{candidates with lo <= i}, a 5-step search over the candidates' lo
// values sorted by rank.  Same result as warp_merge_topk.  `ok`, (d, id): this lane's
// candidate (ok = beats R's tail); slo: 32 ints of scratch.  Returns the lowest position that
// received a new entry, or K.
template <class Less>
SB_DEV int warp_merge_lanes(double* rd, uint32_t* rid, int K, bool ok, double d, uint32_t id,
                            uint32_t idmask, int* slo, Less lt) {
  const int lane = lane_id();
  const unsigned bal = __ballot_sync(0xffffffffu, ok);
  if (!bal) return K;
  const int kept = __popc(bal);
  const uint32_t idk = id & idmask;
  int lo = 0;
  if (ok) {
    int hi = K;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (lt(rd[mid], rid[mid] & idmask, d, idk)) lo = mid + 1; else hi = mid;
    }
  }
  // rank among the candidates: lo_k < lo_j orders k first; equal lo compares keys
  int rank = 0;
  unsigned rem = bal;
  while (rem) {
    const int src = __ffs(rem) - 1;
    rem &= rem - 1u;
    const double dk = __shfl_sync(0xffffffffu, d, src);
    const uint32_t ik = __shfl_sync(0xffffffffu, idk, src);
    const int lk = __shfl_sync(0xffffffffu, lo, src);
    if (ok && src != lane) rank += (lk < lo) || (lk == lo && lt(dk, ik, d, idk));
  }
  if (ok) slo[rank] = lo;
  int first = ok ? lo : K;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
  __syncwarp();
  if (first >= K) return K;
  // move R entries at or after `first`, highest first (targets never precede sources)
  for (int top = K - 1; top >= first; top -= 32) {
    const int i = top - lane;
    const bool act = i >= first;
    double di = 0.0;
    uint32_t wi = 0;
    int tgt = K;
    if (act) {
      di = rd[i];
      wi = rid[i];
      int a = 0, b = kept;  // #{j : slo[j] <= i}
      while (a < b) {
        const int mid = (a + b) >> 1;
        if (slo[mid] <= i) a = mid + 1; else b = mid;
      }
      tgt = i + a;
    }
    __syncwarp();
    if (act && tgt < K) {
      rd[tgt] = di;
      rid[tgt] = wi;
    }
    __syncwarp();
  }
  const int pos = lo + rank;
  if (ok && pos < K) {
    rd[pos] = d;
    rid[pos] = id;
  }
  __syncwarp();
  return first;
}

// number of elements of sorted u64 array s[0..n) strictly less than x
SB_DEV int lower_bound_u64(const uint64_t* s, int n, uint64_t x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (s[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// NumPy's pairwise sum of squared differences (x_v - q)^2 for one pair (the order
// evaluate.py:48's (diff*diff).sum(axis=1) uses): 8-way unrolled blocks of <= 128 elements,
// halves (rounded down to a multiple of 8) above that.
static __device__ __noinline__ double np_pairwise_sq(const float* x, const double* q, int n) {
  if (n > 128) {
    int n2 = n / 2;
    n2 -= n2 % 8;
    return dadd(np_pairwise_sq(x, q, n2), np_pairwise_sq(x + n2, q + n2, n - n2));
  }
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) {
      double d = dsub((double)x[i], q[i]);
      res = dadd(res, dmul(d, d));
    }
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    double d = dsub((double)x[j], q[j]);
    r[j] = dmul(d, d);
  }
  int i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double d = dsub((double)x[i + j], q[i + j]);
      r[j] = dadd(r[j], dmul(d, d));
    }
  double res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])), dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
  for (; i < n; ++i) {
    double d = dsub((double)x[i], q[i]);
    res = dadd(res, dmul(d, d));
  }
  return res;
}

}  // namespace sb

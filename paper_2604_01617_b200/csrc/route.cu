// route.cu — batched Dynamic Heterogeneity Routing (reference _kernels.py:504-610,
// router.py:48-124) and device entry points (router.py:42-45).
//
// One warp per query, persistent grid (one warp = one visited-bitset slot).
//
// * Result list R (K entries) lives in shared memory as parallel arrays dist f64 / id u32,
//   sorted by (dist, id).  Two flag bits ride in the id word: bit 31 = "checked" for the
//   phase-2 walk, bit 30 = "checked" for the phase-1 pioneer walk.
// * The pioneer list P needs no storage: P is always the first P entries of R.  (P starts as
//   R[:P]; both are top lists of the same evaluated set, so top-P(P ∪ c) = top-P(R ∪ c).)
// * An expansion evaluates every unvisited neighbour as one batch and then merges the batch
//   into R.  Sequential bounded insertion into a strictly ordered list equals top-K of the
//   union (evicted entries can never return), so ids, distances and all four SearchStats
//   counters equal the reference's.
// * Distances: one neighbour row per lane, fp64, ascending dimension order, explicitly
//   rounded ops — bit-identical to _query_dist (_kernels.py:26-35).  Rows are gathered
//   with 128-bit loads, 8 in flight per lane.
// * Visited set: exact, one bitset of ceil(n/32) words per warp slot in HBM, set with
//   atomicOr (test-and-set); cleared after each query from a per-slot log of visited ids
//   (a full clear when the log overflows).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "rng.cuh"
#include "sb_internal.h"

namespace sb {

constexpr uint32_t kChkR = 0x80000000u;   // phase-2 checked
constexpr uint32_t kChkP = 0x40000000u;   // phase-1 (pioneer) checked
constexpr uint32_t kIdMask = 0x3FFFFFFFu;

// exact fp64 AUTO distance of node v against the query held in shared memory
__device__ __noinline__ double query_dist(const RouteArgs& a, int64_t v, const double* qs, const double* qas,
                         const double* qms) {
  const float* x = a.F + v * (int64_t)a.m;
  double s = 0.0;
  int t = 0;
  if ((a.m & 3) == 0) {
    const float4* vx = reinterpret_cast<const float4*>(x);
    int nq = a.m >> 2;
    int qq = 0;
    for (; qq + 8 <= nq; qq += 8) {
      float4 r[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) r[u] = __ldg(vx + qq + u);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double* qv = qs + 4 * (qq + u);
        s = sq_step(s, r[u].x, qv[0]);
        s = sq_step(s, r[u].y, qv[1]);
        s = sq_step(s, r[u].z, qv[2]);
        s = sq_step(s, r[u].w, qv[3]);
      }
    }
    for (; qq < nq; ++qq) {
      float4 r = __ldg(vx + qq);
      const double* qv = qs + 4 * qq;
      s = sq_step(s, r.x, qv[0]);
      s = sq_step(s, r.y, qv[1]);
      s = sq_step(s, r.z, qv[2]);
      s = sq_step(s, r.w, qv[3]);
    }
    t = a.m;
  }
  for (; t < a.m; ++t) s = sq_step(s, __ldg(x + t), qs[t]);
  const int32_t* av = a.A + v * (int64_t)a.l;
  double sa = 0.0;
  for (int u = 0; u < a.l; ++u)
    sa = dadd(sa, dmul(qms[u], fabs(dsub((double)__ldg(av + u), qas[u]))));
  return auto_finish(s, sa, a.inv_alpha);
}

// Order-free exact distances for a batch of rows (ids in cid[0..c) -> cd).  Valid only when
// every (x - q)^2 term and every partial sum is an integer below 2^53, so fp64 addition is
// exact in any order and the result equals the sequential one bit for bit.  lpr lanes share
// a row (128-bit loads, coalesced), kRows rows per lane group in flight, xor-shuffle reduce.
constexpr int kRows = 4;
__device__ __noinline__ void batch_dist_warp(const RouteArgs& a, const uint32_t* cid, double* cd, int c,
                            const double* qs, const double* qas, const double* qms) {
  const int lane = lane_id();
  const int lpr = a.lpr;
  const int rpp = 32 / lpr;
  const int sub = lane & (lpr - 1);
  const int grp = lane / lpr;
  const int nq = a.m >> 2;
  const float4* F4 = reinterpret_cast<const float4*>(a.F);
  for (int base = 0; base < c; base += rpp * kRows) {
    double part[kRows];
    uint32_t rid[kRows];
#pragma unroll
    for (int g = 0; g < kRows; ++g) {
      int r = base + grp + rpp * g;
      rid[g] = r < c ? cid[r] : 0xFFFFFFFFu;
      part[g] = 0.0;
    }
    for (int k = sub; k < nq; k += lpr) {
      float4 x[kRows];
#pragma unroll
      for (int g = 0; g < kRows; ++g)
        if (rid[g] != 0xFFFFFFFFu) x[g] = __ldg(F4 + (int64_t)rid[g] * nq + k);
      const double* qv = qs + 4 * k;
      const double q0 = qv[0], q1 = qv[1], q2 = qv[2], q3 = qv[3];
#pragma unroll
      for (int g = 0; g < kRows; ++g)
        if (rid[g] != 0xFFFFFFFFu) {
          double d0 = dsub(x[g].x, q0), d1 = dsub(x[g].y, q1);
          double d2 = dsub(x[g].z, q2), d3 = dsub(x[g].w, q3);
          part[g] = dadd(part[g], dadd(dadd(dmul(d0, d0), dmul(d1, d1)), dadd(dmul(d2, d2), dmul(d3, d3))));
        }
    }
#pragma unroll
    for (int g = 0; g < kRows; ++g)
      for (int o = lpr >> 1; o > 0; o >>= 1) part[g] = dadd(part[g], __shfl_xor_sync(0xffffffffu, part[g], o));
    if (sub == 0) {
#pragma unroll
      for (int g = 0; g < kRows; ++g) {
        int r = base + grp + rpp * g;
        if (r < c) {
          const int32_t* av = a.A + (int64_t)cid[r] * a.l;
          double sa = 0.0;
          for (int u = 0; u < a.l; ++u)
            sa = dadd(sa, dmul(qms[u], fabs(dsub((double)__ldg(av + u), qas[u]))));
          cd[r] = auto_finish(part[g], sa, a.inv_alpha);
        }
      }
    }
  }
}

struct WarpSmem {
  double* rd;     // Kpad
  uint32_t* rid;  // Kpad
  double* cd;     // Cpad
  uint32_t* cid;  // Cpad
  int* cpos;      // Cpad
  double* qs;     // m
  double* qas;    // l
  double* qms;    // l
};

SB_HD size_t route_warp_smem_bytes(int Kpad, int Cpad, int m, int l) {
  size_t b = (size_t)Kpad * 8 + (size_t)Cpad * 8 + (size_t)m * 8 + (size_t)l * 16;  // doubles
  b += (size_t)Kpad * 4 + (size_t)Cpad * 8;                                          // u32/int
  return (b + 15) & ~(size_t)15;
}

SB_DEV WarpSmem carve(char* base, int Kpad, int Cpad, int m, int l) {
  WarpSmem w;
  double* dp = reinterpret_cast<double*>(base);
  w.rd = dp; dp += Kpad;
  w.cd = dp; dp += Cpad;
  w.qs = dp; dp += m;
  w.qas = dp; dp += l;
  w.qms = dp; dp += l;
  uint32_t* up = reinterpret_cast<uint32_t*>(dp);
  w.rid = up; up += Kpad;
  w.cid = up; up += Cpad;
  w.cpos = reinterpret_cast<int*>(up);
  return w;
}

// first position in [lb, hi) whose id word lacks `bit`; -1 if none
SB_DEV int first_unchecked(const uint32_t* rid, int lb, int hi, uint32_t bit) {
  for (int base = lb; base < hi; base += 32) {
    int i = base + lane_id();
    bool un = i < hi && !(rid[i] & bit);
    unsigned bal = __ballot_sync(0xffffffffu, un);
    if (bal) return base + __ffs(bal) - 1;
  }
  return -1;
}

// Merge the c candidates in (cd, cid) into R (size K); see warp_merge_topk.
SB_DEV int merge_into_r(WarpSmem& w, int K, int c) {
  return warp_merge_topk(w.rd, w.rid, K, w.cd, w.cid, w.cpos, c, kIdMask);
}

struct Counters {
  int64_t evals, p1_evals, p1_exp, hops, scanned;
};

// Expand `node` over its first `cnt` stored neighbours: test-and-set the visited bits,
// evaluate the unvisited ones, merge into R.  Returns min insert position (or K).
__device__ __noinline__ int expand(const RouteArgs& a, WarpSmem& w, int64_t node, int cnt, uint32_t* vis,
                  uint32_t* vlog, int& logn, int64_t& evals_out, bool fast) {
  const int lane = lane_id();
  const int32_t* nb = a.nbr_ids + node * (int64_t)a.g;
  // gather unvisited neighbours into the candidate buffer (ids only)
  int c = 0;
  for (int base = 0; base < cnt; base += 32) {
    int t = base + lane;
    bool fresh = false;
    uint32_t v = 0;
    if (t < cnt) {
      v = (uint32_t)__ldg(nb + t);
      uint32_t bit = 1u << (v & 31);
      uint32_t old = atomicOr(vis + (v >> 5), bit);
      fresh = !(old & bit);
    }
    unsigned bal = __ballot_sync(0xffffffffu, fresh);
    if (fresh) {
      int pos = c + __popc(bal & ((1u << lane) - 1u));
      w.cid[pos] = v;
      int lp = logn + pos;
      if (lp < a.logcap) vlog[lp] = v;
    }
    c += __popc(bal);
  }
  logn += c;
  evals_out += c;
  __syncwarp();
  // evaluate: warp-split rows (order-free exact mode) or one row per lane, sequential order
  if (fast) {
    batch_dist_warp(a, w.cid, w.cd, c, w.qs, w.qas, w.qms);
  } else {
    for (int j = lane; j < c; j += 32) w.cd[j] = query_dist(a, w.cid[j], w.qs, w.qas, w.qms);
  }
  __syncwarp();
  if (c == 0) return a.K;
  return merge_into_r(w, a.K, c);
}

// 256 threads x 3 CTAs per SM (<= 85 registers per thread, 24 warps resident)
__global__ void __launch_bounds__(256, 3) route_kernel(RouteArgs a) {
  extern __shared__ __align__(16) char smem_raw[];
  const int lane = lane_id();
  const int wid = warp_id();
  const int nw = blockDim.x >> 5;
  const size_t wbytes = route_warp_smem_bytes(a.Kpad, a.Cpad, a.m, a.l);
  WarpSmem w = carve(smem_raw + wbytes * wid, a.Kpad, a.Cpad, a.m, a.l);
  const int64_t slot = (int64_t)blockIdx.x * nw + wid;
  uint32_t* vis = a.visited + slot * a.vwords;
  uint32_t* vlog = a.vlog + slot * (int64_t)a.logcap;
  const int K = a.K;

  for (;;) {
    int qi = 0;
    if (lane == 0) qi = atomicAdd(a.counter, 1);
    qi = __shfl_sync(0xffffffffu, qi, 0);
    if (qi >= a.q) break;

    for (int t = lane; t < a.m; t += 32) w.qs[t] = a.qf[(int64_t)qi * a.m + t];
    for (int t = lane; t < a.l; t += 32) {
      w.qas[t] = a.qa[(int64_t)qi * a.l + t];
      w.qms[t] = a.qm ? a.qm[(int64_t)qi * a.l + t] : 1.0;
    }
    __syncwarp();
    // order-free exact mode for this query: integral coordinates, sums below 2^53
    bool fast = false;
    if (a.int_exact) {
      bool integral = true;
      double qmax = 0.0;
      for (int t = lane; t < a.m; t += 32) {
        double v = w.qs[t];
        integral = integral && v == rint(v);
        qmax = fmax(qmax, fabs(v));
      }
      for (int o = 16; o > 0; o >>= 1) qmax = fmax(qmax, __shfl_xor_sync(0xffffffffu, qmax, o));
      integral = __all_sync(0xffffffffu, integral);
      double lim = (a.fmax + qmax) * (a.fmax + qmax) * (double)a.m;
      fast = integral && lim < 9007199254740992.0;  // 2^53
    }

    Counters ct = {0, 0, 0, 0, 0};
    int logn = 0;
    // entries: mark visited, evaluate, sort (_kernels.py:535-551)
    const int64_t* ent = a.entries + (int64_t)qi * K;
    for (int t = lane; t < K; t += 32) {
      uint32_t v = (uint32_t)ent[t];
      atomicOr(vis + (v >> 5), 1u << (v & 31));
      if (t < a.logcap) vlog[t] = v;
      w.rid[t] = v;
    }
    __syncwarp();
    if (fast) {
      batch_dist_warp(a, w.rid, w.rd, K, w.qs, w.qas, w.qms);
    } else {
      for (int t = lane; t < K; t += 32) w.rd[t] = query_dist(a, w.rid[t], w.qs, w.qas, w.qms);
    }
    __syncwarp();
    for (int t = K + lane; t < a.Kpad; t += 32) {
      w.rd[t] = __longlong_as_double(0x7FF0000000000000ll);
      w.rid[t] = 0xFFFFFFFFu;
    }
    logn = K;
    ct.evals = K;
    __syncwarp();
    if (a.Kpad > 1) warp_bitonic_did(w.rd, w.rid, a.Kpad);

    // phase 1: pioneer walk over R[:P], expanding ceil(deg/2) neighbours (_kernels.py:556-585)
    if (a.use_coarse) {
      int lb = 0;
      for (;;) {
        int sel = first_unchecked(w.rid, lb, a.P, kChkP);
        if (sel < 0) break;
        uint32_t node = w.rid[sel] & kIdMask;
        __syncwarp();
        if (lane == 0) w.rid[sel] |= kChkP;
        __syncwarp();
        ct.p1_exp += 1;
        int deg = __ldg(a.nbr_counts + node);
        int half = (deg + 1) >> 1;
        ct.scanned += half;
        int64_t before = ct.evals;
        int ins = expand(a, w, node, half, vis, vlog, logn, ct.evals, fast);
        ct.p1_evals += ct.evals - before;
        lb = sel + 1;
        if (ins < lb) lb = ins;
      }
    }
    // phase 2: clear checked flags, greedy walk over R (_kernels.py:587-609)
    for (int t = lane; t < K; t += 32) w.rid[t] &= ~kChkR;
    __syncwarp();
    {
      int lb = 0;
      for (;;) {
        int sel = first_unchecked(w.rid, lb, K, kChkR);
        if (sel < 0) break;
        uint32_t node = w.rid[sel] & kIdMask;
        __syncwarp();
        if (lane == 0) w.rid[sel] |= kChkR;
        __syncwarp();
        ct.hops += 1;
        int deg = __ldg(a.nbr_counts + node);
        ct.scanned += deg;
        int ins = expand(a, w, node, deg, vis, vlog, logn, ct.evals, fast);
        lb = sel + 1;
        if (ins < lb) lb = ins;
      }
    }
    // results
    for (int t = lane; t < K; t += 32) {
      a.out_ids[(int64_t)qi * K + t] = (int64_t)(w.rid[t] & kIdMask);
      a.out_dists[(int64_t)qi * K + t] = w.rd[t];
    }
    if (a.stats && lane == 0) {
      int64_t* st = a.stats + (int64_t)qi * 5;
      st[0] = ct.evals;
      st[1] = ct.p1_evals;
      st[2] = ct.p1_exp;
      st[3] = ct.hops;
      st[4] = ct.scanned;
    }
    // clear the visited bits this query set
    if (logn <= a.logcap) {
      for (int t = lane; t < logn; t += 32) vis[vlog[t] >> 5] = 0u;
    } else {
      for (int64_t t = lane; t < a.vwords; t += 32) vis[t] = 0u;
    }
    __syncwarp();
  }
}

// one thread per query: entry_points(n, K, seed, qi0 + i) into out (q x K)
__global__ void entry_points_kernel(int64_t n, int K, uint64_t seed, int64_t qi0, int64_t q,
                                    int64_t* out, int64_t* scratch, uint64_t scratch_slots) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= q) return;
  sbrng::entry_points(n, K, seed, (uint64_t)(qi0 + i), out + i * K, scratch + i * scratch_slots);
}

int launch_entry_points(int64_t n, int K, uint64_t seed, int64_t qi0, int64_t q, int64_t* out,
                        int64_t* scratch, uint64_t scratch_slots, cudaStream_t st) {
  int bs = 128;
  int64_t gb = (q + bs - 1) / bs;
  if (gb > 0) entry_points_kernel<<<(unsigned)gb, bs, 0, st>>>(n, K, seed, qi0, q, out, scratch,
                                                               scratch_slots);
  return (int)cudaGetLastError();
}

size_t route_smem_per_warp(int Kpad, int Cpad, int m, int l) {
  return route_warp_smem_bytes(Kpad, Cpad, m, l);
}

int launch_route(const RouteArgs& a, int warps_per_cta, int ctas, cudaStream_t st) {
  size_t smem = route_warp_smem_bytes(a.Kpad, a.Cpad, a.m, a.l) * warps_per_cta;
  cudaError_t e = cudaFuncSetAttribute(route_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return (int)e;
  route_kernel<<<ctas, warps_per_cta * 32, smem, st>>>(a);
  return (int)cudaGetLastError();
}

int route_occupancy(int warps_per_cta, size_t smem, int* ctas_per_sm) {
  cudaError_t e = cudaFuncSetAttribute(route_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, route_kernel,
                                                            warps_per_cta * 32, smem);
}

}  // namespace sb

namespace sb {

// index property for the order-free exact mode: are all features integral, and max |x|
__global__ void feature_scan_kernel(const float* F, int64_t count, unsigned* nonint,
                                    unsigned* maxbits) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool bad = false;
  float mx = 0.f;
  for (; i < count; i += stride) {
    float v = F[i];
    bad = bad || v != rintf(v) || !isfinite(v);
    mx = fmaxf(mx, fabsf(v));
  }
  if (__any_sync(0xffffffffu, bad) && lane_id() == 0) atomicOr(nonint, 1u);
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane_id() == 0) atomicMax(maxbits, __float_as_uint(mx));
}

int launch_feature_scan(const float* F, int64_t count, unsigned* nonint, unsigned* maxbits,
                        cudaStream_t st) {
  cudaMemsetAsync(nonint, 0, sizeof(unsigned), st);
  cudaMemsetAsync(maxbits, 0, sizeof(unsigned), st);
  feature_scan_kernel<<<1184, 256, 0, st>>>(F, count, nonint, maxbits);
  return (int)cudaGetLastError();
}

}  // namespace sb

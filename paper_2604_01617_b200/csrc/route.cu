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
// * Memory round trips per expansion are the bound (each query is a serial walk), so each
//   step issues everything it can at once: the neighbour count and the whole id row load
//   together; all visited test-and-sets go out together; a few lanes share each unvisited
//   row so that the whole row is in flight at once (eval_rows).
// * Distances: fp64, ascending dimension order, explicitly rounded operations, the running
//   sum handed lane to lane — bit-identical to _query_dist (_kernels.py:26-35) for any data.
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

// ---- fallback when rows are not 16-byte aligned (m % 4 != 0): lane-owned global reads ---
__device__ __noinline__ double query_dist_global(const RouteArgs& a, int64_t v, const double* qs,
                                                 const double* qas, const double* qms) {
  const float* x = a.F + v * (int64_t)a.m;
  double s = 0.0;
  for (int t = 0; t < a.m; ++t) s = sq_step(s, __ldg(x + t), qs[t]);
  const int32_t* av = a.A + v * (int64_t)a.l;
  double sa = 0.0;
  for (int u = 0; u < a.l; ++u)
    sa = dadd(sa, dmul(qms[u], fabs(dsub((double)__ldg(av + u), qas[u]))));
  return auto_finish(s, sa, a.inv_alpha);
}

struct WarpSmem {
  double* rd;     // Kpad
  double* cd;     // Cpad
  double* qs;     // m
  double* qas;    // l
  double* qms;    // l
  uint32_t* rid;  // Kpad
  uint32_t* cid;  // Cpad
  int* cpos;      // Cpad
};

SB_HD size_t route_warp_smem_bytes_full(int Kpad, int Cpad, int m, int l) {
  size_t b = (size_t)Kpad * 8 + (size_t)Cpad * 8 + (size_t)m * 8 + (size_t)l * 16;
  b += (size_t)Kpad * 4 + (size_t)Cpad * 8;
  return (b + 15) & ~(size_t)15;
}

SB_DEV WarpSmem carve(char* base, const RouteArgs& a) {
  WarpSmem w;
  double* dp = reinterpret_cast<double*>(base);
  w.rd = dp; dp += a.Kpad;
  w.cd = dp; dp += a.Cpad;
  w.qs = dp; dp += a.m;
  w.qas = dp; dp += a.l;
  w.qms = dp; dp += a.l;
  uint32_t* up = reinterpret_cast<uint32_t*>(dp);
  w.rid = up; up += a.Kpad;
  w.cid = up; up += a.Cpad;
  w.cpos = reinterpret_cast<int*>(up);
  return w;
}

// Exact distances of rows ids[0..c) -> out[0..c).  `lpr` lanes share a row: lane q of the
// group loads float4s [q*per, (q+1)*per) of the row up front (so a 128-d row arrives in one
// memory round trip), then the groups' lanes take turns extending the fp64 sum in ascending
// dimension order, handing the running sum on with a shuffle — the sequential order of
// _query_dist (_kernels.py:26-35), bit for bit.
constexpr int kVec = 8;  // float4s a lane keeps in flight
SB_DEV void eval_rows(const RouteArgs& a, WarpSmem& w, const uint32_t* ids, double* out, int c) {
  const int lane = lane_id();
  if (a.lpr == 0) {
    for (int j = lane; j < c; j += 32) out[j] = query_dist_global(a, ids[j], w.qs, w.qas, w.qms);
    __syncwarp();
    return;
  }
  const int lpr = a.lpr;
  const int q = lane & (lpr - 1);
  const int gbase = lane & ~(lpr - 1);
  const int rows_pp = 32 / lpr;
  const int nq = a.m >> 2;
  const int per = (nq + lpr - 1) / lpr;
  const int f0 = q * per;
  const int f1 = f0 + per < nq ? f0 + per : nq;
  const float4* F4 = reinterpret_cast<const float4*>(a.F);
  for (int base = 0; base < c; base += rows_pp) {
    const int r = base + lane / lpr;
    const bool valid = r < c;
    const float4* row = F4 + (int64_t)(valid ? ids[r] : 0) * nq;
    float4 x[kVec];
#pragma unroll
    for (int k = 0; k < kVec; ++k)
      if (valid && f0 + k < f1) x[k] = __ldg(row + f0 + k);
    double s = 0.0;
    for (int step = 0; step < lpr; ++step) {
      if (q == step && valid) {
#pragma unroll
        for (int k = 0; k < kVec; ++k)
          if (f0 + k < f1) {
            const double* qv = w.qs + 4 * (f0 + k);
            s = sq_step(s, x[k].x, qv[0]);
            s = sq_step(s, x[k].y, qv[1]);
            s = sq_step(s, x[k].z, qv[2]);
            s = sq_step(s, x[k].w, qv[3]);
          }
        for (int f = f0 + kVec; f < f1; f += kVec) {
#pragma unroll
          for (int k = 0; k < kVec; ++k)
            if (f + k < f1) x[k] = __ldg(row + f + k);
#pragma unroll
          for (int k = 0; k < kVec; ++k)
            if (f + k < f1) {
              const double* qv = w.qs + 4 * (f + k);
              s = sq_step(s, x[k].x, qv[0]);
              s = sq_step(s, x[k].y, qv[1]);
              s = sq_step(s, x[k].z, qv[2]);
              s = sq_step(s, x[k].w, qv[3]);
            }
        }
      }
      if (lpr > 1) s = __shfl_sync(0xffffffffu, s, gbase | step);
    }
    if (q == 0 && valid) {
      const int32_t* av = a.A + (int64_t)ids[r] * a.l;
      double sa = 0.0;
      for (int u = 0; u < a.l; ++u)
        sa = dadd(sa, dmul(w.qms[u], fabs(dsub((double)__ldg(av + u), w.qas[u]))));
      out[r] = auto_finish(s, sa, a.inv_alpha);
    }
  }
  __syncwarp();
}

// first (and second) position in [lb, hi) whose id word lacks `bit`; -1 if none
SB_DEV int first_unchecked(const uint32_t* rid, int lb, int hi, uint32_t bit, int* second) {
  *second = -1;
  for (int base = lb; base < hi; base += 32) {
    int i = base + lane_id();
    bool un = i < hi && !(rid[i] & bit);
    unsigned bal = __ballot_sync(0xffffffffu, un);
    if (bal) {
      int f = __ffs(bal) - 1;
      unsigned rest = bal & (bal - 1u);
      if (rest) *second = base + __ffs(rest) - 1;
      return base + f;
    }
  }
  return -1;
}

struct Counters {
  int64_t evals, p1_evals, p1_exp, hops, scanned;
};

// warm L2 with the neighbour row of a node we will probably expand next
SB_DEV void prefetch_row(const RouteArgs& a, uint32_t node) {
  const int lane = lane_id();
  const char* p = reinterpret_cast<const char*>(a.nbr_ids + (int64_t)node * a.g);
  const int bytes = a.g * 4;
  if (lane * 128 < bytes) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + lane * 128));
}

// Expand `node`: read its count and id row together, test-and-set the visited bits of the
// first cnt neighbours (cnt = ceil(deg/2) in phase 1), evaluate the unvisited ones, merge
// into R.  Returns the lowest position that received an entry (or K).
__device__ __noinline__ int expand(const RouteArgs& a, WarpSmem& w, uint32_t node, bool half,
                                   uint32_t* vis, uint32_t* vlog, int& logn, Counters& ct) {
  const int lane = lane_id();
  const int32_t* nb = a.nbr_ids + (int64_t)node * a.g;
  const int deg = __ldg(a.nbr_counts + node);
  int c = 0;
  for (int base = 0; base < a.g; base += 128) {
    // up to 4 ids per lane per pass, loaded before the count is known
    uint32_t v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int t = base + lane + 32 * k;
      v[k] = t < a.g ? (uint32_t)__ldg(nb + t) : 0u;
    }
    const int cnt = half ? (deg + 1) >> 1 : deg;
    if (base >= cnt) break;
    bool fresh[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int t = base + lane + 32 * k;
      fresh[k] = false;
      if (t < cnt) {
        uint32_t bit = 1u << (v[k] & 31);
        uint32_t old = atomicOr(vis + (v[k] >> 5), bit);
        fresh[k] = !(old & bit);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      unsigned bal = __ballot_sync(0xffffffffu, fresh[k]);
      if (fresh[k]) {
        int pos = c + __popc(bal & ((1u << lane) - 1u));
        w.cid[pos] = v[k];
        int lp = logn + pos;
        if (lp < a.logcap) vlog[lp] = v[k];
      }
      c += __popc(bal);
    }
  }
  const int cnt = half ? (deg + 1) >> 1 : deg;
  ct.scanned += cnt;
  logn += c;
  ct.evals += c;
  if (half) ct.p1_evals += c;
  __syncwarp();
  if (c == 0) return a.K;
  eval_rows(a, w, w.cid, w.cd, c);
  return warp_merge_topk(w.rd, w.rid, a.K, w.cd, w.cid, w.cpos, c, kIdMask);
}

// 256 threads x 4 CTAs per SM: <= 64 registers per thread, 32 warps resident
__global__ void __launch_bounds__(256, 4) route_kernel(RouteArgs a) {
  extern __shared__ __align__(16) char smem_raw[];
  const int lane = lane_id();
  const int wid = warp_id();
  const int nw = blockDim.x >> 5;
  const size_t wbytes = route_warp_smem_bytes_full(a.Kpad, a.Cpad, a.m, a.l);
  WarpSmem w = carve(smem_raw + wbytes * wid, a);
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
    eval_rows(a, w, w.rid, w.rd, K);
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
        int nxt;
        int sel = first_unchecked(w.rid, lb, a.P, kChkP, &nxt);
        if (sel < 0) break;
        uint32_t node = w.rid[sel] & kIdMask;
        if (nxt >= 0) prefetch_row(a, w.rid[nxt] & kIdMask);
        __syncwarp();
        if (lane == 0) w.rid[sel] |= kChkP;
        __syncwarp();
        ct.p1_exp += 1;
        int ins = expand(a, w, node, true, vis, vlog, logn, ct);
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
        int nxt;
        int sel = first_unchecked(w.rid, lb, K, kChkR, &nxt);
        if (sel < 0) break;
        uint32_t node = w.rid[sel] & kIdMask;
        if (nxt >= 0) prefetch_row(a, w.rid[nxt] & kIdMask);
        __syncwarp();
        if (lane == 0) w.rid[sel] |= kChkR;
        __syncwarp();
        ct.hops += 1;
        int ins = expand(a, w, node, false, vis, vlog, logn, ct);
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

size_t route_smem_per_warp(const RouteArgs& a) {
  return route_warp_smem_bytes_full(a.Kpad, a.Cpad, a.m, a.l);
}

int launch_route(const RouteArgs& a, int warps_per_cta, int ctas, cudaStream_t st) {
  size_t smem = route_smem_per_warp(a) * warps_per_cta;
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

// index property: are all features integral, and max |x| (used by the exhaustive top-k
// filter to pick an exact low-precision path)
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

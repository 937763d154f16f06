// bf_topk.cu — exhaustive AUTO top-k.
//
// Two modes share one tiled fp64 kernel:
//  * node mode  = brute_force_topk (_kernels.py:176-204): sample node u vs every v != u,
//    fp64 sequential-order _pair_dist, top-k by (d, id), ids padded with -1.  Bit-exact.
//  * query mode = oracle_auto_topk (evaluate.py:32-55): f64 query vs every node; the
//    reference sums squared differences with NumPy's pairwise order and divides s_a by
//    alpha.  The tiled pass ranks in sequential order and keeps k + kExtra candidates per
//    query; the merge kernel recomputes those exactly in NumPy's order (a 1-2 ulp change at
//    most), re-sorts, and certifies that no node outside the kept set could enter the top k.
//
// Tiling: a CTA owns QG queries x a node range; each thread computes a 2 x 4 (query x node)
// register tile of independent fp64 chains over ascending dimensions (node tile staged in
// shared memory transposed [dim][node], queries [dim][query] as f64), dimension chunks of 32.
// Candidates that beat a query's current tail are appended to its shared buffer and merged
// by a warp after each node tile (warp_merge_topk).  Each CTA writes its partial lists; a
// second kernel merges the node-range splits per query.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "sb_internal.h"

namespace sb {

constexpr int kBfThreads = 256;
constexpr int kNT = 64;   // nodes per tile
constexpr int kDC = 32;   // dimensions per chunk
constexpr int kTQ = 2;    // queries per thread
constexpr int kTN = 4;    // nodes per thread
// QG = (kBfThreads / (kNT / kTN)) * kTQ = 16 * 2 = 32 queries per CTA
constexpr int kQG = (kBfThreads / (kNT / kTN)) * kTQ;

struct BfSmem {
  float* xt;        // [kDC][kNT]
  double* qt;       // [kDC][kQG]
  double* ld;       // [kQG][kpad] list dists
  uint32_t* li;     // [kQG][kpad] list ids
  double* bd;       // [kQG][kNT] buffer dists
  uint32_t* bi;     // [kQG][kNT]
  int* bpos;        // [kQG][kNT]
  int* bcnt;        // [kQG]
};

static size_t bf_smem_bytes(int kpad) {
  size_t b = sizeof(float) * kDC * kNT + sizeof(double) * kDC * kQG;
  b += (sizeof(double) + sizeof(uint32_t)) * (size_t)kQG * kpad;
  b += (sizeof(double) + sizeof(uint32_t) + sizeof(int)) * (size_t)kQG * kNT;
  b += sizeof(int) * kQG;
  return b + 64;
}

__global__ void __launch_bounds__(kBfThreads) bf_partial_kernel(BfArgs a, int kk, int kpad) {
  extern __shared__ __align__(16) char smem_raw[];
  BfSmem s;
  {
    char* p = smem_raw;
    s.qt = reinterpret_cast<double*>(p); p += sizeof(double) * kDC * kQG;
    s.ld = reinterpret_cast<double*>(p); p += sizeof(double) * (size_t)kQG * kpad;
    s.bd = reinterpret_cast<double*>(p); p += sizeof(double) * (size_t)kQG * kNT;
    s.xt = reinterpret_cast<float*>(p); p += sizeof(float) * kDC * kNT;
    s.li = reinterpret_cast<uint32_t*>(p); p += sizeof(uint32_t) * (size_t)kQG * kpad;
    s.bi = reinterpret_cast<uint32_t*>(p); p += sizeof(uint32_t) * (size_t)kQG * kNT;
    s.bpos = reinterpret_cast<int*>(p); p += sizeof(int) * (size_t)kQG * kNT;
    s.bcnt = reinterpret_cast<int*>(p);
  }
  const int tid = threadIdx.x;
  const int tn = tid % (kNT / kTN);   // 0..15
  const int tq = tid / (kNT / kTN);   // 0..15
  const int64_t q0 = (int64_t)blockIdx.x * kQG;
  const int split = blockIdx.y;
  const int64_t per = (a.n + a.splits - 1) / a.splits;
  const int64_t v_begin = per * split;
  const int64_t v_end = v_begin + per < a.n ? v_begin + per : a.n;
  const bool node_mode = a.self_ids != nullptr;
  const double inf = __longlong_as_double(0x7FF0000000000000ll);

  for (int i = tid; i < kQG * kpad; i += kBfThreads) {
    s.ld[i] = inf;
    s.li[i] = 0xFFFFFFFFu;
  }
  for (int i = tid; i < kQG; i += kBfThreads) s.bcnt[i] = 0;

  // per-thread query ids / attribute pointers
  int64_t qid[kTQ];
  bool qok[kTQ];
#pragma unroll
  for (int u = 0; u < kTQ; ++u) {
    int64_t qq = q0 + tq * kTQ + u;
    qok[u] = qq < a.q;
    qid[u] = qok[u] ? qq : 0;
  }
  __syncthreads();

  for (int64_t vb = v_begin; vb < v_end; vb += kNT) {
    double acc[kTQ][kTN];
#pragma unroll
    for (int u = 0; u < kTQ; ++u)
#pragma unroll
      for (int w = 0; w < kTN; ++w) acc[u][w] = 0.0;

    for (int d0 = 0; d0 < a.m; d0 += kDC) {
      const int dc = a.m - d0 < kDC ? a.m - d0 : kDC;
      __syncthreads();
      // stage node tile (transposed) and query tile
      for (int i = tid; i < kNT * kDC; i += kBfThreads) {
        int node = i / kDC, dd = i % kDC;
        int64_t v = vb + node;
        float x = 0.f;
        if (v < v_end && dd < dc) x = __ldg(a.F + v * (int64_t)a.m + d0 + dd);
        s.xt[dd * kNT + node] = x;
      }
      for (int i = tid; i < kQG * kDC; i += kBfThreads) {
        int qq = i / kDC, dd = i % kDC;
        int64_t g = q0 + qq;
        double x = 0.0;
        if (g < a.q && dd < dc) {
          if (node_mode) x = (double)__ldg(a.F + a.self_ids[g] * (int64_t)a.m + d0 + dd);
          else x = a.qf[g * (int64_t)a.m + d0 + dd];
        }
        s.qt[dd * kQG + qq] = x;
      }
      __syncthreads();
      for (int dd = 0; dd < dc; ++dd) {
        float4 xv = *reinterpret_cast<const float4*>(s.xt + dd * kNT + tn * kTN);
        double2 qv = *reinterpret_cast<const double2*>(s.qt + dd * kQG + tq * kTQ);
        const double qx[2] = {qv.x, qv.y};
        const double nx[4] = {(double)xv.x, (double)xv.y, (double)xv.z, (double)xv.w};
#pragma unroll
        for (int u = 0; u < kTQ; ++u)
#pragma unroll
          for (int w = 0; w < kTN; ++w) {
            // node mode: (x_u - x_v)^2 exactly as _pair_dist(u, v); query mode: (x_v - q)^2
            double diff = node_mode ? dsub(qx[u], nx[w]) : dsub(nx[w], qx[u]);
            acc[u][w] = dadd(acc[u][w], dmul(diff, diff));
          }
      }
    }
    // finish distances, append candidates that beat the current tail
#pragma unroll
    for (int u = 0; u < kTQ; ++u) {
      if (!qok[u]) continue;
      const int ql = tq * kTQ + u;
      const double wd = s.ld[ql * kpad + kk - 1];
      const uint32_t wi = s.li[ql * kpad + kk - 1];
#pragma unroll
      for (int w = 0; w < kTN; ++w) {
        int64_t v = vb + tn * kTN + w;
        if (v >= v_end) continue;
        double sa;
        double dist;
        if (node_mode) {
          int64_t uu = a.self_ids[qid[u]];
          if (v == uu) continue;
          sa = attr_l1(a.A + uu * (int64_t)a.l, a.A + v * (int64_t)a.l, a.l);
          dist = auto_finish(acc[u][w], sa, a.inv_alpha);
        } else {
          int64_t si = 0;
          for (int t = 0; t < a.l; ++t) {
            int64_t ad = (int64_t)__ldg(a.A + v * (int64_t)a.l + t) - a.qa[qid[u] * a.l + t];
            ad = ad < 0 ? -ad : ad;
            si += a.qmask ? ad * a.qmask[qid[u] * a.l + t] : ad;
          }
          dist = dmul(sqrt(acc[u][w]), dadd(1.0, __ddiv_rn((double)si, a.alpha)));
        }
        if (dlt(dist, (uint32_t)v, wd, wi)) {
          int slot = atomicAdd(s.bcnt + ql, 1);
          s.bd[ql * kNT + slot] = dist;
          s.bi[ql * kNT + slot] = (uint32_t)v;
        }
      }
    }
    __syncthreads();
    // warps merge the buffers into the per-query lists
    for (int ql = warp_id(); ql < kQG; ql += kBfThreads / 32) {
      int c = s.bcnt[ql];
      if (c > 0) {
        warp_merge_topk(s.ld + ql * kpad, s.li + ql * kpad, kk, s.bd + ql * kNT,
                        s.bi + ql * kNT, s.bpos + ql * kNT, c, 0xFFFFFFFFu);
        if (lane_id() == 0) s.bcnt[ql] = 0;
      }
    }
    __syncthreads();
  }
  // write partial lists
  for (int i = tid; i < kQG * kk; i += kBfThreads) {
    int ql = i / kk, t = i % kk;
    int64_t g = q0 + ql;
    if (g >= a.q) continue;
    size_t o = ((size_t)g * a.splits + split) * kk + t;
    a.part_d[o] = s.ld[ql * kpad + t];
    a.part_i[o] = s.li[ql * kpad + t];
  }
}

// merge the splits of each query (warp per query), then (query mode) exact re-rank
__global__ void bf_merge_kernel(BfArgs a, int kk, int kpad, int kout, int64_t* out_ids64,
                                int32_t* out_ids32, double* out_dists, int* uncertain) {
  extern __shared__ __align__(16) char smem_raw[];
  const int wpb = blockDim.x >> 5;
  const int wid = warp_id();
  const int lane = lane_id();
  char* base = smem_raw + (size_t)wid * (kpad * 2 * (sizeof(double) + sizeof(uint32_t)) + kpad * sizeof(int));
  double* ld = reinterpret_cast<double*>(base);
  double* cd = ld + kpad;
  uint32_t* li = reinterpret_cast<uint32_t*>(cd + kpad);
  uint32_t* ci = li + kpad;
  int* cp = reinterpret_cast<int*>(ci + kpad);
  int64_t g = (int64_t)blockIdx.x * wpb + wid;
  if (g >= a.q) return;
  size_t o = (size_t)g * a.splits * kk;
  for (int t = lane; t < kk; t += 32) { ld[t] = a.part_d[o + t]; li[t] = a.part_i[o + t]; }
  __syncwarp();
  for (int sp = 1; sp < a.splits; ++sp) {
    size_t os = o + (size_t)sp * kk;
    for (int t = lane; t < kk; t += 32) { cd[t] = a.part_d[os + t]; ci[t] = a.part_i[os + t]; }
    __syncwarp();
    warp_merge_topk(ld, li, kk, cd, ci, cp, kk, 0xFFFFFFFFu);
  }
  if (a.self_ids) {  // node mode: exact already
    for (int t = lane; t < kout; t += 32)
      out_ids32[g * kout + t] = li[t] == 0xFFFFFFFFu ? -1 : (int32_t)li[t];
    return;
  }
  // query mode: recompute kept candidates in NumPy's summation order, re-sort
  const double* q = a.qf + g * (int64_t)a.m;
  int valid = 0;
  for (int t = 0; t < kk; ++t) valid += li[t] != 0xFFFFFFFFu;
  double last_seq = ld[kk - 1];
  for (int t = lane; t < kk; t += 32) {
    if (li[t] == 0xFFFFFFFFu) { cd[t] = ld[t]; ci[t] = li[t]; continue; }
    int64_t v = li[t];
    double sv = np_pairwise_sq(a.F + v * (int64_t)a.m, q, a.m);
    int64_t si = 0;
    for (int u = 0; u < a.l; ++u) {
      int64_t ad = (int64_t)a.A[v * (int64_t)a.l + u] - a.qa[g * a.l + u];
      ad = ad < 0 ? -ad : ad;
      si += a.qmask ? ad * a.qmask[g * a.l + u] : ad;
    }
    cd[t] = dmul(sqrt(sv), dadd(1.0, __ddiv_rn((double)si, a.alpha)));
    ci[t] = li[t];
  }
  for (int t = kk + lane; t < kpad; t += 32) {
    cd[t] = __longlong_as_double(0x7FF0000000000000ll);
    ci[t] = 0xFFFFFFFFu;
  }
  __syncwarp();
  warp_bitonic_did(cd, ci, kpad);
  for (int t = lane; t < kout; t += 32) {
    out_ids64[g * kout + t] = (int64_t)ci[t];
    out_dists[g * kout + t] = cd[t];
  }
  // certificate: a node outside the kept set has sequential distance >= last_seq; it could
  // only enter the exact top kout if last_seq is within a few ulps of the exact kout-th.
  if (lane == 0 && valid == kk && kk > kout) {
    double dk = cd[kout - 1];
    if (!(last_seq > dk * (1.0 + 1e-12))) atomicAdd(uncertain, 1);
  }
}

int launch_bf_partial(const BfArgs& a, cudaStream_t st) {
  int kpad = next_pow2(a.k);
  size_t smem = bf_smem_bytes(kpad);
  cudaError_t e = cudaFuncSetAttribute(bf_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return (int)e;
  dim3 grid((unsigned)((a.q + kQG - 1) / kQG), (unsigned)a.splits);
  bf_partial_kernel<<<grid, kBfThreads, smem, st>>>(a, a.k, kpad);
  return (int)cudaGetLastError();
}

int bf_group_size() { return kQG; }
size_t bf_partial_smem(int k) { return bf_smem_bytes(next_pow2(k)); }

int launch_bf_merge_k(const BfArgs& a, int kout, int64_t* out_ids64, int32_t* out_ids32,
                      double* out_dists, int* uncertain, cudaStream_t st) {
  int kpad = next_pow2(a.k < 2 ? 2 : a.k);  // even, so every warp's slice stays 8-byte aligned
  int wpb = 4;
  size_t per_warp = (size_t)kpad * 2 * (sizeof(double) + sizeof(uint32_t)) + kpad * sizeof(int);
  size_t smem = per_warp * wpb;
  cudaError_t e = cudaFuncSetAttribute(bf_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return (int)e;
  unsigned grid = (unsigned)((a.q + wpb - 1) / wpb);
  bf_merge_kernel<<<grid, wpb * 32, smem, st>>>(a, a.k, kpad, kout, out_ids64, out_ids32,
                                                out_dists, uncertain);
  return (int)cudaGetLastError();
}

}  // namespace sb

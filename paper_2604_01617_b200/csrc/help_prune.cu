// help_prune.cu — HELP build, part 3: heterogeneous semantic pruning (graph.py:202-232).
//
// prune_pass (_kernels.py:266-303) processes rows in ascending order; the only sequential
// coupling is the in-degree safeguard.  Restated: the safeguard can only fire on
// the edge smax(p) -> p, where smax(p) is p's largest-id in-neighbour, and it fires iff that
// edge is redundant and every other in-edge of p was dropped.  So
//   guard[p] = (#dropped in-edges of p from rows != smax(p)) == indeg0[p] - 1
// and row s drops entry t iff redundant(t | kept entries before t) and not (s == smax(p) and
// guard[p]).  Guards depend only on rows below smax(p), so Jacobi rounds from guard = 0 reach
// the sequential result exactly; the loop stops when no guard changes.
//
//   bits    CTA per row: redundancy matrix R[t][u] (u < t) = attrs_equal(p_t, p_u) and
//           cos(p_t - s, p_u - s) > sigma, cosines in fp64 with the reference's exact
//           operation order (_kernels.py:235-253), 4 x 4 register tiles.
//   scan    thread per row: keep-mask walk under the current guards.
//   guard   thread per node.
//   compact thread per row, order-preserving, stale tails left as the reference leaves them.
//
// reinforce_pass (_kernels.py:398-409) equals symmetrisation when no row j would exceed
// capacity, |row_j ∪ {s : j in row_s}| <= gamma — checked exactly first.  Rows
// then get their missing reverse entries merged in by (f32 dist, id).  Otherwise the exact
// overflow path of help_reinforce.cu runs.  reconnect_islands keeps its sequential order over
// nodes and runs in one CTA (reconnect_cta_kernel below).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "sb_internal.h"

namespace sb {

constexpr int kPruneThreads = 256;
#ifndef PRUNE_F64_THREADS
#define PRUNE_F64_THREADS 256
#endif
constexpr int kPruneThreadsF64 = PRUNE_F64_THREADS;  // fp64 kernel: tiles of a full row per pass
constexpr int kPT = 4;

__global__ void __launch_bounds__(kPruneThreadsF64) prune_bits_kernel(PruneArgs a) {
  extern __shared__ __align__(16) char smem_raw[];
  const int cpad = a.cpad;
  // the float tile goes first: its float4 reads need 16-byte alignment
  char* p = smem_raw;
  float* xr = reinterpret_cast<float*>(p); p += sizeof(float) * (size_t)a.dc * cpad;
  double* xs = reinterpret_cast<double*>(p); p += sizeof(double) * a.m;
  double* nrm = reinterpret_cast<double*>(p); p += sizeof(double) * cpad;
  int32_t* eid = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * cpad;
  int32_t* eat = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * (size_t)cpad * a.l;
  uint32_t* bits = reinterpret_cast<uint32_t*>(p); p += sizeof(uint32_t) * (size_t)cpad * a.W;
  const int64_t s = blockIdx.x;
  const int cnt = a.counts[s];
  if (cnt <= 1) return;
  const int tid = threadIdx.x;
  const bool whole = a.dc >= a.m;
  for (int t = tid; t < a.m; t += blockDim.x) xs[t] = (double)__ldg(a.F + s * a.m + t);
  for (int t = tid; t < cpad; t += blockDim.x) {
    int32_t v = t < cnt ? a.ids[s * a.g + t] : 0;
    eid[t] = v;
    for (int u = 0; u < a.l; ++u) eat[t * a.l + u] = t < cnt ? __ldg(a.A + (int64_t)v * a.l + u) : 0;
  }
  for (int t = tid; t < cpad * a.W; t += blockDim.x) bits[t] = 0u;
  __syncthreads();

  // dimensions [d0, d0 + dc) of every row entry, transposed into [dimension][entry], by 4-byte
  // asynchronous copies: a warp per entry, lanes along the dimensions (coalesced), the whole
  // chunk in flight at once (a load -> store loop waits for one load per thread at a time)
  auto stage = [&](int d0, int dc) {
    const int lane_ = tid & 31, nwarp = blockDim.x >> 5;
    for (int t = tid >> 5; t < cnt; t += nwarp) {
      const float* src = a.F + (int64_t)eid[t] * a.m + d0;
      for (int dd = lane_; dd < dc; dd += 32)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(xr + dd * cpad + t)),
                     "l"(src + dd)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  };
  // norms |p_t - s|^2, sequential over dimensions (np2 / nk2 of _diff_cosine)
  {
    double acc = 0.0;
    for (int d0 = 0; d0 < a.m; d0 += a.dc) {
      const int dc = a.m - d0 < a.dc ? a.m - d0 : a.dc;
      __syncthreads();
      stage(d0, dc);
      __syncthreads();
      if (tid < cnt)
        for (int dd = 0; dd < dc; ++dd) {
          double dp = dsub((double)xr[dd * cpad + tid], xs[d0 + dd]);
          acc = dadd(acc, dmul(dp, dp));
        }
    }
    if (tid < cnt) nrm[tid] = acc;
  }
  __syncthreads();
  // dot products on lower-triangle 4 x 4 tiles (row block tb >= column block ub)
  const int nb = (cnt + kPT - 1) / kPT;
  const int ntiles = nb * (nb + 1) / 2;
  for (int pass = 0; pass * kPruneThreadsF64 < ntiles; ++pass) {
    const int ti = pass * kPruneThreadsF64 + tid;
    const bool have = ti < ntiles;
    int tb = 0, ub = 0;
    if (have) {
      // ti -> (tb, ub) with ub <= tb, row-major over the lower triangle
      tb = (int)((sqrt(8.0 * ti + 1.0) - 1.0) * 0.5);
      while ((tb + 1) * (tb + 2) / 2 <= ti) ++tb;
      while (tb * (tb + 1) / 2 > ti) --tb;
      ub = ti - tb * (tb + 1) / 2;
    }
    double acc[kPT][kPT];
#pragma unroll
    for (int u = 0; u < kPT; ++u)
#pragma unroll
      for (int w = 0; w < kPT; ++w) acc[u][w] = 0.0;
    for (int d0 = 0; d0 < a.m; d0 += a.dc) {
      const int dc = a.m - d0 < a.dc ? a.m - d0 : a.dc;
      if (!whole || pass == 0) {
        __syncthreads();
        stage(d0, dc);
        __syncthreads();
      }
      if (have) {
        for (int dd = 0; dd < dc; ++dd) {
          const float* row = xr + (size_t)dd * cpad;
          const double xsd = xs[d0 + dd];
          float4 tv = *reinterpret_cast<const float4*>(row + tb * kPT);
          float4 uv = *reinterpret_cast<const float4*>(row + ub * kPT);
          const double dt[4] = {dsub((double)tv.x, xsd), dsub((double)tv.y, xsd),
                                dsub((double)tv.z, xsd), dsub((double)tv.w, xsd)};
          const double du[4] = {dsub((double)uv.x, xsd), dsub((double)uv.y, xsd),
                                dsub((double)uv.z, xsd), dsub((double)uv.w, xsd)};
#pragma unroll
          for (int u = 0; u < kPT; ++u)
#pragma unroll
            for (int w = 0; w < kPT; ++w) acc[u][w] = dadd(acc[u][w], dmul(dt[u], du[w]));
        }
      }
    }
    if (have) {
#pragma unroll
      for (int u = 0; u < kPT; ++u)
#pragma unroll
        for (int w = 0; w < kPT; ++w) {
          const int t = tb * kPT + u, v = ub * kPT + w;
          if (t >= cnt || v >= t) continue;
          bool eq = true;
          for (int z = 0; z < a.l; ++z) eq = eq && eat[t * a.l + z] == eat[v * a.l + z];
          if (!eq) continue;
          const double np2 = nrm[t], nk2 = nrm[v];
          double c = (np2 == 0.0 || nk2 == 0.0) ? 1.0
                                                 : __ddiv_rn(acc[u][w], sqrt(dmul(np2, nk2)));
          if (c > a.sigma) atomicOr(bits + t * a.W + (v >> 5), 1u << (v & 31));
        }
    }
  }
  __syncthreads();
  uint32_t* out = a.rbits + s * (int64_t)a.g * a.W;
  for (int t = tid; t < cnt * a.W; t += blockDim.x) out[t] = bits[t];
}

// Integer features in [0, 255] (the u8 copy F8 with exact squared norms nx8): every product and
// partial sum of _diff_cosine's fp64 loops (_kernels.py:236-253) is an integer below 2^53, so
// dot, np2 and nk2 are exact in any order; from the u8 rows
//   dot(p, k) = x_p.x_k - x_p.x_s - x_k.x_s + |x_s|^2,  np2 = |x_p|^2 - 2 x_p.x_s + |x_s|^2
// with dp4a, and the cosine is then formed exactly as the reference forms it.  Same bits as
// prune_bits_kernel.  Rows are staged with a 33-word stride (no bank conflicts between rows).
__global__ void __launch_bounds__(kPruneThreads) prune_bits_u8_kernel(PruneArgs a, const uint8_t* __restrict__ F8,
                                                                     const int32_t* __restrict__ nx8) {
  extern __shared__ __align__(16) char smem_raw[];
  const int cpad = a.cpad;
  const int mw = a.m >> 2;       // 32-bit words per row
  const int rs = mw | 1;         // odd word stride
  char* p = smem_raw;
  uint32_t* xr = reinterpret_cast<uint32_t*>(p); p += sizeof(uint32_t) * (size_t)cpad * rs;
  uint32_t* xs = reinterpret_cast<uint32_t*>(p); p += sizeof(uint32_t) * (size_t)rs;
  int32_t* ax = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * cpad;   // x_p . x_s
  int32_t* nr = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * cpad;   // |x_p|^2
  int32_t* eid = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * cpad;
  int32_t* eat = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * (size_t)cpad * a.l;
  uint32_t* bits = reinterpret_cast<uint32_t*>(p); p += sizeof(uint32_t) * (size_t)cpad * a.W;
  const int64_t s = blockIdx.x;
  const int cnt = a.counts[s];
  if (cnt <= 1) return;
  const int tid = threadIdx.x;
  const uint32_t* F8w = reinterpret_cast<const uint32_t*>(F8);
  for (int t = tid; t < mw; t += blockDim.x) xs[t] = __ldg(F8w + s * mw + t);
  for (int t = tid; t < cpad; t += blockDim.x) {
    const int32_t v = t < cnt ? a.ids[s * a.g + t] : 0;
    eid[t] = v;
    nr[t] = t < cnt ? __ldg(nx8 + v) : 0;
    for (int u = 0; u < a.l; ++u) eat[t * a.l + u] = t < cnt ? __ldg(a.A + (int64_t)v * a.l + u) : 0;
  }
  for (int t = tid; t < cpad * a.W; t += blockDim.x) bits[t] = 0u;
  __syncthreads();
  {  // every row entry's u8 words, a warp per entry, by 4-byte asynchronous copies
    const int lane_ = tid & 31, nwarp = blockDim.x >> 5;
    for (int t = tid >> 5; t < cnt; t += nwarp) {
      const uint32_t* src = F8w + (int64_t)eid[t] * mw;
      for (int w = lane_; w < mw; w += 32)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(xr + t * rs + w)),
                     "l"(src + w)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
  __syncthreads();
  for (int t = tid; t < cnt; t += blockDim.x) {
    uint32_t acc = 0u;  // u8 x u8 products: unsigned dp4a
    for (int w = 0; w < mw; ++w) acc = __dp4a(xr[t * rs + w], xs[w], acc);
    ax[t] = (int32_t)acc;
  }
  __syncthreads();
  const int64_t c0 = __ldg(nx8 + s);
  const int npairs = cnt * (cnt - 1) / 2;
  for (int pi = tid; pi < npairs; pi += blockDim.x) {
    // pi -> (t, v), v < t, row-major over the strict lower triangle
    int t = (int)((1.0 + sqrt(1.0 + 8.0 * pi)) * 0.5);
    while (t * (t - 1) / 2 > pi) --t;
    while ((t + 1) * t / 2 <= pi) ++t;
    const int v = pi - t * (t - 1) / 2;
    bool eq = true;
    for (int z = 0; z < a.l; ++z) eq = eq && eat[t * a.l + z] == eat[v * a.l + z];
    if (!eq) continue;
    uint32_t g = 0u;
    const uint32_t* rt = xr + t * rs;
    const uint32_t* rv = xr + v * rs;
    for (int w = 0; w < mw; ++w) g = __dp4a(rt[w], rv[w], g);
    const int64_t dot = (int64_t)g - ax[t] - ax[v] + c0;
    const int64_t np2 = (int64_t)nr[t] - 2 * (int64_t)ax[t] + c0;
    const int64_t nk2 = (int64_t)nr[v] - 2 * (int64_t)ax[v] + c0;
    const double cs = (np2 == 0 || nk2 == 0) ? 1.0
                    : __ddiv_rn((double)dot, sqrt(dmul((double)np2, (double)nk2)));
    if (cs > a.sigma) atomicOr(bits + t * a.W + (v >> 5), 1u << (v & 31));
  }
  __syncthreads();
  uint32_t* out = a.rbits + s * (int64_t)a.g * a.W;
  for (int t = tid; t < cnt * a.W; t += blockDim.x) out[t] = bits[t];
}

size_t prune_bits_u8_smem(int cpad, int m, int l, int W) {
  const int rs = (m >> 2) | 1;
  return sizeof(uint32_t) * ((size_t)cpad + 1) * rs + sizeof(int32_t) * (size_t)cpad * (3 + l) +
         sizeof(uint32_t) * (size_t)cpad * W + 64;
}

int launch_prune_bits_u8(const PruneArgs& a, const uint8_t* F8, const int32_t* nx8, size_t smem,
                         cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(prune_bits_u8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return (int)e;
  prune_bits_u8_kernel<<<(unsigned)a.n, kPruneThreads, smem, st>>>(a, F8, nx8);
  return (int)cudaGetLastError();
}

__global__ void prune_scan_kernel(PruneArgs a) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.n) return;
  const int cnt = a.counts[s];
  uint32_t keep[8];
  for (int w = 0; w < a.W; ++w) keep[w] = 0u;
  if (cnt <= 1) {
    if (cnt == 1) keep[0] = 1u;
  } else {
    const uint32_t* rb = a.rbits + s * (int64_t)a.g * a.W;
    keep[0] = 1u;
    for (int t = 1; t < cnt; ++t) {
      bool red = false;
      for (int w = 0; w <= (t >> 5); ++w) red = red || (rb[t * a.W + w] & keep[w]) != 0u;
      const int32_t p = a.ids[s * a.g + t];
      const bool last = a.smax[p] == (int32_t)s;
      if (red && !(last && a.guard[p])) {
        if (!last) atomicAdd(a.drop_other + p, 1);
      } else {
        keep[t >> 5] |= 1u << (t & 31);
      }
    }
  }
  for (int w = 0; w < a.W; ++w) a.keep[s * a.W + w] = keep[w];
}

__global__ void prune_guard_kernel(PruneArgs a, int* changed) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= a.n) return;
  uint8_t gnew = (a.indeg0[p] >= 1 && a.drop_other[p] == a.indeg0[p] - 1) ? 1 : 0;
  if (gnew != a.guard[p]) {
    a.guard[p] = gnew;
    atomicOr(changed, 1);
  }
}

__global__ void prune_compact_kernel(PruneArgs a) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.n) return;
  const int cnt = a.counts[s];
  int w = 0;
  for (int t = 0; t < cnt; ++t) {
    int32_t id = a.ids[s * a.g + t];
    if (a.keep[s * a.W + (t >> 5)] & (1u << (t & 31))) {
      a.ids[s * a.g + w] = id;
      a.dists[s * a.g + w] = a.dists[s * a.g + t];
      ++w;
    } else {
      atomicSub(a.in_deg + id, 1);
    }
  }
  a.counts[s] = w;
}

size_t prune_bits_smem(int cpad, int dc, int m, int l, int W) {
  return sizeof(double) * m + sizeof(double) * cpad + sizeof(float) * (size_t)dc * cpad +
         sizeof(int32_t) * cpad + sizeof(int32_t) * (size_t)cpad * l +
         sizeof(uint32_t) * (size_t)cpad * W + 64;
}

int launch_prune_bits(const PruneArgs& a, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(prune_bits_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return (int)e;
  prune_bits_kernel<<<(unsigned)a.n, kPruneThreadsF64, smem, st>>>(a);
  return (int)cudaGetLastError();
}
int launch_prune_scan(const PruneArgs& a, cudaStream_t st) {
  prune_scan_kernel<<<(unsigned)((a.n + 127) / 128), 128, 0, st>>>(a);
  return (int)cudaGetLastError();
}
int launch_prune_guard(const PruneArgs& a, int* changed, cudaStream_t st) {
  prune_guard_kernel<<<(unsigned)((a.n + 255) / 256), 256, 0, st>>>(a, changed);
  return (int)cudaGetLastError();
}
int launch_prune_compact(const PruneArgs& a, cudaStream_t st) {
  prune_compact_kernel<<<(unsigned)((a.n + 127) / 128), 128, 0, st>>>(a);
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// reinforce, fast path
SB_DEV bool row_has_key(const int32_t* ids, const float* dists, int cnt, uint64_t key) {
  int lo = 0, hi = cnt;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    uint64_t k = row_key(dists[mid], (uint32_t)ids[mid]);
    if (k < key) lo = mid + 1; else hi = mid;
  }
  return lo < cnt && row_key(dists[lo], (uint32_t)ids[lo]) == key;
}

// count, per target j, reverse entries s (j in row_s) that row j lacks
__global__ void rev_missing_kernel(const int32_t* ids, const float* dists, const int32_t* counts,
                                   int64_t n, int g, int64_t* rev_extra) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * g) return;
  int64_t s = e / g;
  int t = (int)(e % g);
  if (t >= counts[s]) return;
  int32_t j = ids[e];
  uint64_t key = row_key(dists[e], (uint32_t)s);
  if (!row_has_key(ids + (int64_t)j * g, dists + (int64_t)j * g, counts[j], key))
    atomicAdd(reinterpret_cast<unsigned long long*>(rev_extra + j), 1ull);
}

__global__ void overflow_kernel(const int32_t* counts, const int64_t* rev_extra, int64_t n, int g,
                                unsigned long long* over) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  if ((int64_t)counts[j] + rev_extra[j] > g) atomicAdd(over, 1ull);
}

__global__ void rev_missing_scatter_kernel(const int32_t* ids, const float* dists,
                                           const int32_t* counts, int64_t n, int g,
                                           const int64_t* off, int64_t* cur, uint64_t* seg) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * g) return;
  int64_t s = e / g;
  int t = (int)(e % g);
  if (t >= counts[s]) return;
  int32_t j = ids[e];
  uint64_t key = row_key(dists[e], (uint32_t)s);
  if (!row_has_key(ids + (int64_t)j * g, dists + (int64_t)j * g, counts[j], key)) {
    unsigned long long p = atomicAdd(reinterpret_cast<unsigned long long*>(cur + j), 1ull);
    seg[off[j] + (int64_t)p] = key;
  }
}

// warp per row: sorted union of the row and its missing reverse entries
__global__ void symmetrize_merge_kernel(int32_t* ids, float* dists, int32_t* counts, int64_t n,
                                        int g, int gpad, const int64_t* off,
                                        const int64_t* extra, const uint64_t* seg) {
  extern __shared__ __align__(16) char smem_raw[];
  const int wpb = blockDim.x >> 5;
  uint64_t* L = reinterpret_cast<uint64_t*>(smem_raw) + (size_t)warp_id() * 2 * gpad;
  uint64_t* C = L + gpad;
  int64_t j = (int64_t)blockIdx.x * wpb + warp_id();
  if (j >= n) return;
  const int E = (int)extra[j];
  if (E == 0) return;
  const int lane = lane_id();
  const int cnt = counts[j];
  for (int t = lane; t < cnt; t += 32) L[t] = row_key(dists[j * g + t], (uint32_t)ids[j * g + t]);
  int np = next_pow2(E);
  for (int t = lane; t < np; t += 32) C[t] = t < E ? seg[off[j] + t] : kKeyInf;
  __syncwarp();
  if (np > 1) warp_bitonic_u64(C, np);
  // positions in the union (no duplicates by construction)
  for (int t = lane; t < cnt; t += 32) {
    uint64_t k = L[t];
    int pos = t + lower_bound_u64(C, E, k);
    ids[j * g + pos] = (int32_t)key_id(k);
    dists[j * g + pos] = key_dist(k);
  }
  for (int t = lane; t < E; t += 32) {
    uint64_t k = C[t];
    int pos = t + lower_bound_u64(L, cnt, k);
    ids[j * g + pos] = (int32_t)key_id(k);
    dists[j * g + pos] = key_dist(k);
  }
  if (lane == 0) counts[j] = cnt + E;
}

int launch_row_union_merge(int32_t* ids, float* dists, int32_t* counts, int64_t n, int g,
                           const int64_t* off, const int64_t* extra, const uint64_t* seg,
                           cudaStream_t st) {
  int gpad = next_pow2(g);
  int wpb = 4;
  size_t smem = (size_t)wpb * 2 * gpad * sizeof(uint64_t);
  cudaFuncSetAttribute(symmetrize_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  symmetrize_merge_kernel<<<(unsigned)((n + wpb - 1) / wpb), wpb * 32, smem, st>>>(
      ids, dists, counts, n, g, gpad, off, extra, seg);
  return (int)cudaGetLastError();
}

int launch_reinforce_check(const int32_t* ids, const float* dists, const int32_t* counts,
                           int64_t n, int g, int64_t* rev_extra, unsigned long long* over,
                           cudaStream_t st) {
  cudaMemsetAsync(rev_extra, 0, sizeof(int64_t) * n, st);
  cudaMemsetAsync(over, 0, sizeof(unsigned long long), st);
  int64_t tot = n * g;
  rev_missing_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(ids, dists, counts, n, g,
                                                                     rev_extra);
  overflow_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(counts, rev_extra, n, g, over);
  return (int)cudaGetLastError();
}

int launch_symmetrize(int32_t* ids, float* dists, int32_t* counts, int64_t n, int g,
                      const int64_t* rev_extra, int64_t* off, int64_t* cur, uint64_t* seg,
                      int64_t* scan_tmp, cudaStream_t st) {
  exclusive_scan(rev_extra, off, n, scan_tmp, st);
  cudaMemsetAsync(cur, 0, sizeof(int64_t) * n, st);
  int64_t tot = n * g;
  rev_missing_scatter_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(ids, dists, counts, n,
                                                                             g, off, cur, seg);
  int gpad = next_pow2(g);
  int wpb = 4;
  size_t smem = (size_t)wpb * 2 * gpad * sizeof(uint64_t);
  cudaFuncSetAttribute(symmetrize_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  symmetrize_merge_kernel<<<(unsigned)((n + wpb - 1) / wpb), wpb * 32, smem, st>>>(
      ids, dists, counts, n, g, gpad, off, rev_extra, seg);
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// exact sequential semantics (overflow case): _try_insert_edge / reinforce_pass /
// _force_insert_edge / reconnect_islands, single device thread.
struct SeqCtx {
  const float* F;
  const int32_t* A;
  int m, l, g;
  int32_t* ids;
  float* dists;
  int32_t* counts;
  int32_t* in_deg;
  double sigma;
};

SB_DEV bool seq_attrs_equal(const SeqCtx& c, int64_t a, int64_t b) {
  for (int t = 0; t < c.l; ++t)
    if (c.A[a * c.l + t] != c.A[b * c.l + t]) return false;
  return true;
}

SB_DEV int seq_force_insert(SeqCtx& c, int64_t j, int64_t cand, double dd, bool unsafe) {
  const float d = __double2float_rn(dd);
  int32_t* ri = c.ids + j * c.g;
  float* rd = c.dists + j * c.g;
  int cj = c.counts[j];
  for (int t = 0; t < cj; ++t)
    if (ri[t] == cand) return 0;
  if (cj >= c.g) {
    int ev = -1;
    for (int t = cj - 1; t >= 0; --t)
      if (c.in_deg[ri[t]] >= 2) { ev = t; break; }
    if (ev < 0) {
      if (!unsafe) return 0;
      ev = cj - 1;
    }
    c.in_deg[ri[ev]] -= 1;
    for (int t = ev; t < cj - 1; ++t) { ri[t] = ri[t + 1]; rd[t] = rd[t + 1]; }
    --cj;
  }
  int pos = cj;
  while (pos > 0 && (rd[pos - 1] > d || (rd[pos - 1] == d && ri[pos - 1] > cand))) {
    ri[pos] = ri[pos - 1];
    rd[pos] = rd[pos - 1];
    --pos;
  }
  ri[pos] = (int32_t)cand;
  rd[pos] = d;
  c.counts[j] = cj + 1;
  c.in_deg[cand] += 1;
  return 1;
}

// ---- reconnect_islands by one CTA ------------------------------------------------------
// The sweep is sequential over v (_kernels.py:455-487), but the costly part of each
// _try_insert_edge on a full row, the redundancy of every pair of the merged list
// (attrs_equal && cos > sigma, _kernels.py:356-366), is independent per pair: 256 threads
// compute the norms |p - j|^2 and the pair dots in the reference's dimension order (separate
// accumulation chains, same values) into a bit matrix, and thread 0 runs the greedy keep pass
// over it.  In-degrees of the merged entries are loaded up front: within one insertion an
// entry's in-degree changes only when that entry is dropped, and it is not read again.
constexpr int kRcThreads = 256;
constexpr int kRcMaxG = 256;

struct RcShared {
  int64_t mi[kRcMaxG + 1];
  double md[kRcMaxG + 1];
  double nrm[kRcMaxG + 1];
  int32_t midg[kRcMaxG + 1];
  uint8_t keep[kRcMaxG + 1];
  int result, total, pos, flag;
};

// Redundancy bits of the merged list mi[0..total) relative to row owner j (bit u of row t,
// u < t: attrs_equal && cos > sigma) and the norms |p - j|^2, by the whole CTA: dimension
// chunks of every listed row are staged in shared memory (coalesced) and each thread owns up
// to two 4 x 4 tiles of the lower triangle of pair dots in registers, so a row is read once
// per chunk instead of once per pair.  Every dot, norm and cosine is accumulated in ascending
// dimension order with separately rounded fp64 operations (_kernels.py:236-253): the same
// values as the per-pair loops.
constexpr int kRcDc = 32;  // dimensions per staged chunk
SB_DEV void cta_pair_bits(const SeqCtx& c, const int64_t* mi, int total, int64_t j, double* nrm,
                          uint32_t* bits, int W, float* xr, double* xs) {
  const int tid = threadIdx.x;
  const int cpad = (total + kPT - 1) / kPT * kPT;
  const int nb = cpad / kPT;
  const int ntiles = nb * (nb + 1) / 2;
  for (int t = tid; t < c.m; t += kRcThreads) xs[t] = (double)__ldg(c.F + j * c.m + t);
  for (int w = tid; w < total * W; w += kRcThreads) bits[w] = 0u;
  // passes of two tiles per thread (one pass covers up to 123 list entries); the norms of list
  // entries tid and tid + kRcThreads accumulate during the first pass
  for (int pass = 0; pass * 2 * kRcThreads < ntiles; ++pass) {
    int tbs[2], ubs[2];
    bool have[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int ti = pass * 2 * kRcThreads + h * kRcThreads + tid;
      have[h] = ti < ntiles;
      int tb = 0, ub = 0;
      if (have[h]) {
        tb = (int)((sqrt(8.0 * ti + 1.0) - 1.0) * 0.5);
        while ((tb + 1) * (tb + 2) / 2 <= ti) ++tb;
        while (tb * (tb + 1) / 2 > ti) --tb;
        ub = ti - tb * (tb + 1) / 2;
      }
      tbs[h] = tb;
      ubs[h] = ub;
    }
    double acc[2][kPT][kPT];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int u = 0; u < kPT; ++u)
#pragma unroll
        for (int w = 0; w < kPT; ++w) acc[h][u][w] = 0.0;
    double nacc[2] = {0.0, 0.0};
    for (int d0 = 0; d0 < c.m; d0 += kRcDc) {
      const int dc = c.m - d0 < kRcDc ? c.m - d0 : kRcDc;
      __syncthreads();
      {  // a warp per entry, 4-byte asynchronous copies (zeros behind the merged list)
        const int lane_ = tid & 31;
        for (int t = tid >> 5; t < cpad; t += kRcThreads >> 5) {
          if (t < total) {
            const float* src = c.F + mi[t] * c.m + d0;
            for (int dd = lane_; dd < dc; dd += 32)
              asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                               (uint32_t)__cvta_generic_to_shared(xr + dd * cpad + t)),
                           "l"(src + dd)
                           : "memory");
          } else {
            for (int dd = lane_; dd < dc; dd += 32) xr[dd * cpad + t] = 0.f;
          }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      if (pass == 0)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int t = tid + h * kRcThreads;
          if (t < total)
            for (int dd = 0; dd < dc; ++dd) {
              const double dp = dsub((double)xr[dd * cpad + t], xs[d0 + dd]);
              nacc[h] = dadd(nacc[h], dmul(dp, dp));
            }
        }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (!have[h]) continue;
        for (int dd = 0; dd < dc; ++dd) {
          const float* row = xr + (size_t)dd * cpad;
          const double xsd = xs[d0 + dd];
          const float4 tv = *reinterpret_cast<const float4*>(row + tbs[h] * kPT);
          const float4 uv = *reinterpret_cast<const float4*>(row + ubs[h] * kPT);
          const double dt[4] = {dsub((double)tv.x, xsd), dsub((double)tv.y, xsd),
                                dsub((double)tv.z, xsd), dsub((double)tv.w, xsd)};
          const double du[4] = {dsub((double)uv.x, xsd), dsub((double)uv.y, xsd),
                                dsub((double)uv.z, xsd), dsub((double)uv.w, xsd)};
#pragma unroll
          for (int u = 0; u < kPT; ++u)
#pragma unroll
            for (int w = 0; w < kPT; ++w) acc[h][u][w] = dadd(acc[h][u][w], dmul(dt[u], du[w]));
        }
      }
    }
    if (pass == 0)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (tid + h * kRcThreads < total) nrm[tid + h * kRcThreads] = nacc[h];
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (!have[h]) continue;
#pragma unroll
      for (int u = 0; u < kPT; ++u)
#pragma unroll
        for (int w = 0; w < kPT; ++w) {
          const int t = tbs[h] * kPT + u, v = ubs[h] * kPT + w;
          if (t >= total || v >= t) continue;
          if (!seq_attrs_equal(c, mi[t], mi[v])) continue;
          const double np2 = nrm[t], nk2 = nrm[v];
          const double cs = (np2 == 0.0 || nk2 == 0.0) ? 1.0 : __ddiv_rn(acc[h][u][w], sqrt(dmul(np2, nk2)));
          if (cs > c.sigma) atomicOr(bits + t * W + (v >> 5), 1u << (v & 31));
        }
    }
  }
  __syncthreads();
}

// returns 1 if cand ends up in row j (all threads get the value)
SB_DEV int cta_try_insert(SeqCtx& c, RcShared& S, uint32_t* bits, int64_t j, int64_t cand, double dd,
                          float* xr, double* xs) {
  const int tid = threadIdx.x;
  const float d = __double2float_rn(dd);
  int32_t* ri = c.ids + j * c.g;
  float* rd = c.dists + j * c.g;
  if (tid == 0) {
    S.result = -1;
    const int cj = c.counts[j];
    bool dup = false;
    for (int t = 0; t < cj && !dup; ++t) dup = ri[t] == cand;
    if (dup) {
      S.result = 0;
    } else if (cj < c.g) {
      int pos = cj;
      while (pos > 0 && (rd[pos - 1] > d || (rd[pos - 1] == d && ri[pos - 1] > cand))) {
        ri[pos] = ri[pos - 1];
        rd[pos] = rd[pos - 1];
        --pos;
      }
      ri[pos] = (int32_t)cand;
      rd[pos] = d;
      c.counts[j] = cj + 1;
      c.in_deg[cand] += 1;
      S.result = 1;
    } else {
      int pos = cj;
      for (int t = 0; t < cj; ++t) { S.mi[t] = ri[t]; S.md[t] = (double)rd[t]; }
      while (pos > 0 && (S.md[pos - 1] > (double)d ||
                         (S.md[pos - 1] == (double)d && S.mi[pos - 1] > cand))) {
        S.mi[pos] = S.mi[pos - 1];
        S.md[pos] = S.md[pos - 1];
        --pos;
      }
      S.mi[pos] = cand;
      S.md[pos] = (double)d;
      S.total = cj + 1;
    }
  }
  __syncthreads();
  if (S.result >= 0) {
    const int r = S.result;
    __syncthreads();
    return r;
  }
  const int total = S.total;
  const int W = (total + 31) >> 5;
  for (int t = tid; t < total; t += kRcThreads) {
    const int64_t p = S.mi[t];
    S.midg[t] = p == cand ? 0 : c.in_deg[p];
    S.keep[t] = 1;
  }
  cta_pair_bits(c, S.mi, total, j, S.nrm, bits, W, xr, xs);
  if (tid == 0) {
    // kept mask over list positions; at step t it holds exactly the kept u < t
    uint32_t km[(kRcMaxG + 32) / 32];
    for (int w = 0; w < W; ++w) km[w] = 0u;
    km[0] = 1u;
    int kept = 1;
    for (int t = 1; t < total; ++t) {
      bool red = false;
      for (int w = 0; w <= (t >> 5) && !red; ++w) red = (bits[t * W + w] & km[w]) != 0u;
      const int64_t p = S.mi[t];
      if (red && (p == cand || S.midg[t] >= 2)) {
        S.keep[t] = 0;
      } else {
        ++kept;
        km[t >> 5] |= 1u << (t & 31);
      }
    }
    if (kept > c.g) {
      for (int t = total - 1; t >= 0; --t) {
        if (!S.keep[t]) continue;
        const int64_t p = S.mi[t];
        if (p == cand) { S.keep[t] = 0; break; }
        if (S.midg[t] >= 2) { S.keep[t] = 0; break; }
      }
    }
    int w = 0, inserted = 0;
    for (int t = 0; t < total; ++t) {
      if (!S.keep[t]) {
        if (S.mi[t] != cand) c.in_deg[S.mi[t]] -= 1;
        continue;
      }
      ri[w] = (int32_t)S.mi[t];
      rd[w] = __double2float_rn(S.md[t]);
      if (S.mi[t] == cand) inserted = 1;
      ++w;
    }
    c.counts[j] = w;
    if (inserted) c.in_deg[cand] += 1;
    S.result = inserted;
  }
  __syncthreads();
  const int r = S.result;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kRcThreads) reconnect_cta_kernel(SeqCtx c, int64_t n) {
  extern __shared__ __align__(16) uint32_t rc_bits[];
  // dynamic shared memory: bits [(g + 1) x W words] | staged chunk [kRcDc x cpad floats] | owner row [m doubles]
  const int cpad_max = (c.g + 1 + kPT - 1) / kPT * kPT;
  const size_t bits_words = (size_t)(c.g + 1) * ((c.g + 32) / 32);
  float* rc_xr = reinterpret_cast<float*>(rc_bits + ((bits_words + 3) & ~(size_t)3));
  double* rc_xs = reinterpret_cast<double*>(rc_xr + (size_t)kRcDc * cpad_max);
  __shared__ RcShared S;
  const int tid = threadIdx.x;
  const volatile int32_t* indeg = c.in_deg;
  for (int64_t base = 0; base < n; base += kRcThreads) {
    int64_t from = base;
    for (;;) {
      // first node of this chunk at or after `from` with in-degree 0 (re-read after every
      // node: an insertion can drop a later node's in-degree to 0)
      if (tid == 0) S.flag = 0x7FFFFFFF;
      __syncthreads();
      const int64_t v0 = base + tid;
      if (v0 >= from && v0 < n && indeg[v0] <= 0) atomicMin(&S.flag, tid);
      __syncthreads();
      const int first = S.flag;
      __syncthreads();
      if (first == 0x7FFFFFFF) break;
      const int64_t v = base + first;
      from = v + 1;
      bool done = false;
      const int cv = c.counts[v];
      for (int t = 0; t < cv && !done; ++t) {
        const int64_t u = c.ids[v * c.g + t];
        done = cta_try_insert(c, S, rc_bits, u, v, (double)c.dists[v * c.g + t], rc_xr, rc_xs) != 0;
      }
      if (tid == 0 && !done) {
        for (int t = 0; t < c.counts[v] && !done; ++t) {
          const int64_t u = c.ids[v * c.g + t];
          done = seq_force_insert(c, u, v, (double)c.dists[v * c.g + t], false) != 0;
        }
        if (!done && c.counts[v] > 0)
          seq_force_insert(c, c.ids[v * c.g], v, (double)c.dists[v * c.g], true);
      }
      __syncthreads();
    }
  }
}

__global__ void min_kernel(const int32_t* x, int64_t n, int* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicMin(out, x[i]);
}

int launch_reconnect(const float* F, const int32_t* A, int m, int l, int g, int32_t* ids,
                     float* dists, int32_t* counts, int32_t* in_deg, double sigma, int64_t n,
                     cudaStream_t st) {
  SeqCtx c;
  c.F = F; c.A = A; c.m = m; c.l = l; c.g = g;
  c.ids = ids; c.dists = dists; c.counts = counts; c.in_deg = in_deg; c.sigma = sigma;
  if (g > kRcMaxG) return (int)cudaErrorInvalidValue;
  const int cpad_max = (g + 1 + kPT - 1) / kPT * kPT;
  const size_t bits_words = (size_t)(g + 1) * ((g + 32) / 32);
  const size_t bits = sizeof(uint32_t) * ((bits_words + 3) & ~(size_t)3) + sizeof(float) * (size_t)kRcDc * cpad_max +
                      sizeof(double) * (size_t)m + 16;
  cudaError_t e = cudaFuncSetAttribute(reconnect_cta_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bits);
  if (e != cudaSuccess) return (int)e;
  reconnect_cta_kernel<<<1, kRcThreads, bits, st>>>(c, n);
  return (int)cudaGetLastError();
}

int launch_min_i32(const int32_t* x, int64_t n, int* out, cudaStream_t st) {
  min_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, n, out);
  return (int)cudaGetLastError();
}

}  // namespace sb

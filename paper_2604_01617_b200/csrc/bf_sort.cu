// bf_sort.cu — exhaustive top-k by a full radix sort of every node's exact key.
//
// The tiled top-k kernels (bf_topk.cu, bf_tc.cu, bf_tf.cu) keep per-query lists in shared
// memory or registers, so their k is bounded.  The reference is not: brute_force_topk and
// oracle_auto_topk accept any k <= n (_kernels.py:176-204, evaluate.py:32-55), and
// oracle_hybrid_groundtruth ranks every attribute-matching node (evaluate.py:58-77).  This file
// serves those cases exactly:
//
//  1. keys kernel: one thread per (query, node) computes the exact distance the reference
//     would (mode below) and writes key = its IEEE bits (non-negative doubles order like their
//     bit patterns as u64), value = node id;
//  2. one CUB segmented radix sort per chunk of queries (LSD radix sort is stable, the input
//     is in ascending id order, so equal distances stay in ascending id order — the
//     reference's (distance, id) tie rule, lexsort((arange(n), fused)));
//  3. a gather kernel copies the first k of every segment.
//
// Modes:
//  kNodeMode   brute_force_topk: sequential fp64 _pair_dist (s_a * inv_alpha), self excluded
//              (key = ~0, sorts last), ids past n-1 padded with -1 (_kernels.py:187,202-203).
//  kQueryMode  oracle_auto_topk: NumPy's pairwise sum order (evaluate.py:48), s_a / alpha.
//  kHybridMode oracle_hybrid_groundtruth: nodes whose masked |a - qa| sum is 0 keyed by
//              sqrt(NumPy pairwise sum) (evaluate.py:69-75); others key ~0; the number of
//              matching nodes is returned so the caller can truncate to min(k, matches).
//
// Bound: HBM/L2 (each key reads one feature row; the sort moves 12 B per key per pass).
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "sb_internal.h"

namespace sb {

namespace {

__global__ void bf_sort_keys_kernel(BfArgs a, int mode, int64_t q0, uint64_t* keys,
                                    uint32_t* vals, unsigned long long* matches) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t b = blockIdx.y;  // query within the chunk
  const int64_t g = q0 + b;
  if (v >= a.n) return;
  const size_t o = (size_t)b * a.n + v;
  uint64_t key;
  if (mode == kBfSortNode) {
    const int64_t u = a.self_ids[g];
    key = v == u ? ~0ull
                 : (uint64_t)__double_as_longlong(pair_dist(a.F, a.A, a.m, a.l, u, v, a.inv_alpha));
  } else {
    const int64_t* qa = a.qa + g * a.l;
    const int64_t* qm = a.qmask ? a.qmask + g * a.l : nullptr;
    int64_t si = 0;
    for (int t = 0; t < a.l; ++t) {
      int64_t ad = (int64_t)__ldg(a.A + v * (int64_t)a.l + t) - qa[t];
      ad = ad < 0 ? -ad : ad;
      si += qm ? ad * qm[t] : ad;
    }
    if (mode == kBfSortHybrid && si != 0) {
      key = ~0ull;
    } else {
      const double sv = sqrt(np_pairwise_sq(a.F + v * (int64_t)a.m, a.qf + g * (int64_t)a.m, a.m));
      const double d = mode == kBfSortHybrid ? sv : dmul(sv, dadd(1.0, __ddiv_rn((double)si, a.alpha)));
      key = (uint64_t)__double_as_longlong(d);
      if (mode == kBfSortHybrid) atomicAdd(matches + b, 1ull);
    }
  }
  keys[o] = key;
  vals[o] = (uint32_t)v;
}

__global__ void bf_sort_offsets_kernel(int64_t* offs, int64_t b, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= b) offs[i] = i * n;
}

__global__ void bf_sort_gather_kernel(int mode, int64_t n, int64_t q0, int64_t b, int kout,
                                      const uint64_t* keys, const uint32_t* vals,
                                      const unsigned long long* matches, int64_t* out64,
                                      int32_t* out32, double* outd, int64_t* out_counts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= b * kout) return;
  const int64_t bq = i / kout, t = i % kout;
  const int64_t g = q0 + bq;
  const size_t src = (size_t)bq * n + t;
  if (mode == kBfSortNode) {
    out32[g * kout + t] = t < n - 1 ? (int32_t)vals[src] : -1;
    return;
  }
  int64_t valid = t < n ? 1 : 0;
  if (mode == kBfSortHybrid) {
    const int64_t c = (int64_t)matches[bq];
    valid = t < c;
    if (t == 0 && out_counts) out_counts[g] = c < kout ? c : kout;
  }
  out64[g * kout + t] = valid ? (int64_t)vals[src] : -1;
  if (outd)
    outd[g * kout + t] = valid ? __longlong_as_double((long long)keys[src])
                               : __longlong_as_double(0x7FF0000000000000ll);
}

}  // namespace

int64_t bf_sort_chunk(int64_t n, int64_t q) {
  const int64_t cap = std::max<int64_t>(1, (int64_t(1) << 26) / std::max<int64_t>(1, n));
  return std::min<int64_t>(std::min<int64_t>(q, cap), 65535);  // grid.y limit
}

size_t bf_sort_scratch_bytes(int64_t n, int64_t b) {
  const size_t keys = (size_t)n * b;
  size_t temp = 0;
  cub::DeviceSegmentedRadixSort::SortPairs(nullptr, temp, (const uint64_t*)nullptr,
                                           (uint64_t*)nullptr, (const uint32_t*)nullptr,
                                           (uint32_t*)nullptr, (int64_t)keys, (int64_t)b,
                                           (const int64_t*)nullptr, (const int64_t*)nullptr);
  return keys * 2 * (sizeof(uint64_t) + sizeof(uint32_t)) + sizeof(int64_t) * (b + 1) +
         sizeof(unsigned long long) * b + temp + 8192;  // + 256-byte alignment of six arrays
}

int launch_bf_sorted(const BfArgs& a, int mode, int64_t q0, int64_t b, int kout, void* scratch,
                     size_t scratch_bytes, int64_t* out64, int32_t* out32, double* outd,
                     int64_t* out_counts, cudaStream_t st) {
  const int64_t n = a.n;
  const size_t keys = (size_t)n * b;
  char* p = static_cast<char*>(scratch);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) & ~(size_t)255;
    return r;
  };
  uint64_t* k_in = reinterpret_cast<uint64_t*>(take(keys * sizeof(uint64_t)));
  uint64_t* k_out = reinterpret_cast<uint64_t*>(take(keys * sizeof(uint64_t)));
  uint32_t* v_in = reinterpret_cast<uint32_t*>(take(keys * sizeof(uint32_t)));
  uint32_t* v_out = reinterpret_cast<uint32_t*>(take(keys * sizeof(uint32_t)));
  int64_t* offs = reinterpret_cast<int64_t*>(take(sizeof(int64_t) * (b + 1)));
  unsigned long long* matches = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long) * b));
  const size_t used = (size_t)(p - static_cast<char*>(scratch));
  if (used > scratch_bytes) return (int)cudaErrorInvalidValue;
  size_t temp = scratch_bytes - used;
  cudaError_t e = cudaMemsetAsync(matches, 0, sizeof(unsigned long long) * b, st);
  if (e != cudaSuccess) return (int)e;
  dim3 grid((unsigned)((n + 255) / 256), (unsigned)b);
  bf_sort_keys_kernel<<<grid, 256, 0, st>>>(a, mode, q0, k_in, v_in, matches);
  bf_sort_offsets_kernel<<<(unsigned)((b + 256) / 256), 256, 0, st>>>(offs, b, n);
  if ((e = cudaGetLastError()) != cudaSuccess) return (int)e;
  e = cub::DeviceSegmentedRadixSort::SortPairs(p, temp, k_in, k_out, v_in, v_out, (int64_t)keys,
                                               (int64_t)b, offs, offs + 1, 0, 64, st);
  if (e != cudaSuccess) return (int)e;
  const int64_t outs = b * kout;
  bf_sort_gather_kernel<<<(unsigned)((outs + 255) / 256), 256, 0, st>>>(
      mode, n, q0, b, kout, k_out, v_out, matches, out64, out32, outd, out_counts);
  return (int)cudaGetLastError();
}

}  // namespace sb

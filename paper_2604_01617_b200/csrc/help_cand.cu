// help_cand.cu — HELP build, part 1: random-init distances + row sort, in-degrees, a device
// exclusive scan, and NN-descent candidate construction.
//
//  init      compute_row_distances (_kernels.py:71-78) + lexsort((ids, dists)) per row
//            (graph.py:134-136): warp per row, exact fp64 _pair_dist, key (f32 d, id).
//  cand      build_candidates (_kernels.py:81-135), order-independent restatement:
//              forward: first gamma_new new-flagged entries in row order (flags cleared),
//                       old-flagged entries seen before the break;
//              reverse: for target j, sources i with j in fwd(i) in ascending i, skipping
//                       those already in fwd(j), until capacity (gamma_new / gamma) —
//                       i.e. the smallest (cap) non-duplicate sources.
//            Reverse lists are built by a counting sort of the forward edges by target and a
//            per-target warp selection of the smallest sources.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "sb_internal.h"

namespace sb {

// ---------------------------------------------------------------------------
// init: distances of the random graph and per-row sort by (f32 dist, id)
__global__ void init_rows_kernel(const float* __restrict__ F, const int32_t* __restrict__ A,
                                 int64_t n, int m, int l, int g, int gpad, double inv_alpha,
                                 int32_t* ids, float* dists) {
  extern __shared__ __align__(16) char smem_raw[];
  const int wpb = blockDim.x >> 5;
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem_raw) + (size_t)warp_id() * gpad;
  int64_t i = (int64_t)blockIdx.x * wpb + warp_id();
  if (i >= n) return;
  for (int t = lane_id(); t < gpad; t += 32) {
    uint64_t k = kKeyInf;
    if (t < g) {
      int32_t j = ids[i * g + t];
      double d = pair_dist(F, A, m, l, i, j, inv_alpha);
      k = row_key(__double2float_rn(d), (uint32_t)j);
    }
    keys[t] = k;
  }
  __syncwarp();
  warp_bitonic_u64(keys, gpad);
  for (int t = lane_id(); t < g; t += 32) {
    ids[i * g + t] = (int32_t)key_id(keys[t]);
    dists[i * g + t] = key_dist(keys[t]);
  }
}

int launch_init_dists(const float* F, const int32_t* A, int64_t n, int m, int l, int g,
                      double inv_alpha, int32_t* ids, float* dists, cudaStream_t st) {
  int gpad = next_pow2(g);
  int wpb = 4;
  size_t smem = (size_t)wpb * gpad * sizeof(uint64_t);
  cudaFuncSetAttribute(init_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned grid = (unsigned)((n + wpb - 1) / wpb);
  init_rows_kernel<<<grid, wpb * 32, smem, st>>>(F, A, n, m, l, g, gpad, inv_alpha, ids, dists);
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// in-degrees (count_in_degrees, _kernels.py:256-263) and the largest in-neighbour id
__global__ void indeg_kernel(const int32_t* __restrict__ ids, const int32_t* __restrict__ counts,
                             int64_t n, int g, int32_t* in_deg, int32_t* smax) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * g) return;
  int64_t i = e / g;
  int t = (int)(e % g);
  if (t >= counts[i]) return;
  int32_t p = ids[e];
  atomicAdd(in_deg + p, 1);
  if (smax) atomicMax(smax + p, (int32_t)i);
}

int launch_count_in_degrees(const int32_t* ids, const int32_t* counts, int64_t n, int g,
                            int32_t* in_deg, int32_t* smax, cudaStream_t st) {
  cudaMemsetAsync(in_deg, 0, sizeof(int32_t) * n, st);
  if (smax) cudaMemsetAsync(smax, 0xFF, sizeof(int32_t) * n, st);  // -1
  int64_t tot = n * g;
  indeg_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(ids, counts, n, g, in_deg, smax);
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// exclusive scan of int64 counts (n up to ~2^31): block scans + scan of block sums
constexpr int kScanBlock = 1024;

__global__ void scan_block_kernel(const int64_t* in, int64_t* out, int64_t n, int64_t* sums) {
  __shared__ int64_t s[kScanBlock];
  int64_t i = (int64_t)blockIdx.x * kScanBlock + threadIdx.x;
  int64_t v = i < n ? in[i] : 0;
  s[threadIdx.x] = v;
  __syncthreads();
  for (int o = 1; o < kScanBlock; o <<= 1) {
    int64_t t = threadIdx.x >= o ? s[threadIdx.x - o] : 0;
    __syncthreads();
    s[threadIdx.x] += t;
    __syncthreads();
  }
  if (i < n) out[i] = s[threadIdx.x] - v;  // exclusive
  if (threadIdx.x == kScanBlock - 1) sums[blockIdx.x] = s[threadIdx.x];
}

__global__ void scan_add_kernel(int64_t* out, int64_t n, const int64_t* offs) {
  int64_t i = (int64_t)blockIdx.x * kScanBlock + threadIdx.x;
  if (i < n) out[i] += offs[blockIdx.x];
}

// out[i] = sum(in[0..i)); returns total in *total_dev (device scalar) if non-null.
// tmp must hold scan_tmp_slots(n) int64s.
int64_t scan_tmp_slots(int64_t n) {
  int64_t b = (n + kScanBlock - 1) / kScanBlock;
  int64_t s = 0;
  while (b > 1) {
    s += 2 * b + 2;
    b = (b + kScanBlock - 1) / kScanBlock;
  }
  return s + 8;
}

int exclusive_scan(const int64_t* in, int64_t* out, int64_t n, int64_t* tmp, cudaStream_t st) {
  if (n <= 0) return 0;
  int64_t nb = (n + kScanBlock - 1) / kScanBlock;
  int64_t* sums = tmp;
  int64_t* offs = tmp + nb + 1;
  scan_block_kernel<<<(unsigned)nb, kScanBlock, 0, st>>>(in, out, n, sums);
  if (nb > 1) {
    exclusive_scan(sums, offs, nb, offs + nb + 1, st);
    scan_add_kernel<<<(unsigned)nb, kScanBlock, 0, st>>>(out, n, offs);
  }
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// candidates, forward split (warp per row)
__global__ void cand_forward_kernel(const int32_t* __restrict__ ids, uint8_t* flags, int64_t n,
                                    int g, int gn, int32_t* new_cand, int32_t* new_cnt,
                                    int32_t* old_cand, int32_t* old_cnt) {
  const int wpb = blockDim.x >> 5;
  int64_t i = (int64_t)blockIdx.x * wpb + warp_id();
  if (i >= n) return;
  const int lane = lane_id();
  const unsigned lt = (1u << lane) - 1u;
  int newc = 0, oldc = 0;
  bool done = false;
  for (int base = 0; base < g && !done; base += 32) {
    int t = base + lane;
    bool valid = t < g;
    uint8_t fl = valid ? flags[i * g + t] : 0;
    bool isnew = valid && fl == 1;
    bool isold = valid && fl != 1;
    unsigned bn = __ballot_sync(0xffffffffu, isnew);
    int rank = newc + __popc(bn & lt);
    bool take_new = isnew && rank < gn;
    // the scan stops right after the gamma_new-th new entry (_kernels.py:103-104)
    unsigned last = __ballot_sync(0xffffffffu, isnew && rank == gn - 1);
    int cut = 31;
    if (last) { cut = __ffs(last) - 1; done = true; }
    bool take_old = isold && lane <= cut;
    unsigned bo = __ballot_sync(0xffffffffu, take_old);
    if (take_new) {
      new_cand[i * gn + rank] = ids[i * g + t];
      flags[i * g + t] = 0;
    }
    if (take_old) old_cand[i * g + oldc + __popc(bo & lt)] = ids[i * g + t];
    newc += __popc(__ballot_sync(0xffffffffu, take_new));
    oldc += __popc(bo);
  }
  for (int t = newc + lane; t < gn; t += 32) new_cand[i * gn + t] = -1;
  for (int t = oldc + lane; t < g; t += 32) old_cand[i * g + t] = -1;
  if (lane == 0) { new_cnt[i] = newc; old_cnt[i] = oldc; }
}

// count forward edges per target (one thread per (row, slot))
__global__ void rev_count_kernel(const int32_t* cand, const int32_t* cnt, int64_t n, int cap,
                                 int64_t* rev_cnt) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * cap) return;
  int64_t i = e / cap;
  int x = (int)(e % cap);
  if (x >= cnt[i]) return;
  atomicAdd(reinterpret_cast<unsigned long long*>(rev_cnt + cand[e]), 1ull);
}

__global__ void rev_scatter_kernel(const int32_t* cand, const int32_t* cnt, int64_t n, int cap,
                                   const int64_t* rev_off, int64_t* rev_cur, int32_t* rev) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * cap) return;
  int64_t i = e / cap;
  int x = (int)(e % cap);
  if (x >= cnt[i]) return;
  int32_t j = cand[e];
  unsigned long long p = atomicAdd(reinterpret_cast<unsigned long long*>(rev_cur + j), 1ull);
  rev[rev_off[j] + (int64_t)p] = (int32_t)i;
}

// Per target j (warp): append the smallest non-duplicate reverse sources to cand[j] until it
// holds `cap` entries.  fwd_cnt = forward counts (before any append).
constexpr int kSelChunk = 256;
__global__ void rev_select_kernel(int32_t* cand, int32_t* cnt, const int32_t* fwd_cnt, int64_t n,
                                  int cap, const int64_t* rev_off, const int64_t* rev_num,
                                  const int32_t* rev, int tpad) {
  extern __shared__ __align__(16) char smem_raw[];
  const int wpb = blockDim.x >> 5;
  const size_t per_warp = (size_t)tpad * 12 + (size_t)kSelChunk * 16 + (size_t)cap * 4;
  char* base = smem_raw + per_warp * warp_id();
  double* ld = reinterpret_cast<double*>(base);
  double* cd = ld + tpad;
  uint32_t* li = reinterpret_cast<uint32_t*>(cd + kSelChunk);
  uint32_t* ci = li + tpad;
  int* cp = reinterpret_cast<int*>(ci + kSelChunk);
  int32_t* fw = reinterpret_cast<int32_t*>(cp + kSelChunk);
  int64_t j = (int64_t)blockIdx.x * wpb + warp_id();
  if (j >= n) return;
  const int lane = lane_id();
  const int fc = fwd_cnt[j];
  const int room = cap - fc;
  const int64_t S = rev_num[j];
  if (room <= 0 || S == 0) return;
  const int32_t* seg = rev + rev_off[j];
  // the smallest T = min(S, room + fc) sources suffice: at most fc of them are duplicates
  int T = (int)(S < (int64_t)(room + fc) ? S : (int64_t)(room + fc));
  for (int t = lane; t < fc; t += 32) fw[t] = cand[j * cap + t];
  for (int t = lane; t < T; t += 32) {
    ld[t] = __longlong_as_double(0x7FF0000000000000ll);
    li[t] = 0xFFFFFFFFu;
  }
  __syncwarp();
  for (int64_t b = 0; b < S; b += kSelChunk) {
    int c = (int)(S - b < kSelChunk ? S - b : kSelChunk);
    for (int t = lane; t < c; t += 32) {
      uint32_t v = (uint32_t)seg[b + t];
      cd[t] = (double)v;
      ci[t] = v;
    }
    __syncwarp();
    warp_merge_topk(ld, li, T, cd, ci, cp, c, 0xFFFFFFFFu);
  }
  // ascending sources; skip those already in the forward list; append until full
  int appended = 0;
  for (int b = 0; b < T && appended < room; b += 32) {
    int t = b + lane;
    bool ok = false;
    uint32_t v = 0;
    if (t < T) {
      v = li[t];
      ok = true;
      for (int u = 0; u < fc; ++u)
        if ((uint32_t)fw[u] == v) { ok = false; break; }
    }
    unsigned bal = __ballot_sync(0xffffffffu, ok);
    int pos = appended + __popc(bal & ((1u << lane) - 1u));
    if (ok && pos < room) cand[j * cap + fc + pos] = (int32_t)v;
    appended += __popc(bal);
  }
  if (lane == 0) cnt[j] = fc + (appended < room ? appended : room);
}

int launch_build_candidates(const int32_t* ids, uint8_t* flags, int64_t n, int g, int gn,
                            int32_t* new_cand, int32_t* new_cnt, int32_t* old_cand,
                            int32_t* old_cnt, BuildScratch& s, cudaStream_t st) {
  {
    int wpb = 8;
    cand_forward_kernel<<<(unsigned)((n + wpb - 1) / wpb), wpb * 32, 0, st>>>(
        ids, flags, n, g, gn, new_cand, new_cnt, old_cand, old_cnt);
  }
  cudaMemcpyAsync(s.fwd_new, new_cnt, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(s.fwd_old, old_cnt, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st);
  for (int pass = 0; pass < 2; ++pass) {
    int32_t* cand = pass == 0 ? new_cand : old_cand;
    int32_t* cnt = pass == 0 ? new_cnt : old_cnt;
    const int32_t* fwd = pass == 0 ? s.fwd_new : s.fwd_old;
    int cap = pass == 0 ? gn : g;
    int64_t tot = n * (int64_t)cap;
    cudaMemsetAsync(s.rev_cnt, 0, sizeof(int64_t) * n, st);
    rev_count_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(cand, fwd, n, cap, s.rev_cnt);
    exclusive_scan(s.rev_cnt, s.rev_off, n, s.scan_tmp, st);
    cudaMemsetAsync(s.rev_cur, 0, sizeof(int64_t) * n, st);
    rev_scatter_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(cand, fwd, n, cap, s.rev_off,
                                                                       s.rev_cur, s.rev);
    int tpad = next_pow2(2 * cap);
    int wpb = 4;
    size_t per_warp = (size_t)tpad * 12 + (size_t)kSelChunk * 16 + (size_t)cap * 4;
    size_t smem = per_warp * wpb;
    cudaFuncSetAttribute(rev_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    rev_select_kernel<<<(unsigned)((n + wpb - 1) / wpb), wpb * 32, smem, st>>>(
        cand, cnt, fwd, n, cap, s.rev_off, s.rev_cnt, s.rev, tpad);
  }
  return (int)cudaGetLastError();
}

}  // namespace sb

// help_join.cu — HELP build, part 2: the NN-descent local join (_kernels.py:138-173).
//
// The reference pushes, for every candidate pair (j, k) of every node i (new x new with
// x < y, new x old), k into row j and j into row k with _heap_push (_kernels.py:38-68).
// Restated order-independently: each row ends as the top-gamma, under the
// (f32 dist, id) key, of (its entries before the join) ∪ (everything pushed to it), and an
// id gets flag 1 iff it was not in the row before the join.  Pushes that do not beat the
// row's current tail can never survive, so they are filtered at the source.
//
// Pipeline per node chunk (chunks are sized so the worst-case push count fits the buffer):
//   emit     persistent CTAs take nodes i; gather the candidate rows (new ∪ old) into shared
//            memory; each thread evaluates a 4 x 4 tile of pairs as 16 independent fp64 chains
//            in ascending dimension order (bit-exact _pair_dist); pushes that beat the target
//            row's tail are appended (target, key) to a global buffer, and counted per target.
//   scatter  counting sort of the pushes into per-row segments.
//   merge    warp per touched row: chunks of its segment are filtered against the tail,
//            sorted, de-duplicated (identical keys = identical (dist, id): distances are
//            computed by one canonical exact function, so a repeated id has the same key)
//            and merged into the row; flags of surviving old entries are kept, new ids get 1.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "sb_internal.h"

namespace sb {

constexpr int kJoinThreads = 256;
constexpr int kJT = 4;            // pair tile edge
constexpr int kEmitBlock = 1024;  // push slots a warp reserves at a time (<= 6% padding)

struct JoinCta {
  int32_t* slot_id;   // [spad]
  int32_t* slot_attr; // [spad * l]
  float* xs;          // [dc][spad] (u8 path: uint32 words [m / 4][spad])
  int* tiles;         // tile list
  int32_t* nrm;       // [spad] |x|^2 (u8 path)
  uint64_t* thr;      // [spad] the slots' row tails (push filter)
};

// warp-aggregated append of up to two pushes per lane into the global push buffer
struct Emitter {
  uint64_t base;  // current reserved block start
  int used;       // slots used in the block (warp-uniform)
};

SB_DEV void emit2(const JoinArgs& a, Emitter& em, bool p1, uint32_t t1, uint64_t k1, bool p2,
                  uint32_t t2, uint64_t k2) {
  const int lane = lane_id();
  int cnt = (int)p1 + (int)p2;
  // inclusive warp scan
  int inc = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  int total = __shfl_sync(0xffffffffu, inc, 31);
  if (total == 0) return;
  int excl = inc - cnt;
  if (em.used + total > kEmitBlock) {
    // pad out the rest of the block, reserve a new one
    for (int s = em.used + lane; s < kEmitBlock; s += 32)
      if (em.base + s < a.push_cap) a.push_tgt[em.base + s] = 0xFFFFFFFFu;
    uint64_t nb = 0;
    if (lane == 0) nb = atomicAdd(reinterpret_cast<unsigned long long*>(a.push_count), (unsigned long long)kEmitBlock);
    em.base = __shfl_sync(0xffffffffu, nb, 0);
    em.used = 0;
  }
  uint64_t pos = em.base + em.used + excl;
  if (pos + cnt <= a.push_cap) {
    if (p1) {
      a.push_tgt[pos] = t1;
      a.push_key[pos] = k1;
      atomicAdd(reinterpret_cast<unsigned long long*>(a.row_cnt + t1), 1ull);
      ++pos;
    }
    if (p2) {
      a.push_tgt[pos] = t2;
      a.push_key[pos] = k2;
      atomicAdd(reinterpret_cast<unsigned long long*>(a.row_cnt + t2), 1ull);
    }
  } else if (cnt) {
    atomicExch(a.overflow, 1);
  }
  em.used += total;
}

// U8: integer features in [0, 255]: the slots' rows are staged as u8 words and each pair's
// S = |x|^2 + |y|^2 - 2 x.y comes from byte dot products (dp4a), exact in int32 and equal to
// the reference's fp64 sum of squares.
template <bool U8>
__global__ void __launch_bounds__(kJoinThreads, U8 ? 3 : 2) join_emit_kernel(JoinArgs a) {
  extern __shared__ __align__(16) char smem_raw[];
  const int spad = a.spad;
  JoinCta s;
  {
    char* p = smem_raw;
    s.thr = reinterpret_cast<uint64_t*>(p); p += sizeof(uint64_t) * (size_t)spad;
    s.xs = reinterpret_cast<float*>(p); p += sizeof(float) * (size_t)a.dc * spad;
    s.slot_id = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * spad;
    s.slot_attr = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * (size_t)spad * a.l;
    s.tiles = reinterpret_cast<int*>(p); p += sizeof(int) * (size_t)a.ntiles_max;
    s.nrm = reinterpret_cast<int32_t*>(p);
  }
  __shared__ int sh_node[2];
  const int tid = threadIdx.x;
  Emitter em;
  em.base = 0;
  em.used = kEmitBlock;  // forces a reservation on first use
  const bool whole = a.dc >= a.m;  // all dimensions staged at once
  unsigned same = 0;  // (x, y) slots holding one id twice (in both the new and the old list)

  // the node after the current one is claimed while the current one is processed (the counter's
  // round trip and two barriers per node left the critical path)
  auto claim = [&]() {
    const int64_t i = a.node_begin + atomicAdd(a.node_counter, 1);
    return i < a.node_end ? (int)i : -1;
  };
  if (tid == 0) sh_node[0] = claim();
  for (int it = 0;; ++it) {
    __syncthreads();  // the claim is visible; the previous node's shared-memory reads are done
    const int node = sh_node[it & 1];
    if (node < 0) break;
    if (tid == 0) sh_node[(it + 1) & 1] = claim();
    const int na = __ldg(a.new_cnt + node), nb = __ldg(a.old_cnt + node);
    const int ns = na + nb;
    if (na == 0) continue;
    for (int t = tid; t < ns; t += blockDim.x) {
      int32_t v = t < na ? a.new_cand[(int64_t)node * a.gn + t] : a.old_cand[(int64_t)node * a.g + (t - na)];
      s.slot_id[t] = v;
      s.thr[t] = a.thr[v];
      for (int u = 0; u < a.l; ++u) s.slot_attr[t * a.l + u] = __ldg(a.A + (int64_t)v * a.l + u);
    }
    for (int t = ns + tid; t < spad; t += blockDim.x) s.slot_id[t] = -1;
    // tile list: row block rb (x in [4rb, 4rb+4) ⊂ new), col block cb (y in [4cb, 4cb+4)),
    // keep tiles holding at least one pair with y > x, y < ns
    // (row block rb owns the ncb - rb tiles from offset rb ncb - rb (rb - 1) / 2: the threads
    // fill the list row block by row block, eight threads per row block)
    const int nrb = (na + kJT - 1) / kJT, ncb = (ns + kJT - 1) / kJT;
    for (int rb = tid >> 3; rb < nrb; rb += blockDim.x >> 3) {
      const int off = rb * ncb - rb * (rb - 1) / 2 - rb;
      for (int cb = rb + (tid & 7); cb < ncb; cb += 8) s.tiles[off + cb] = (rb << 16) | cb;
    }
    __syncthreads();
    const int ntiles = nrb * ncb - nrb * (nrb - 1) / 2;
    // whole rows staged once per node, transposed into [word][slot], by 4-byte asynchronous
    // copies (a warp per slot, lanes along the row: coalesced; every copy in flight at once)
    auto stage_whole = [&](const void* base, int64_t row_bytes, int nwords) {
      const int lane_ = tid & 31, nwarp = blockDim.x >> 5;
      for (int t = tid >> 5; t < ns; t += nwarp) {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(
            reinterpret_cast<const char*>(base) + (int64_t)s.slot_id[t] * row_bytes);
        for (int dw = lane_; dw < nwords; dw += 32)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                           (uint32_t)__cvta_generic_to_shared(s.xs + dw * spad + t)),
                       "l"(src + dw)
                       : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (U8) {
      stage_whole(a.F8, a.m, a.m >> 2);
      for (int t = tid; t < ns; t += blockDim.x) s.nrm[t] = __ldg(a.nx8 + s.slot_id[t]);
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();
    } else if (whole) {
      stage_whole(a.F, (int64_t)a.m * 4, a.m);
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();
    }
    for (int pass = 0; pass * kJoinThreads < ntiles; ++pass) {
      const int ti = pass * kJoinThreads + tid;
      const bool have = ti < ntiles;
      const int tile = have ? s.tiles[ti] : 0;
      const int rb = tile >> 16, cb = tile & 0xFFFF;
      double acc[kJT][kJT];
#pragma unroll
      for (int u = 0; u < kJT; ++u)
#pragma unroll
        for (int w = 0; w < kJT; ++w) acc[u][w] = 0.0;
      if (U8) {
        unsigned dot[kJT][kJT];
#pragma unroll
        for (int u = 0; u < kJT; ++u)
#pragma unroll
          for (int w = 0; w < kJT; ++w) dot[u][w] = 0u;
        if (have) {
          const uint32_t* xw = reinterpret_cast<const uint32_t*>(s.xs);
          for (int dw = 0; dw < (a.m >> 2); ++dw) {
            const uint4 xv = *reinterpret_cast<const uint4*>(xw + dw * spad + rb * kJT);
            const uint4 yv = *reinterpret_cast<const uint4*>(xw + dw * spad + cb * kJT);
            const uint32_t xx[4] = {xv.x, xv.y, xv.z, xv.w};
            const uint32_t yy[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
            for (int u = 0; u < kJT; ++u)
#pragma unroll
              for (int w = 0; w < kJT; ++w) dot[u][w] = __dp4a(xx[u], yy[w], dot[u][w]);
          }
#pragma unroll
          for (int u = 0; u < kJT; ++u)
#pragma unroll
            for (int w = 0; w < kJT; ++w) {
              const int x = rb * kJT + u, y = cb * kJT + w;
              const int nx_ = x < ns ? s.nrm[x] : 0, ny_ = y < ns ? s.nrm[y] : 0;
              acc[u][w] = (double)(nx_ + ny_ - 2 * (int)dot[u][w]);
            }
        }
      }
      // one 4x4 tile's sums over the dimensions staged at xs_ (dc_ rows of spad floats)
      auto tile_dims = [&](const float* xs_, int dc_) {
        for (int dd = 0; dd < dc_; ++dd) {
          const float* row = xs_ + (size_t)dd * spad;
          float4 xv = *reinterpret_cast<const float4*>(row + rb * kJT);
          float4 yv = *reinterpret_cast<const float4*>(row + cb * kJT);
          const double xx[4] = {(double)xv.x, (double)xv.y, (double)xv.z, (double)xv.w};
          const double yy[4] = {(double)yv.x, (double)yv.y, (double)yv.z, (double)yv.w};
#pragma unroll
          for (int u = 0; u < kJT; ++u)
#pragma unroll
            for (int w = 0; w < kJT; ++w) acc[u][w] = sq_step(acc[u][w], xx[u], yy[w]);
        }
      };
      if (!U8 && whole) {
        if (have) tile_dims(s.xs, a.m);
      } else if (!U8) {
        // Dimension chunks through two half stages: the 4-byte asynchronous copies of chunk
        // c + 1 (a warp per slot, lanes along the dimensions: coalesced, transposed into
        // [dimension][slot]) run under the pair sums of chunk c.  (A load -> store staging loop
        // spent half of this kernel's stall samples waiting for one load per thread:
        // profiles/README.md.)
        const int dch = a.dc >> 1;
        const int lane_ = tid & 31, nwarp = blockDim.x >> 5;
        auto stage = [&](int c) {
          const int d0 = c * dch;
          const int dc_ = a.m - d0 < dch ? a.m - d0 : dch;
          float* dst = s.xs + (size_t)(c & 1) * dch * spad;
          for (int t = tid >> 5; t < ns; t += nwarp) {
            const float* src = a.F + (int64_t)s.slot_id[t] * a.m + d0;
            for (int dd = lane_; dd < dc_; dd += 32)
              asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                               (uint32_t)__cvta_generic_to_shared(dst + dd * spad + t)),
                           "l"(src + dd)
                           : "memory");
          }
          asm volatile("cp.async.commit_group;" ::: "memory");
        };
        const int nchunk = (a.m + dch - 1) / dch;
        __syncthreads();  // the previous pass is done with both half stages
        stage(0);
        for (int c = 0; c < nchunk; ++c) {
          if (c + 1 < nchunk) {
            stage(c + 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
          } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
          }
          __syncthreads();  // chunk c has landed for every thread
          const int d0 = c * dch;
          if (have) tile_dims(s.xs + (size_t)(c & 1) * dch * spad, a.m - d0 < dch ? a.m - d0 : dch);
          __syncthreads();  // its half stage may be overwritten (by chunk c + 2)
        }
      }
      // pushes (warp-uniform loop; lanes without a tile contribute nothing).  The tile's rows
      // go through one copy of the push code (the accumulator rows rotate through acc[0], so
      // the indices stay static): a quarter of the instructions of the fully unrolled form,
      // which stalled on instruction fetch (16% of the u8 kernel's samples).
#pragma unroll 1
      for (int u = 0; u < kJT; ++u) {
#pragma unroll
        for (int w = 0; w < kJT; ++w) {
          const int x = rb * kJT + u, y = cb * kJT + w;
          bool valid = have && x < na && y < ns && y > x;
          int32_t j = valid ? s.slot_id[x] : 0;
          int32_t k = valid ? s.slot_id[y] : 0;
          same += (valid && j == k) ? 1u : 0u;
          valid = valid && j != k;
          bool p1 = false, p2 = false;
          uint64_t k1 = 0, k2 = 0;
          if (valid) {
            double sa = 0.0;
            for (int t = 0; t < a.l; ++t)
              sa = dadd(sa, fabs(dsub((double)s.slot_attr[x * a.l + t], (double)s.slot_attr[y * a.l + t])));
            float d = __double2float_rn(auto_finish(acc[0][w], sa, a.inv_alpha));
            k1 = row_key(d, (uint32_t)k);  // into row j
            k2 = row_key(d, (uint32_t)j);  // into row k
            p1 = k1 < s.thr[x];
            p2 = k2 < s.thr[y];
          }
          emit2(a, em, p1, (uint32_t)j, k1, p2, (uint32_t)k, k2);
        }
#pragma unroll
        for (int r = 0; r + 1 < kJT; ++r)
#pragma unroll
          for (int w = 0; w < kJT; ++w) acc[r][w] = acc[r + 1][w];
      }
    }
  }
  if (same) atomicAdd(a.same_pairs, (unsigned long long)same);
  // pad this warp's unused reservation
  const int lane = lane_id();
  if (em.used < kEmitBlock)
    for (int s2 = em.used + lane; s2 < kEmitBlock; s2 += 32)
      if (em.base + s2 < a.push_cap) a.push_tgt[em.base + s2] = 0xFFFFFFFFu;
}

// ---------------------------------------------------------------------------
__global__ void push_scatter_kernel(const uint32_t* tgt, const uint64_t* key, uint64_t total,
                                    const int64_t* row_off, int64_t* row_cur, uint64_t* seg) {
  uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  uint32_t t = tgt[e];
  if (t == 0xFFFFFFFFu) return;
  unsigned long long p = atomicAdd(reinterpret_cast<unsigned long long*>(row_cur + t), 1ull);
  seg[row_off[t] + (int64_t)p] = key[e];
}

// ---------------------------------------------------------------------------
// merge a row's pushes into it (warp per row)
constexpr int kMergeChunk = 256;

__global__ void row_merge_kernel(int32_t* ids, float* dists, uint8_t* flags, uint64_t* thr,
                                 int64_t n, int g, int gpad, const int64_t* row_off,
                                 const int64_t* row_cnt, const uint64_t* seg,
                                 unsigned long long* inserted) {
  extern __shared__ __align__(16) char smem_raw[];
  const int wpb = blockDim.x >> 5;
  const size_t per_warp = (size_t)gpad * 9 + (size_t)kMergeChunk * 12 + 16;
  char* base = smem_raw + ((per_warp + 15) & ~(size_t)15) * warp_id();
  uint64_t* L = reinterpret_cast<uint64_t*>(base);
  uint64_t* C = L + gpad;
  int* cpos = reinterpret_cast<int*>(C + kMergeChunk);
  uint8_t* LF = reinterpret_cast<uint8_t*>(cpos + kMergeChunk);
  int64_t r = (int64_t)blockIdx.x * wpb + warp_id();
  if (r >= n) return;
  const int64_t S = row_cnt[r];
  if (S == 0) return;
  const int lane = lane_id();
  const unsigned lt = (1u << lane) - 1u;
  for (int t = lane; t < g; t += 32) {
    L[t] = row_key(dists[r * g + t], (uint32_t)ids[r * g + t]);
    LF[t] = flags[r * g + t];
  }
  __syncwarp();
  const uint64_t* sg = seg + row_off[r];
  int new_total = 0;
  for (int64_t b = 0; b < S; b += kMergeChunk) {
    const int c = (int)(S - b < kMergeChunk ? S - b : kMergeChunk);
    const uint64_t tail = L[g - 1];
    // 1. load + filter (strictly below the tail)
    int kept = 0;
    for (int o = 0; o < c; o += 32) {
      int t = o + lane;
      uint64_t k = t < c ? sg[b + t] : kKeyInf;
      bool ok = k < tail;
      unsigned bal = __ballot_sync(0xffffffffu, ok);
      if (ok) C[kept + __popc(bal & lt)] = k;
      kept += __popc(bal);
    }
    __syncwarp();
    if (kept == 0) continue;
    // 2. sort
    int np = next_pow2(kept);
    for (int t = kept + lane; t < np; t += 32) C[t] = kKeyInf;
    __syncwarp();
    if (np > 1) warp_bitonic_u64(C, np);
    // 3. de-duplicate (within the chunk, and against the row) and compact
    int uniq = 0;
    for (int o = 0; o < kept; o += 32) {
      int t = o + lane;
      uint64_t k = 0;
      bool ok = false;
      if (t < kept) {
        k = C[t];
        ok = (t == 0 || C[t - 1] != k);
        if (ok) {
          int p = lower_bound_u64(L, g, k);
          ok = !(p < g && L[p] == k);
        }
      }
      unsigned bal = __ballot_sync(0xffffffffu, ok);
      __syncwarp();
      if (ok) C[uniq + __popc(bal & lt)] = k;
      uniq += __popc(bal);
      __syncwarp();
    }
    if (uniq == 0) continue;
    // 4. merge: candidate j -> j + #{L < C[j]}; L[i] -> i + #{C < L[i]}
    for (int t = lane; t < uniq; t += 32) cpos[t] = t + lower_bound_u64(L, g, C[t]);
    __syncwarp();
    const int first = cpos[0];
    if (first >= g) continue;
    for (int top = g - 1; top >= first; top -= 32) {
      int i = top - lane;
      bool act = i >= first;
      uint64_t k = 0;
      uint8_t f = 0;
      int tg = g;
      if (act) {
        k = L[i];
        f = LF[i];
        tg = i + lower_bound_u64(C, uniq, k);
      }
      __syncwarp();
      if (act && tg < g) { L[tg] = k; LF[tg] = f; }
      __syncwarp();
    }
    int ins = 0;
    for (int t = lane; t < uniq; t += 32) {
      int p = cpos[t];
      if (p < g) { L[p] = C[t]; LF[p] = 1; ++ins; }
    }
    new_total += warp_sum(ins);
    __syncwarp();
  }
  if (new_total == 0) return;
  for (int t = lane; t < g; t += 32) {
    ids[r * g + t] = (int32_t)key_id(L[t]);
    dists[r * g + t] = key_dist(L[t]);
    flags[r * g + t] = LF[t];
  }
  if (lane == 0) {
    thr[r] = L[g - 1];
    atomicAdd(inserted, (unsigned long long)new_total);
  }
}

__global__ void thr_init_kernel(const int32_t* ids, const float* dists, int64_t n, int g,
                                uint64_t* thr) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  thr[r] = row_key(dists[r * g + g - 1], (uint32_t)ids[r * g + g - 1]);
}

size_t join_emit_smem(int spad, int dc, int l, int ntiles_max) {
  return sizeof(uint64_t) * (size_t)spad + sizeof(float) * (size_t)dc * spad + sizeof(int32_t) * spad +
         sizeof(int32_t) * (size_t)spad * l + sizeof(int) * (size_t)ntiles_max +
         sizeof(int32_t) * spad + 64;
}

int launch_thr_init(const int32_t* ids, const float* dists, int64_t n, int g, uint64_t* thr,
                    cudaStream_t st) {
  thr_init_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ids, dists, n, g, thr);
  return (int)cudaGetLastError();
}

int launch_join_emit(const JoinArgs& a, int ctas, size_t smem, cudaStream_t st) {
  auto kern = a.F8 ? join_emit_kernel<true> : join_emit_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  kern<<<ctas, kJoinThreads, smem, st>>>(a);
  return (int)cudaGetLastError();
}

int join_emit_occupancy(size_t smem, int* ctas_per_sm) {
  cudaFuncSetAttribute(join_emit_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(join_emit_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int a = 0, b = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, join_emit_kernel<false>,
                                                                kJoinThreads, smem);
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, join_emit_kernel<true>, kJoinThreads, smem);
  *ctas_per_sm = a < b ? a : b;
  return (int)e;
}

int launch_push_scatter(const uint32_t* tgt, const uint64_t* key, uint64_t total,
                        const int64_t* row_off, int64_t* row_cur, uint64_t* seg, cudaStream_t st) {
  if (total == 0) return 0;
  push_scatter_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(tgt, key, total, row_off,
                                                                        row_cur, seg);
  return (int)cudaGetLastError();
}

int launch_row_merge(int32_t* ids, float* dists, uint8_t* flags, uint64_t* thr, int64_t n, int g,
                     const int64_t* row_off, const int64_t* row_cnt, const uint64_t* seg,
                     unsigned long long* inserted, cudaStream_t st) {
  int gpad = next_pow2(g);
  int wpb = 4;
  size_t per_warp = (size_t)gpad * 9 + (size_t)kMergeChunk * 12 + 16;
  per_warp = (per_warp + 15) & ~(size_t)15;
  size_t smem = per_warp * wpb;
  cudaFuncSetAttribute(row_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  row_merge_kernel<<<(unsigned)((n + wpb - 1) / wpb), wpb * 32, smem, st>>>(
      ids, dists, flags, thr, n, g, gpad, row_off, row_cnt, seg, inserted);
  return (int)cudaGetLastError();
}

}  // namespace sb

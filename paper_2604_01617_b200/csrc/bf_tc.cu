// bf_tc.cu — exhaustive AUTO top-k on the 5th-generation tensor cores (tcgen05 + TMEM),
// query mode (oracle_auto_topk, evaluate.py:32-55) for integer-valued data.
//
// Exactness: when features and queries are integers with d * max(|x|,|q|)^2 < 2^24, every
// bf16 operand is exact and every partial dot product in the fp32 TMEM accumulator is an
// integer below 2^24, so x.q is exact whatever order the tensor core adds in.  Then
//   S = |x|^2 + |q|^2 - 2 x.q            (int32, exact)
// equals the reference's fp64 sum of squared differences exactly, and
//   U = sqrt(S) * (1 + s_a / alpha)       (fp64, as evaluate.py:48-53)
// is bit-identical to the reference's value.  No re-rank is needed; the split merge
// (bf_merge_kernel) recomputes the kept candidates in NumPy order, which changes nothing.
//
// CTA = 128 queries (one per TMEM lane) x a range of node tiles (N = 256 or 128 nodes).
// A producer thread bulk-copies each tile's bf16 rows and per-node metadata into one of two
// shared-memory stages and issues d/16 tcgen05.mma (M=128, N, K=16, BF16 -> F32) into one of
// two TMEM accumulators; 256 epilogue threads (two per query, one per column half) read the
// dot products with tcgen05.ld while the next tile loads and multiplies, and keep private
// top-kk lists.  A node can enter a list only if S * f^2 <= T^2 (f = 1 + s_a/alpha), so the
// epilogue mostly costs one fp32 compare per (query, node).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <limits.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "tc_ptx.cuh"
#include "sb_internal.h"

#include <cub/device/device_radix_sort.cuh>

namespace sb {

constexpr int kTcM = 128;       // queries per CTA (UMMA M)
constexpr int kTcThreads = 256;  // two threads per query row, each owning half the columns
constexpr int kTcMaxKK = 32;    // per-thread list length limit
constexpr int kTcPad = 256;     // node arrays are zero-padded to a multiple of this
constexpr int kTcMeta = 4;      // node-metadata ring stages (ahead of the accumulators)

// Operand layout in HBM and shared memory (both operands, identical): K-major core matrices in
// row-group-major order.  The 8 rows of group g occupy one contiguous 8 * m * 2-byte block;
// inside it, 16-byte k-chunk kc of row r sits at kc * 128 + (r & 7) * 16.  A tile of N rows is
// therefore N/8 consecutive groups, whatever N is, and lands in shared memory with one bulk
// copy.  UMMA descriptor per 16-wide k-step s: start = base + 2 s * 128, LBO (next k-chunk)
// = 128 B, SBO (next 8-row group) = m / 8 * 128 B.
SB_DEV size_t rg_off(int64_t row, int kc, int m) {
  return (size_t)(row >> 3) * (size_t)(8 * m * 2) + (size_t)kc * 128 + (size_t)(row & 7) * 16;
}
// the same layout for 8-bit operands: a 16-byte chunk holds 16 elements, rows are m bytes
SB_DEV size_t rg_off8(int64_t row, int t, int m) {
  return (size_t)(row >> 3) * (size_t)(8 * m) + (size_t)(t >> 4) * 128 + (size_t)(row & 7) * 16 +
         (size_t)(t & 15);
}

// ---- prep kernels ----------------------------------------------------------------------
// queries -> bf16 in the row-group layout of K = mk columns (rows up to qpad, zero past q)
// + exact |q|^2.  Folded operands (mk = m + 16): columns 0..m-1 hold 2q, columns m..m+2 hold
// -2^16, -2^8, -1 (all exact in bf16), so that against a node row ending in the three bytes
// of |x|^2 the tensor core produces y = 2 x.q - |x|^2 directly.
__global__ void tc_prep_queries_kernel(const double* qf, int64_t q, int64_t qpad, int m, int mk,
                                       char* Qb, int32_t* nq) {
  int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id();
  if (i >= qpad) return;
  const bool fold = mk > m;
  int acc = 0;
  for (int t = lane_id(); t < mk; t += 32) {
    float x = 0.f;
    if (t < m) {
      const double v = i < q ? qf[i * m + t] : 0.0;
      acc += (int)v * (int)v;
      x = fold ? 2.0f * (float)v : (float)v;
    } else if (t == m) {
      x = -65536.f;
    } else if (t == m + 1) {
      x = -256.f;
    } else if (t == m + 2) {
      x = -1.f;
    }
    reinterpret_cast<__nv_bfloat16*>(Qb + rg_off(i, t >> 3, mk))[t & 7] = __float2bfloat16_rn(x);
  }
  acc = warp_sum(acc);
  if (lane_id() == 0 && i < q) nq[i] = acc;
}

// u8 operands: queries and node rows as bytes in the row-group layout (m-byte rows)
__global__ void tc_prep_queries_u8_kernel(const double* qf, int64_t q, int64_t qpad, int m,
                                          uint8_t* Qb, int32_t* nq) {
  int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id();
  if (i >= qpad) return;
  int acc = 0;
  for (int t = lane_id(); t < m; t += 32) {
    const int x = i < q ? (int)qf[i * m + t] : 0;
    Qb[rg_off8(i, t, m)] = (uint8_t)x;
    acc += x * x;
  }
  acc = warp_sum(acc);
  if (lane_id() == 0 && i < q) nq[i] = acc;
}

// ---- main kernel -------------------------------------------------------------------------
struct TcArgs {
  // node arrays in attribute-grouped order (tc_prepare): nodes with one attribute tuple are
  // contiguous, so the epilogue recomputes the attribute factor only when the tuple changes.
  // All node arrays are padded with zeros to a multiple of kTcPad nodes.
  const char* Fb;           // bf16 rows, row-group layout
  const int32_t* nx;        // |x|^2 as fp32 bits
  const int32_t* A;         // attributes, n x l
  const int32_t* code;      // attribute-tuple code (equal codes <=> equal tuples)
  const int32_t* orig;      // original node id
  const char* Qb;           // bf16 queries, row-group layout, padded to 128-row groups
  const int32_t* nq;        // q
  const int64_t* qa;        // q x l
  const int64_t* qmask;     // q x l or null
  int64_t n, q;
  int m, l, kk, splits, N;  // m = operand K (features, plus 16 folded columns when folded)
  double alpha;
  double* part_d;           // q x (2 splits) x kk
  uint32_t* part_i;
  int* gthr;                // q: best list-tail bound of the query over all CTAs (fp32 bits)
  // u8 path: per 16-node chunk {min |x|^2, the chunk's attribute code or -1 when mixed}; nodes
  // are ordered by |x|^2 inside each attribute tuple, so 2 max(x.q) - min |x|^2 bounds the
  // chunk's y tightly and skips it on raw accumulators
  const int2* cmeta;
  int nacc;                 // TMEM accumulators (2, or 4 for 64-node tiles)
};

// One CTA = 128 queries x one node range, 9 warps:
//   warps 0..7  epilogue: thread (row = tid % 128, half = tid / 128) reads its query's dot
//               products for half of each tile's columns from TMEM and keeps a top-kk list;
//   warp 8      producer: one thread bulk-copies tile i's bf16 rows into B stage i % 2 and its
//               per-node metadata into meta stage i % 2, and issues the tile's MMAs into TMEM
//               accumulator i % 2.
// Barriers per stage s: fullB (rows landed), fullM (metadata landed), done (MMAs complete:
// accumulator ready and B stage free again), empty (all 256 epilogue threads finished the
// tile: accumulator and metadata free).  Rows for tile i + 1 load while MMA i runs; MMA i + 1
// starts as soon as the epilogue leaves tile i - 1.
// NBS = shared-memory stages for node rows (1 or 2), CTAS = CTAs per SM the shape is sized
// for (the other CTA's epilogue covers this one's waits)
// KIND: 0 = bf16 operands, 1 = bf16 with |x|^2 folded into the MMA, 2 = u8 operands
// (tcgen05 kind::i8, exact int32 accumulation; integer data in [0, 255])
template <int KIND, int NBS, int CTAS>
__global__ void __launch_bounds__(kTcThreads + 32, CTAS) bf_tc_kernel(TcArgs a) {
  constexpr bool FOLD = KIND == 1;
  constexpr bool U8 = KIND == 2;
  constexpr int ESZ = U8 ? 1 : 2;  // operand bytes per element
  extern __shared__ __align__(1024) char smem[];
  const int tid = threadIdx.x;
  const int m = a.m, N = a.N, l = a.l;
  const int rowb = m * ESZ;        // operand bytes per row
  const size_t b_bytes = (size_t)N * rowb;
  const size_t meta_bytes = (size_t)N * (3 + l) * 4 + (U8 ? (size_t)(N / 16) * 8 : 0);
  // shared layout: A tile | 2 x B tile | 2 x (nx | code | orig | attrs) | lists | t2 | barriers
  char* p = smem;
  char* sA = p; p += (size_t)kTcM * rowb;
  char* sB = p; p += NBS * b_bytes;
  char* sM = p; p += kTcMeta * meta_bytes;
  double* ld = reinterpret_cast<double*>(p); p += sizeof(double) * (size_t)a.kk * kTcThreads;
  uint32_t* li = reinterpret_cast<uint32_t*>(p); p += sizeof(uint32_t) * (size_t)a.kk * kTcThreads;
  volatile float* s_t2 = reinterpret_cast<float*>(p); p += sizeof(float) * kTcThreads;
  p = reinterpret_cast<char*>(((uintptr_t)p + 7) & ~(uintptr_t)7);
  uint64_t* bars = reinterpret_cast<uint64_t*>(p); p += 8 * 32;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(p);
  // fullB[4] done[2] empty[2] a fullM[kTcMeta] emptyM[kTcMeta] freeB[4]
  // fullB[4] done[4] empty[4] a fullM[kTcMeta] emptyM[kTcMeta] freeB[4]
  const uint32_t bar_fullB = smem_u32(bars), bar_done = smem_u32(bars + 4),
                 bar_empty = smem_u32(bars + 8), bar_a = smem_u32(bars + 12),
                 bar_fullM = smem_u32(bars + 13), bar_emptyM = smem_u32(bars + 13 + kTcMeta),
                 bar_freeB = smem_u32(bars + 13 + 2 * kTcMeta);
  const int nacc = a.nacc;  // TMEM accumulators in the MMA -> epilogue ring (2 or 4)

  const int64_t q0 = (int64_t)blockIdx.x * kTcM;
  const int64_t tiles = (a.n + N - 1) / N;
  const int64_t per = (tiles + a.splits - 1) / a.splits;
  const int64_t t_begin = per * blockIdx.y;
  const int64_t t_end = t_begin + per < tiles ? t_begin + per : tiles;
  const int ntl = t_end > t_begin ? (int)(t_end - t_begin) : 0;

  if (warp_id() == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(nacc * N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == kTcThreads) {
    for (int s = 0; s < nacc; ++s) {
      mbar_init(bar_done + 8 * s, 1);
      mbar_init(bar_empty + 8 * s, kTcThreads);
    }
    for (int s = 0; s < 4; ++s) {
      mbar_init(bar_fullB + 8 * s, 1);
      mbar_init(bar_freeB + 8 * s, 1);
    }
    for (int s = 0; s < kTcMeta; ++s) {
      mbar_init(bar_fullM + 8 * s, 1);
      mbar_init(bar_emptyM + 8 * s, kTcThreads);
    }
    mbar_init(bar_a, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < kTcThreads) {
    for (int i = 0; i < a.kk; ++i) {
      ld[i * kTcThreads + tid] = __longlong_as_double(0x7FF0000000000000ll);
      li[i * kTcThreads + tid] = 0xFFFFFFFFu;
    }
    s_t2[tid] = 3.4e38f;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp_id() == kTcThreads / 32) {
    // ---------------- producer / MMA issuer ----------------
    if (lane_id() == 0) {
      const uint32_t a_bytes = (uint32_t)(kTcM * rowb);
      mbar_expect_tx(bar_a, a_bytes);
      bulk_g2s(smem_u32(sA), a.Qb + (size_t)q0 * rowb, a_bytes, bar_a);
      auto load_rows = [&](int i) {
        const int s = NBS == 1 ? 0 : (i % NBS);
        const int64_t v0 = (t_begin + i) * (int64_t)N;
        mbar_expect_tx(bar_fullB + 8 * s, (uint32_t)b_bytes);
        bulk_g2s(smem_u32(sB + s * b_bytes), a.Fb + (size_t)v0 * rowb, (uint32_t)b_bytes,
                 bar_fullB + 8 * s);
      };
      // NBS == 1: this lane loads each tile's rows once the previous MMA is done; NBS >= 2:
      // lane 2 keeps the ring of row stages full on its own (below)
      if (NBS == 1 && ntl > 0) load_rows(0);
      mbar_wait(bar_a, 0);
      // BF16 x BF16 -> F32, or U8 x U8 -> S32 (c_format bits [4,6), a/b formats [7,13))
      const uint32_t idesc = (U8 ? (2u << 4) : ((1u << 4) | (1u << 7) | (1u << 10))) |
                             ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kTcM >> 4) << 24);
      const uint32_t sbo = (uint32_t)(rowb / 16) * 128;
      for (int i = 0; i < ntl; ++i) {
        const int s = i % nacc;
        const uint32_t ph = (uint32_t)((i / nacc) & 1);
        // accumulator s: free once the epilogue has left tile i - nacc
        if (i >= nacc) mbar_wait(bar_empty + 8 * s, ph ^ 1u);
        const int sb = NBS == 1 ? 0 : i % NBS;
        mbar_wait(bar_fullB + 8 * sb, NBS == 1 ? (uint32_t)(i & 1) : (uint32_t)((i / NBS) & 1));
        tc_fence_after();
        const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB + sb * b_bytes);
        // one MMA per 32 bytes of K (16 bf16 or 32 u8 elements)
        for (int k = 0; k < rowb / 32; ++k) {
          uint64_t ad = umma_desc(a0 + (uint32_t)k * 256, 128, sbo);
          uint64_t bd = umma_desc(b0 + (uint32_t)k * 256, 128, sbo);
          if (U8)
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "setp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem + (uint32_t)(s * N)),
                "l"(ad), "l"(bd), "r"(idesc), "r"(k > 0 ? 1u : 0u));
          else
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "setp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem + (uint32_t)(s * N)),
                "l"(ad), "l"(bd), "r"(idesc), "r"(k > 0 ? 1u : 0u));
        }
        mma_commit(bar_done + 8 * s);
        if (NBS == 1) {
          // one stage: rows of tile i + 1 once MMA i has completed
          if (i + 1 < ntl) {
            mbar_wait(bar_done + 8 * s, ph);
            load_rows(i + 1);
          }
        } else {
          mma_commit(bar_freeB + 8 * sb);  // the stage refills as soon as these MMAs complete
        }
      }
    } else if (NBS >= 2 && lane_id() == 2) {
      // row loader: stage i % NBS gets tile i as soon as the MMAs of tile i - NBS are done, so
      // up to NBS tiles are in flight whatever the epilogue does (issuing the refill from the
      // MMA lane after MMA i - 1 left only NBS - 1 tiles of L2 latency covered)
      for (int i = 0; i < ntl; ++i) {
        const int sb = i % NBS;
        if (i >= NBS) mbar_wait(bar_freeB + 8 * sb, (uint32_t)(((i / NBS) - 1) & 1));
        const int64_t v0 = (t_begin + i) * (int64_t)N;
        mbar_expect_tx(bar_fullB + 8 * sb, (uint32_t)b_bytes);
        bulk_g2s(smem_u32(sB + sb * b_bytes), a.Fb + (size_t)v0 * rowb, (uint32_t)b_bytes, bar_fullB + 8 * sb);
      }
    } else if (lane_id() == 1) {
      // node metadata on its own ring, kTcMeta tiles ahead of the epilogue
      for (int i = 0; i < ntl; ++i) {
        const int ms = i % kTcMeta;
        if (i >= kTcMeta) mbar_wait(bar_emptyM + 8 * ms, (uint32_t)(((i / kTcMeta) - 1) & 1));
        const int64_t v0 = (t_begin + i) * (int64_t)N;
        char* meta = sM + ms * meta_bytes;
        const uint32_t fm = bar_fullM + 8 * ms;
        mbar_expect_tx(fm, (uint32_t)meta_bytes);
        bulk_g2s(smem_u32(meta), a.nx + v0, (uint32_t)(N * 4), fm);
        bulk_g2s(smem_u32(meta + N * 4), a.code + v0, (uint32_t)(N * 4), fm);
        bulk_g2s(smem_u32(meta + N * 8), a.orig + v0, (uint32_t)(N * 4), fm);
        bulk_g2s(smem_u32(meta + N * 12), a.A + v0 * l, (uint32_t)(N * l * 4), fm);
        if (U8) bulk_g2s(smem_u32(meta + (size_t)N * (3 + l) * 4), a.cmeta + v0 / 16, (uint32_t)(N / 16 * 8), fm);
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue ----------------
    const int row = tid & (kTcM - 1);  // query row = TMEM lane
    const int half = tid >> 7;         // which half of each tile's columns this thread owns
    const int64_t my_q = q0 + row;
    const bool qok = my_q < a.q;
    const double inf = __longlong_as_double(0x7FF0000000000000ll);
    const int32_t my_nq = qok ? a.nq[my_q] : 0;
    const float nqf = (float)my_nq;
    int32_t qa_row[8];
    int32_t qm_row[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      qa_row[u] = (qok && u < l) ? (int32_t)a.qa[my_q * l + u] : 0;
      qm_row[u] = (qok && u < l) ? (int32_t)(a.qmask ? a.qmask[my_q * l + u] : 1) : 0;
    }
    // Conservative fp32 filter.  The exact distance is d = sqrt(S) * (1 + sa/alpha) with
    // S = |x|^2 + |q|^2 - 2 x.q, so a node can beat the list tail T only if S * f^2 <= T^2
    // (f = 1 + sa * ia, ia <= 1/alpha), i.e. only if  y = 2 x.q - |x|^2 >= |q|^2 - T^2 / f^2.
    // t2 = T^2 (1 + 1e-5) and the 8-unit margin cover every fp32 rounding; survivors are
    // decided in exact integer / fp64 arithmetic below.
    const float ia = __double2float_rd(1.0 / a.alpha);
    float t2 = 3.4e38f;      // own list tail bound
    float t2_eff = 3.4e38f;  // min over both halves of this query
    int last_code = -2, sa = 0;
    float f2 = 1.0f, inv_f2 = 1.0f;
    float thr = -3.4e38f;    // y threshold for the current tuple and t2_eff
    const int cols = N >> 1;
    const uint32_t lane_base = tmem + ((uint32_t)((warp_id() & 3) * 32) << 16) + (uint32_t)(half * cols);
    float gnext = 3.4e38f;
    for (int i = 0; i < ntl; ++i) {
      const int s = i % nacc;
      const uint32_t ph = (uint32_t)((i / nacc) & 1);
      const int ms = i % kTcMeta;
      const char* meta = sM + ms * meta_bytes;
      const float* s_nx = reinterpret_cast<const float*>(meta);
      const int32_t* s_code = reinterpret_cast<const int32_t*>(meta) + N;
      const int32_t* s_orig = reinterpret_cast<const int32_t*>(meta) + 2 * N;
      const int32_t* s_at = reinterpret_cast<const int32_t*>(meta) + 3 * N;
      const int2* s_cm = reinterpret_cast<const int2*>(meta + (size_t)N * (3 + l) * 4);
      const int64_t vb = (t_begin + i) * (int64_t)N;
      const int nvalid = (int)(a.n - vb < N ? a.n - vb : N);
      // the query's tightest bound published by any CTA: the value loaded one tile ago (its
      // latency hides behind a whole tile), and the load for the next tile issued now
      const float gpre = gnext;
      gnext = qok ? __int_as_float(*reinterpret_cast<volatile int*>(a.gthr + my_q)) : 3.4e38f;
      mbar_wait(bar_fullM + 8 * ms, (uint32_t)((i / kTcMeta) & 1));
      mbar_wait(bar_done + 8 * s, ph);
      tc_fence_after();
      for (int c = 0; c < cols / 16; ++c) {
        uint32_t r[16];
        tmem_ld16(lane_base + (uint32_t)(s * N + c * 16), r);
        if (!qok) continue;
        const int c0 = half * cols + c * 16;
        // columns are in attribute-grouped order: if both ends of the chunk carry the current
        // tuple, the whole chunk does, and one threshold covers all 16 columns
        int2 cm = make_int2(0, -1);
        if (U8) cm = s_cm[c0 >> 4];
        const bool uniform = U8 ? cm.y == last_code : (s_code[c0] == last_code && s_code[c0 + 15] == last_code);
        unsigned cand = 0;
        if (U8) {
          // the chunk test on raw dot products: y_j = 2 x_j.q - |x_j|^2 <= 2 max x.q - min |x|^2
          // (exact int32; nodes sorted by |x|^2 inside a tuple keep the bound tight)
          const int thri0 = thr < -2.0e9f ? INT_MIN : (thr > 2.0e9f ? INT_MAX : __float2int_rd(thr));
          if (uniform) {
            int t5[6];
#pragma unroll
            for (int j = 0; j < 5; ++j)
              t5[j] = max(max((int)r[3 * j], (int)r[3 * j + 1]), (int)r[3 * j + 2]);
            t5[5] = (int)r[15];
            const int mr = max(max(max(t5[0], t5[1]), t5[2]), max(max(t5[3], t5[4]), t5[5]));
            if (2 * mr - cm.x < thri0) continue;
          }
          // int32 dot products and |x|^2: y = 2 x.q - |x|^2 and the test stay integer
          // (y >= thr  <=>  y >= floor(thr) for integer y, conservatively)
          const int32_t* s_nxi = reinterpret_cast<const int32_t*>(s_nx);
          int yi[21];  // 16 values + 5 partial maxima
          int mxi = INT_MIN;
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const int4 v = *reinterpret_cast<const int4*>(s_nxi + c0 + 4 * q4);
            yi[4 * q4 + 0] = 2 * (int)r[4 * q4 + 0] - v.x;
            yi[4 * q4 + 1] = 2 * (int)r[4 * q4 + 1] - v.y;
            yi[4 * q4 + 2] = 2 * (int)r[4 * q4 + 2] - v.z;
            yi[4 * q4 + 3] = 2 * (int)r[4 * q4 + 3] - v.w;
          }
#pragma unroll
          for (int j = 0; j < 5; ++j)  // tree of 3-input maxima: depth 3, not a 16-long chain
            yi[16 + j] = max(max(yi[3 * j], yi[3 * j + 1]), yi[3 * j + 2]);
          mxi = max(max(max(yi[16], yi[17]), yi[18]), max(max(yi[19], yi[20]), yi[15]));
          const int thri = thr < -2.0e9f ? INT_MIN : (thr > 2.0e9f ? INT_MAX : __float2int_rd(thr));
          if (uniform && mxi < thri) continue;
          if (uniform) {
#pragma unroll
            for (int j = 0; j < 16; ++j) cand |= (yi[j] >= thri ? 1u : 0u) << j;
          } else {
            cand = 0xFFFFu;  // mixed chunk: decide column by column below
          }
        } else {
          float y[16];
          float mx = -3.4e38f;
          if (FOLD) {
            // the accumulator already holds y = 2 x.q - |x|^2 (exact integers below 2^24)
#pragma unroll
            for (int j = 0; j < 16; ++j) y[j] = __uint_as_float(r[j]);
          } else {
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              const float4 v = *reinterpret_cast<const float4*>(s_nx + c0 + 4 * q4);
              y[4 * q4 + 0] = fmaf(2.0f, __uint_as_float(r[4 * q4 + 0]), -v.x);
              y[4 * q4 + 1] = fmaf(2.0f, __uint_as_float(r[4 * q4 + 1]), -v.y);
              y[4 * q4 + 2] = fmaf(2.0f, __uint_as_float(r[4 * q4 + 2]), -v.z);
              y[4 * q4 + 3] = fmaf(2.0f, __uint_as_float(r[4 * q4 + 3]), -v.w);
            }
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) mx = fmaxf(mx, y[j]);  // (bf16 path)
          if (uniform && mx < thr) continue;
          if (uniform) {
#pragma unroll
            for (int j = 0; j < 16; ++j) cand |= (y[j] >= thr ? 1u : 0u) << j;
          } else {
            cand = 0xFFFFu;  // mixed chunk: decide column by column below
          }
        }
        if (c0 + 16 > nvalid) cand &= (nvalid > c0) ? ((1u << (nvalid - c0)) - 1u) : 0u;
        while (cand) {
          const int j = __ffs(cand) - 1;
          cand &= cand - 1u;
          const int col = c0 + j;
          const int code = s_code[col];
          if (code != last_code) {  // new attribute tuple: its factor for this query
            last_code = code;
            int s2 = 0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (u < l) s2 += abs(s_at[col * l + u] - qa_row[u]) * qm_row[u];
            sa = s2;
            const float f = fmaf((float)sa, ia, 1.0f);
            f2 = f * f;
            inv_f2 = __frcp_ru(f2);
            thr = nqf - t2_eff * inv_f2 - 8.0f;
          }
          uint32_t rr = 0u;
#pragma unroll
          for (int jj = 0; jj < 16; ++jj)
            if (jj == j) rr = r[jj];
          // exact: x.q (or y when folded) is an integer below 2^24 held exactly by the fp32
          // accumulator, or an int32 (u8 operands)
          const int S = U8 ? reinterpret_cast<const int32_t*>(s_nx)[col] + my_nq - 2 * (int)rr
                      : FOLD ? my_nq - (int)__uint_as_float(rr)
                             : (int)s_nx[col] + my_nq - 2 * (int)__uint_as_float(rr);
          if ((float)S * f2 > t2_eff) continue;
          // exact fp64 decision (evaluate.py:48-53), ties by original id
          const double dist = dmul(sqrt((double)S), dadd(1.0, __ddiv_rn((double)sa, a.alpha)));
          const uint32_t vid = (uint32_t)s_orig[col];
          double wd = ld[(a.kk - 1) * kTcThreads + tid];
          uint32_t wi = li[(a.kk - 1) * kTcThreads + tid];
          if (!dlt(dist, vid, wd, wi)) continue;
          int pos = a.kk - 1;
          while (pos > 0) {
            double pd = ld[(pos - 1) * kTcThreads + tid];
            uint32_t pi = li[(pos - 1) * kTcThreads + tid];
            if (!dlt(dist, vid, pd, pi)) break;
            ld[pos * kTcThreads + tid] = pd;
            li[pos * kTcThreads + tid] = pi;
            --pos;
          }
          ld[pos * kTcThreads + tid] = dist;
          li[pos * kTcThreads + tid] = vid;
          const double t = ld[(a.kk - 1) * kTcThreads + tid];
          if (t < inf) {
            t2 = (float)(t * t * (1.0 + 1e-5));
            if (t2 < t2_eff) {
              t2_eff = t2;
              thr = nqf - t2_eff * inv_f2 - 8.0f;
              atomicMin(a.gthr + my_q, __float_as_int(t2));  // positive floats order as ints
            }
          }
        }
      }
      // release accumulator s and meta stage ms to the producers
      tc_fence_before();
      mbar_arrive(bar_empty + 8 * s);
      mbar_arrive(bar_emptyM + 8 * ms);
      // Share list tails between all partial lists of a query (the other column half in
      // this CTA, the other node ranges in other CTAs): a node beyond any list's kk-th
      // cannot enter the merged top-kk either, so the tightest bound filters every list.
      // Stale (larger) values only weaken the filter.
      s_t2[tid] = t2_eff;
      const float pt = fminf(s_t2[tid ^ kTcM], gpre);
      if (pt < t2_eff) {
        t2_eff = pt;
        thr = nqf - t2_eff * inv_f2 - 8.0f;
      }
    }
    // partial lists out: split index 2 * split + half
    if (qok) {
      const int sp = 2 * blockIdx.y + half;
      size_t o = ((size_t)my_q * (2 * a.splits) + sp) * a.kk;
      for (int i = 0; i < a.kk; ++i) {
        a.part_d[o + i] = ld[i * kTcThreads + tid];
        a.part_i[o + i] = li[i * kTcThreads + tid];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(nacc * N));
  }
}

// rowb = operand bytes per row (2 m for bf16, m for u8)
size_t bf_tc_smem_n(int rowb, int l, int kk, int N, int nbs) {
  return (size_t)kTcM * rowb + (size_t)nbs * N * rowb + kTcMeta * ((size_t)N * (3 + l) * 4 + (size_t)(N / 16) * 8) +
         (sizeof(double) + sizeof(uint32_t)) * (size_t)kk * kTcThreads + sizeof(float) * kTcThreads +
         8 + 8 * 32 + 16;
}

// Tile shapes (N nodes per tile, row stages, CTAs per SM), in order of preference; the first
// that fits shared memory is used.  SB_BF_TILE = "N,stages,ctas" forces one (testing).
struct TcShape { int N, nbs, ctas; };
static const TcShape kTcShapes[] = {{128, 3, 2}, {128, 2, 2}, {256, 1, 2}, {128, 1, 2}, {64, 2, 2},
                                    {128, 4, 1}, {256, 2, 1}, {128, 2, 1}};
// TMEM accumulators of a shape: 2 x N columns, or 4 when 4 N fits the CTA's share of the 512
// columns (SB_BF_NACC=2 forces two)
static int tc_nacc(const TcShape& t) {
  static const int force = [] { const char* e = getenv("SB_BF_NACC"); return e ? atoi(e) : 0; }();
  if (force == 2 || force == 4) return (force * t.N <= 512 / t.ctas) ? force : 2;
  return 4 * t.N <= 512 / t.ctas ? 4 : 2;
}

static bool tc_shape_fits(int rowb, int l, int kk, const TcShape& t) {
  const size_t limit = t.ctas == 2 ? 113 * 1024 : 227 * 1024;
  return bf_tc_smem_n(rowb, l, kk, t.N, t.nbs) <= limit;
}

// m = operand bytes per row here (2 x features for bf16, features for u8)
static TcShape tc_shape(int m, int l, int kk) {
  if (m % 32 != 0 || m > 512 || l > 8 || kk > kTcMaxKK) return {0, 0, 0};
  if (const char* e = getenv("SB_BF_TILE")) {
    TcShape t{0, 0, 0};
    if (sscanf(e, "%d,%d,%d", &t.N, &t.nbs, &t.ctas) == 3 && tc_shape_fits(m, l, kk, t)) return t;
  }
  for (const TcShape& t : kTcShapes)
    if (tc_shape_fits(m, l, kk, t)) return t;
  return {0, 0, 0};
}

int bf_tc_tile(int rowb, int l, int kk, int* nbs = nullptr) {
  const TcShape t = tc_shape(rowb, l, kk);
  if (nbs) *nbs = t.nbs;
  return t.N;
}

int bf_tc_supported(int rowb, int l, int kk) { return bf_tc_tile(rowb, l, kk) != 0; }

int bf_tc_ctas_per_sm(int rowb, int l, int kk) {
  const TcShape t = tc_shape(rowb, l, kk);
  return t.N ? t.ctas : 1;
}

// ---- attribute-grouped node order ---------------------------------------------------
__global__ void tc_attr_range_kernel(const int32_t* A, int64_t n, int l, int32_t* lo, int32_t* hi) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int u = 0; u < l; ++u) {
    atomicMin(lo + u, A[i * l + u]);
    atomicMax(hi + u, A[i * l + u]);
  }
}

// code = mixed-radix attribute tuple (or the node id when tuples are too many to group)
__global__ void tc_code_kernel(const int32_t* A, int64_t n, int l, const int32_t* lo,
                               const int64_t* stride, int grouped, int32_t* code,
                               unsigned long long* hist) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t c = 0;
  if (grouped) {
    for (int u = 0; u < l; ++u) c += (int64_t)(A[i * l + u] - lo[u]) * stride[u];
  } else {
    c = i;
  }
  code[i] = (int32_t)c;
  atomicAdd(hist + c, 1ull);
}

__global__ void tc_scatter_kernel(const int32_t* code, int64_t n, const int64_t* off,
                                  unsigned long long* cur, int32_t* orig) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t c = code[i];
  unsigned long long p = atomicAdd(cur + c, 1ull);
  orig[off[c] + (int64_t)p] = (int32_t)i;
}

// sorted copies: bf16 rows (row-group layout, K = mk columns), exact squared norms, codes,
// attributes (warp per node).  Folded rows (mk = m + 16) end in the bytes of |x|^2
// (|x|^2 < 2^24: h * 2^16 + m * 2^8 + l, each byte exact in bf16).
__global__ void tc_gather_kernel(const float* F, const int32_t* A, const int32_t* code_in,
                                 const int32_t* orig, int64_t n, int m, int mk, int l, char* Fb,
                                 int32_t* nx, int32_t* code, int32_t* As) {
  int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id();
  if (p >= n) return;
  const int64_t v = orig[p];
  int acc = 0;
  for (int t = lane_id(); t < m; t += 32) {
    float x = F[v * m + t];
    reinterpret_cast<__nv_bfloat16*>(Fb + rg_off(p, t >> 3, mk))[t & 7] = __float2bfloat16_rn(x);
    acc += (int)x * (int)x;
  }
  acc = warp_sum(acc);
  for (int t = m + lane_id(); t < mk; t += 32) {
    const int b = t - m;
    const float x = b == 0 ? (float)((acc >> 16) & 255) : b == 1 ? (float)((acc >> 8) & 255)
                  : b == 2 ? (float)(acc & 255) : 0.f;
    reinterpret_cast<__nv_bfloat16*>(Fb + rg_off(p, t >> 3, mk))[t & 7] = __float2bfloat16_rn(x);
  }
  if (lane_id() == 0) {
    nx[p] = __float_as_int((float)acc);  // |x|^2 as fp32 (exact: below 2^24)
    code[p] = code_in[v];
  }
  for (int u = lane_id(); u < l; u += 32) As[p * l + u] = A[v * l + u];
}

// sorted u8 copies (row-group layout), exact squared norms as int32, codes, attributes
__global__ void tc_gather_u8_kernel(const float* F, const int32_t* A, const int32_t* code_in,
                                    const int32_t* orig, int64_t n, int m, int l, uint8_t* Fb,
                                    int32_t* nx, int32_t* code, int32_t* As) {
  int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id();
  if (p >= n) return;
  const int64_t v = orig[p];
  int acc = 0;
  for (int t = lane_id(); t < m; t += 32) {
    const int x = (int)F[v * m + t];
    Fb[rg_off8(p, t, m)] = (uint8_t)x;
    acc += x * x;
  }
  acc = warp_sum(acc);
  if (lane_id() == 0) {
    nx[p] = acc;
    code[p] = code_in[v];
  }
  for (int u = lane_id(); u < l; u += 32) As[p * l + u] = A[v * l + u];
}

// ---- |x|^2 order inside each attribute tuple, and the per-chunk records -----------------
// key = (tuple code << 32) | |x|^2 of the node (integer data: exact); the node order keeps the
// tuples contiguous and ascending, and within a tuple runs by |x|^2, so a 16-node chunk spans a
// narrow |x|^2 range (the u8 epilogue's raw chunk test)
__global__ void tc_norm_key_kernel(const float* F, int64_t n, int m, const int32_t* code_in,
                                   const int32_t* orig, uint64_t* key, int32_t* val) {
  const int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id();
  if (p >= n) return;
  const int64_t v = orig[p];
  long long acc = 0;
  for (int t = lane_id(); t < m; t += 32) {
    const long long x = (long long)F[v * m + t];
    acc += x * x;
  }
  acc = warp_sum(acc);
  if (lane_id() == 0) {
    key[p] = ((uint64_t)(uint32_t)code_in[v] << 32) | (uint64_t)(acc > 0xFFFFFFFFll ? 0xFFFFFFFFll : acc);
    val[p] = (int32_t)v;
  }
}

__global__ void tc_chunk_meta_kernel(const int32_t* nx, const int32_t* code, int64_t n, int64_t nchunks,
                                     int2* cm) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  int mn = INT_MAX, cd = -1;
  bool mixed = false;
  for (int j = 0; j < 16; ++j) {
    const int64_t p = c * 16 + j;
    if (p >= n) { mixed = true; break; }
    mn = min(mn, nx[p]);
    if (j == 0) cd = code[p]; else mixed = mixed || code[p] != cd;
  }
  cm[c] = make_int2(mn == INT_MAX ? 0 : mn, mixed ? -1 : cd);
}

size_t tc_norm_order_scratch(int64_t n) {
  size_t temp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)n);
  return (size_t)n * (2 * sizeof(uint64_t) + sizeof(int32_t)) + temp + 1024;
}

int launch_tc_norm_order(const float* F, int64_t n, int m, const int32_t* code_in, int32_t* orig,
                         void* scratch, cudaStream_t st) {
  char* p = static_cast<char*>(scratch);
  auto take = [&](size_t b) { char* r = p; p += (b + 255) & ~(size_t)255; return r; };
  uint64_t* k_in = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * n));
  uint64_t* k_out = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * n));
  int32_t* v_in = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * n));
  size_t temp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp, k_in, k_out, v_in, orig, (int)n);
  void* d_temp = take(temp);
  tc_norm_key_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(F, n, m, code_in, orig, k_in, v_in);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(d_temp, temp, k_in, k_out, v_in, orig, (int)n, 0, 64, st);
  return e != cudaSuccess ? (int)e : (int)cudaGetLastError();
}

int launch_tc_chunk_meta(const int32_t* nx, const int32_t* code, int64_t n, int64_t npad, void* cm,
                         cudaStream_t st) {
  const int64_t nch = npad / 16;
  tc_chunk_meta_kernel<<<(unsigned)((nch + 255) / 256), 256, 0, st>>>(nx, code, n, nch, reinterpret_cast<int2*>(cm));
  return (int)cudaGetLastError();
}

int launch_tc_gather_u8(const float* F, const int32_t* A, const int32_t* code_in,
                        const int32_t* orig, int64_t n, int m, int l, void* Fb, int32_t* nx,
                        int32_t* code, int32_t* As, cudaStream_t st) {
  tc_gather_u8_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(F, A, code_in, orig, n, m, l,
                                                                (uint8_t*)Fb, nx, code, As);
  return (int)cudaGetLastError();
}

int launch_bf_tc_prep_queries_u8(const double* qf, int64_t q, int m, void* Qb, int32_t* nq,
                                 cudaStream_t st) {
  const int64_t qpad = (q + kTcM - 1) / kTcM * kTcM;
  tc_prep_queries_u8_kernel<<<(unsigned)((qpad + 7) / 8), 256, 0, st>>>(qf, q, qpad, m,
                                                                        (uint8_t*)Qb, nq);
  return (int)cudaGetLastError();
}

int launch_tc_attr_range(const int32_t* A, int64_t n, int l, int32_t* lo, int32_t* hi,
                         cudaStream_t st) {
  tc_attr_range_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(A, n, l, lo, hi);
  return (int)cudaGetLastError();
}
int launch_tc_code(const int32_t* A, int64_t n, int l, const int32_t* lo, const int64_t* stride,
                   int grouped, int32_t* code, unsigned long long* hist, cudaStream_t st) {
  tc_code_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(A, n, l, lo, stride, grouped, code, hist);
  return (int)cudaGetLastError();
}
int launch_tc_scatter(const int32_t* code, int64_t n, const int64_t* off, unsigned long long* cur,
                      int32_t* orig, cudaStream_t st) {
  tc_scatter_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(code, n, off, cur, orig);
  return (int)cudaGetLastError();
}
int launch_tc_gather(const float* F, const int32_t* A, const int32_t* code_in, const int32_t* orig,
                     int64_t n, int m, int mk, int l, void* Fb, int32_t* nx, int32_t* code,
                     int32_t* As, cudaStream_t st) {
  tc_gather_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(F, A, code_in, orig, n, m, mk, l,
                                                             (char*)Fb, nx, code, As);
  return (int)cudaGetLastError();
}

int launch_bf_tc_prep_queries(const double* qf, int64_t q, int m, int mk, void* Qb, int32_t* nq,
                              cudaStream_t st) {
  const int64_t qpad = (q + kTcM - 1) / kTcM * kTcM;
  tc_prep_queries_kernel<<<(unsigned)((qpad + 7) / 8), 256, 0, st>>>(qf, q, qpad, m, mk, (char*)Qb, nq);
  return (int)cudaGetLastError();
}

int launch_bf_tc(const void* Fb, const int32_t* nx, const int32_t* A, const int32_t* code,
                 const int32_t* orig, const void* Qb, const int32_t* nq, const int64_t* qa,
                 const int64_t* qmask, int64_t n, int64_t q, int m, int l, int kk, int splits,
                 double alpha, double* part_d, uint32_t* part_i, int* gthr, int fold,
                 int u8, const void* cmeta, cudaStream_t st) {
  TcArgs a;
  a.gthr = gthr;
  a.cmeta = reinterpret_cast<const int2*>(cmeta);
  a.Fb = (const char*)Fb; a.nx = nx; a.A = A; a.code = code; a.orig = orig;
  a.Qb = (const char*)Qb;
  a.nq = nq; a.qa = qa; a.qmask = qmask; a.n = n; a.q = q; a.m = m; a.l = l; a.kk = kk;
  a.splits = splits; a.alpha = alpha; a.part_d = part_d; a.part_i = part_i;
  const int kind = u8 ? 2 : (fold ? 1 : 0);
  const TcShape sh = tc_shape(m * (u8 ? 1 : 2), l, kk);
  a.N = sh.N;
  if (a.N == 0) return (int)cudaErrorInvalidValue;
  a.nacc = tc_nacc(sh);
  size_t smem = bf_tc_smem_n(m * (u8 ? 1 : 2), l, kk, a.N, sh.nbs);
  void (*kern)(TcArgs);
#define SB_TC_PICK(NB, CT) \
  (kind == 2 ? bf_tc_kernel<2, NB, CT> : kind == 1 ? bf_tc_kernel<1, NB, CT> : bf_tc_kernel<0, NB, CT>)
  if (sh.nbs == 1) kern = SB_TC_PICK(1, 2);
  else if (sh.nbs == 3) kern = SB_TC_PICK(3, 2);
  else if (sh.nbs == 4) kern = SB_TC_PICK(4, 1);
  else if (sh.ctas == 2) kern = SB_TC_PICK(2, 2);
  else kern = SB_TC_PICK(2, 1);
#undef SB_TC_PICK
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  dim3 grid((unsigned)((q + kTcM - 1) / kTcM), (unsigned)splits);
  kern<<<grid, kTcThreads + 32, smem, st>>>(a);
  return (int)cudaGetLastError();
}

}  // namespace sb

// bf_tf.cu — exhaustive AUTO top-k (oracle_auto_topk, evaluate.py:32-55) for real-valued data
// on the tcgen05 tensor cores: a TF32 filter with a certified error bound, then an exact fp64
// re-rank of the few survivors in NumPy's summation order.
//
// The reference value of a (query, node) pair is U = sqrt(S) * f with S = sum_t (x_t - q_t)^2
// (fp64, NumPy pairwise order, evaluate.py:48) and f = 1 + s_a / alpha (evaluate.py:53).
// The tensor cores compute dot~ = sum_t tf32(x_t) tf32(q_t) in an fp32 TMEM accumulator, and
//   S~ = |x|^2 + |q|^2 - 2 dot~,   |S~ - S| <= cE (|x|^2 + |q|^2)             (1)
// with cE from the rounding analysis in tf_margin() (tf32 operand rounding 2^-11 per element,
// fp32 accumulation over d/8 MMA steps, fp32 evaluation of S~).  Every pair therefore has a
// certified lower key  lo = max(S~ - margin, 0) f^2 <= U^2  and upper key  hi = (S~ + margin) f^2
// >= U^2.  Each epilogue thread keeps the k smallest upper keys it has seen; its k-th, T2, bounds
// the exact k-th U^2 of the query from above (k distinct nodes lie below it), and so does the
// minimum over all threads (published per query through a global atomicMin).  A node can be in
// the exact top k only if lo <= U_k^2 <= T2, so the kernel emits every node with lo <= (current
// T2) into the query's candidate buffer — all true members are emitted, whatever the order.  The
// refine kernel keeps the candidates with lo <= the final T2, recomputes them exactly (fp64,
// NumPy order, ties by id) and sorts: the result is the reference's top k bit for bit.  A
// query whose candidates overflow the buffer is flagged; the host recomputes it on the exact
// fp64 kernel (bf_topk.cu).
//
// Kernel shape: CTA = 128 queries (one per TMEM lane) x a node range walked in tiles of N = 256
// (or 128) nodes; K is streamed in chunks of 32 elements (128 B per row).  Warp 8 loads (bulk
// copies into a ring of S stages, plus per-tile node metadata), warp 9 issues tcgen05.mma
// .kind::tf32 (M = 128, N, K = 8) into one of two TMEM accumulators, warps 0..7 are the
// epilogue (two threads per query, one per column half).  When 128 query rows of all K fit in
// shared memory (d <= 128) the query tile stays resident and only node chunks stream.
#include <cuda_runtime.h>
#include <float.h>
#include <math.h>

#include <cmath>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "sb_internal.h"
#include "tc_ptx.cuh"

namespace sb {

constexpr int kTfM = 128;                 // queries per CTA (UMMA M, TMEM lanes)
constexpr int kTfKC = 32;                 // K elements per streamed chunk
constexpr int kTfChunkBytes = kTfM * kTfKC * 4;  // one full 128-row chunk block

// Operand layout (nodes and queries alike): blocks of 128 rows; inside a block, K chunks of 32
// elements (the last one dpad - 32c wide, dpad = d rounded up to 8) are contiguous 128 x cw x 4
// byte blocks in K-major core-matrix order: 8-row group g at g * 8 cw * 4, core matrix j (4
// elements) at j * 128, row r at r * 16.  UMMA: LBO = 128 B, SBO = 32 cw B, and a K = 8 step
// advances the start address by 256 B.
SB_HD size_t tf_off(int64_t row, int t, int dpad) {
  const int c = t >> 5;
  const int cw = dpad - 32 * c < 32 ? dpad - 32 * c : 32;
  return (size_t)(row >> 7) * (size_t)(kTfM * dpad * 4) + (size_t)c * kTfChunkBytes +
         (size_t)((row & 127) >> 3) * (size_t)(8 * cw * 4) + (size_t)((t & 31) >> 2) * 128 +
         (size_t)(row & 7) * 16 + (size_t)(t & 3) * 4;
}

// K of the operands: the d features, then two columns that fold -(1 - cE)|x|^2 / 2 into the
// product (hi and lo tf32 parts on the node side, 1.0 on the query side), rounded up to 8
SB_HD int tf_dpad(int m) { return (m + 2 + 7) / 8 * 8; }

SB_DEV float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// ---- prep ---------------------------------------------------------------------------------
// node operands in the sorted (attribute-grouped) order: tf32 rows whose columns m, m + 1 hold
// hi + lo = -(1 - cE)|x|^2 / 2 (so the accumulator holds z = x.q - (1 - cE)|x|^2 / 2 and
// y = 2 z = 2 x.q - nxs), and per node nxd = 2 cE |x|^2 (rounded up: hi - lo keys), code, attrs.
__global__ void tf_gather_kernel(const float* __restrict__ F, const int32_t* __restrict__ A,
                                 const int32_t* __restrict__ code_in, const int32_t* __restrict__ orig,
                                 int64_t n, int m, int dpad, int l, double cE, float* Ft,
                                 float* nxd, int32_t* code, int32_t* As) {
  const int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id();
  if (p >= n) return;
  const int64_t v = orig[p];
  double acc = 0.0;
  char* base = reinterpret_cast<char*>(Ft);
  for (int t = lane_id(); t < m; t += 32) {
    const float x = F[v * m + t];
    *reinterpret_cast<float*>(base + tf_off(p, t, dpad)) = to_tf32(x);
    acc += (double)x * (double)x;
  }
  acc = warp_sum(acc);
  const double h = -0.5 * (1.0 - cE) * acc;
  const float hi = to_tf32((float)h);
  const float lo = to_tf32((float)(h - (double)hi));
  for (int t = m + lane_id(); t < dpad; t += 32)
    *reinterpret_cast<float*>(base + tf_off(p, t, dpad)) = t == m ? hi : t == m + 1 ? lo : 0.f;
  if (lane_id() == 0) {
    nxd[p] = __double2float_ru(2.0 * cE * acc);
    code[p] = code_in[v];
  }
  for (int u = lane_id(); u < l; u += 32) As[p * l + u] = A[v * l + u];
}

// end (exclusive) of each node's run of equal attribute codes in the sorted order (the codes
// are ascending): lets the epilogue split a 32-column chunk into runs that share one factor
__global__ void tf_runend_kernel(const int32_t* __restrict__ code, int64_t n, int32_t* runend) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int32_t c = code[p];
  int64_t lo = p + 1, hi = n;  // first index > p whose code differs
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (code[mid] == c) lo = mid + 1; else hi = mid;
  }
  runend[p] = (int32_t)lo;
}

// queries: tf32 rows (zero past q), nqs = (1 - cE)|q|^2 - tiny, nqu = (1 + cE)|q|^2 + tiny
__global__ void tf_prep_queries_kernel(const double* __restrict__ qf, int64_t q, int64_t qpad, int m,
                                       int dpad, double cE, double tiny, float* Qt, float* nqs,
                                       float* nqu) {
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id();
  if (i >= qpad) return;
  double acc = 0.0;
  char* base = reinterpret_cast<char*>(Qt);
  for (int t = lane_id(); t < dpad; t += 32) {
    const double v = (i < q && t < m) ? qf[i * m + t] : 0.0;
    const float w = t < m ? to_tf32((float)v) : (i < q && t < m + 2) ? 1.0f : 0.0f;
    *reinterpret_cast<float*>(base + tf_off(i, t, dpad)) = w;
    acc += v * v;
  }
  acc = warp_sum(acc);
  if (lane_id() == 0 && i < q) {
    nqs[i] = __double2float_rd((1.0 - cE) * acc - tiny);
    nqu[i] = __double2float_ru((1.0 + cE) * acc + tiny);
  }
}

// ---- main kernel ------------------------------------------------------------------------
struct TfArgs {
  const char* Ft;          // node operands (tf_off layout), npad rows
  const float* nxd;        // npad: 2 cE |x|^2 (upper minus lower key offsets)
  const int32_t* code;     // npad
  const int32_t* orig;     // npad
  const int32_t* runend;   // npad: end of the node's run of equal codes
  const int32_t* A;        // npad x l
  const char* Qt;          // query operands, rows padded to a whole CTA query block
  const float* nqs;        // q
  const float* nqu;        // q
  const int64_t* qa;       // q x l
  const int64_t* qmask;    // q x l or null
  int64_t n, q;
  int dpad, l, kk, splits, stages;
  double alpha;
  int* gthr;               // q: best upper bound of U_k^2 over all threads (fp32 bits)
  uint32_t* cnt;           // one per epilogue thread of the grid: candidates it emitted
  uint64_t* cand;          // (CTA, thread) segments of cap: (lower key bits << 32) | original id;
                           // a CTA's segments are contiguous (its stores stay within a few pages)
  int cap;
  uint32_t* ocnt;          // q: entries in the query's shared overflow area (full segments)
  uint64_t* ocand;         // q x ocap
  int ocap;
  int seed;                // > 0: bound-only pass over `seed` evenly spread tiles per split
  // large k (two-pass scheme, see bf_tf_run): bound_only = a full pass that only builds the
  // per-thread lists and writes them to `lists` (q x threads x KR); fixed = the emission pass
  // under the bound the select kernel wrote to gthr (no list work, the bound never moves)
  int bound_only, fixed;
  float* lists;
  int strided;             // 1: split s walks tiles s, s + splits, ...; 0: contiguous ranges
};

constexpr int kTfMetaStages = 4;

SB_HD size_t tf_meta_bytes(int N, int l) { return (size_t)N * (4 + l) * 4; }

// shared layout: [A resident | A stages] | B stages | meta ring | smem lists (KR = 0) | bounds |
// query attributes | barriers
SB_HD size_t tf_smem_bytes(int dpad, int l, int kk, int N, int stages, bool ares, int qt, int ew, int kr) {
  const int epi = 32 * ew;
  const size_t a = ares ? (size_t)qt * kTfM * dpad * 4 : (size_t)stages * qt * kTfChunkBytes;
  return a + (size_t)stages * N * kTfKC * 4 + kTfMetaStages * tf_meta_bytes(N, l) +
         (kr == 0 ? sizeof(float) * (size_t)kk * epi : 0) + sizeof(float) * epi +
         2 * sizeof(int32_t) * (size_t)l * qt * kTfM + 8 * 32 + 16;
}

// N = nodes per tile, ARES = query tiles resident in shared memory, QT = query tiles (of 128)
// per CTA, EW = epilogue warps (8 or 16), KR = register list length (16, 32; 0 = list in shared
// memory).  TMEM: 2 buffers x QT x N fp32 columns.  Epilogue warp w reads TMEM lane group w % 4;
// the EW / 4 warps of a lane group split the QT query tiles and their columns: PPQ = EW / 4 / QT
// threads per query, N / PPQ columns each.
template <int N, bool ARES, int QT, int EW, int KR>
__global__ void __launch_bounds__(32 * EW + 64, 1) bf_tf_kernel(TfArgs a) {
  constexpr int EPI = 32 * EW;              // epilogue threads
  constexpr int PPQ = EW / 4 / QT;          // epilogue threads per query
  constexpr int cols = N / PPQ;             // columns per epilogue thread and tile
  // TMEM columns per load in the scan: 16 for the 32-key register lists (with 32 more live
  // registers the 32-column buffer spilled in the hot loop: 18 warps leave 96 registers)
  constexpr int CW = KR > 16 ? 16 : 32;
  static_assert(cols % 32 == 0, "32-column TMEM loads");
  // (pointer arithmetic on the shared array itself keeps every access an LDS/STS)
  extern __shared__ __align__(1024) char smem[];
  const int tid = threadIdx.x;
  const int dpad = a.dpad, l = a.l, S = a.stages;
  const int nch = (dpad + kTfKC - 1) / kTfKC;
  const size_t meta_bytes = tf_meta_bytes(N, l);
  const size_t qblk_bytes = (size_t)kTfM * dpad * 4;  // one 128-row query block
  char* p = smem;
  char* sA = p; p += ARES ? QT * qblk_bytes : (size_t)S * QT * kTfChunkBytes;
  char* sB = p; p += (size_t)S * N * kTfKC * 4;
  char* sM = p; p += kTfMetaStages * meta_bytes;
  float* ul = reinterpret_cast<float*>(p); p += KR == 0 ? sizeof(float) * (size_t)a.kk * EPI : 0;
  volatile float* s_t2 = reinterpret_cast<float*>(p); p += sizeof(float) * EPI;
  int32_t* s_qa = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * (size_t)l * QT * kTfM;
  int32_t* s_qm = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * (size_t)l * QT * kTfM;
  p += (8 - ((p - smem) & 7)) & 7;
  uint64_t* bars = reinterpret_cast<uint64_t*>(p);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 31);
  // barriers: full[0..7] sfree[8..15] fullM[16..19] emptyM[20..23] accf[24,25] empty[26,27]
  // aready[28]
  const uint32_t b0 = smem_u32(bars);
  auto bar_full = [&](int s) { return b0 + 8u * (uint32_t)s; };
  auto bar_sfree = [&](int s) { return b0 + 8u * (uint32_t)(8 + s); };
  auto bar_fullM = [&](int s) { return b0 + 8u * (uint32_t)(16 + s); };
  auto bar_emptyM = [&](int s) { return b0 + 8u * (uint32_t)(20 + s); };
  auto bar_accf = [&](int s) { return b0 + 8u * (uint32_t)(24 + s); };
  auto bar_empty = [&](int s) { return b0 + 8u * (uint32_t)(26 + s); };
  const uint32_t bar_aready = b0 + 8u * 28;
  auto wait = [&](uint32_t bar, uint32_t parity) { mbar_wait(bar, parity); };

  // tiles of this CTA: i -> tile0 + i * tstride
  const int64_t tiles = (a.n + N - 1) / N;
  int ntl;
  int64_t tile0, tstride;
  if (a.seed) {  // bound-only pass: a.seed tiles per split, spread evenly over the sorted order
    const int64_t total = (int64_t)a.seed * a.splits < tiles ? (int64_t)a.seed * a.splits : tiles;
    ntl = blockIdx.y < total ? (int)((total - blockIdx.y + a.splits - 1) / a.splits) : 0;
    tile0 = (int64_t)blockIdx.y * (tiles / total);
    tstride = tiles / total * a.splits;
  } else if (a.strided) {
    // split s walks tiles s, s + splits, ...: every split sees the same mix of attribute codes,
    // so the survivors of queries with popular codes do not pile up in a few CTAs
    ntl = tiles > blockIdx.y ? (int)((tiles - blockIdx.y + a.splits - 1) / a.splits) : 0;
    tile0 = blockIdx.y;
    tstride = a.splits;
  } else {  // contiguous ranges
    const int64_t per = (tiles + a.splits - 1) / a.splits;
    tile0 = per * blockIdx.y;
    tstride = 1;
    ntl = tile0 < tiles ? (int)(tile0 + per < tiles ? per : tiles - tile0) : 0;
  }

  if (warp_id() == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(2 * QT * N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == EPI) {
    for (int s = 0; s < S; ++s) {
      mbar_init(bar_full(s), 1);
      mbar_init(bar_sfree(s), 1);
    }
    for (int s = 0; s < kTfMetaStages; ++s) {
      mbar_init(bar_fullM(s), 1);
      mbar_init(bar_emptyM(s), EPI);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar_accf(s), 1);
      mbar_init(bar_empty(s), EPI);
    }
    mbar_init(bar_aready, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < EPI) {
    if (KR == 0)
      for (int i = 0; i < a.kk; ++i) ul[i * EPI + tid] = FLT_MAX;
    s_t2[tid] = FLT_MAX;
  }
  // query attributes and masks of the CTA's queries
  for (int i = tid; i < QT * kTfM * l; i += blockDim.x) {
    const int64_t g = (int64_t)blockIdx.x * QT * kTfM + i / l;
    const bool ok = g < a.q;
    s_qa[i] = ok ? (int32_t)a.qa[g * l + i % l] : 0;
    s_qm[i] = ok ? (int32_t)(a.qmask ? a.qmask[g * l + i % l] : 1) : 0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const char* qblk = a.Qt + (size_t)blockIdx.x * QT * qblk_bytes;

  if (warp_id() == EW) {
    // ---------------- loaders: lane 0 operands, lane 1 node metadata (its own ring) --------
    if (lane_id() == 0 && ntl > 0) {
      if (ARES) {
        const uint32_t ab = (uint32_t)(QT * qblk_bytes);
        mbar_expect_tx(bar_aready, ab);
        bulk_g2s(smem_u32(sA), qblk, ab, bar_aready);
      }
      int it = 0;
      for (int i = 0; i < ntl; ++i) {
        const int64_t v0 = ((int64_t)i * tstride + tile0) * (int64_t)N;
        for (int c = 0; c < nch; ++c, ++it) {
          const int st = it % S;
          const int use = it / S;
          if (use >= 1) wait(bar_sfree(st), (uint32_t)((use - 1) & 1));
          const int cw = dpad - 32 * c < 32 ? dpad - 32 * c : 32;
          const uint32_t blk = (uint32_t)(kTfM * cw * 4);  // one 128-row chunk block
          const uint32_t fb = bar_full(st);
          mbar_expect_tx(fb, (ARES ? 0u : (uint32_t)QT * blk) + (uint32_t)(N / kTfM) * blk);
          if (!ARES) {
#pragma unroll
            for (int t = 0; t < QT; ++t)
              bulk_g2s(smem_u32(sA + ((size_t)st * QT + t) * kTfChunkBytes),
                       qblk + t * qblk_bytes + (size_t)c * kTfChunkBytes, blk, fb);
          }
          char* sb = sB + (size_t)st * N * kTfKC * 4;
#pragma unroll
          for (int h = 0; h < N / kTfM; ++h) {
            const char* src = a.Ft + (size_t)(v0 / kTfM + h) * qblk_bytes + (size_t)c * kTfChunkBytes;
            bulk_g2s(smem_u32(sb + (size_t)h * blk), src, blk, fb);
          }
        }
      }
    } else if (lane_id() == 1) {
      for (int i = 0; i < ntl; ++i) {
        const int ms = i % kTfMetaStages;
        const int use = i / kTfMetaStages;
        if (use >= 1) wait(bar_emptyM(ms), (uint32_t)((use - 1) & 1));
        const int64_t v0 = ((int64_t)i * tstride + tile0) * (int64_t)N;
        char* meta = sM + ms * meta_bytes;
        const uint32_t fm = bar_fullM(ms);
        mbar_expect_tx(fm, (uint32_t)meta_bytes);
        bulk_g2s(smem_u32(meta), a.nxd + v0, (uint32_t)(N * 4), fm);
        bulk_g2s(smem_u32(meta + N * 4), a.code + v0, (uint32_t)(N * 4), fm);
        bulk_g2s(smem_u32(meta + N * 8), a.orig + v0, (uint32_t)(N * 4), fm);
        bulk_g2s(smem_u32(meta + N * 12), a.runend + v0, (uint32_t)(N * 4), fm);
        bulk_g2s(smem_u32(meta + N * 16), a.A + v0 * l, (uint32_t)(N * l * 4), fm);
      }
    }
    __syncwarp();
  } else if (warp_id() == EW + 1) {
    // ---------------- MMA issuer ----------------
    if (lane_id() == 0 && ntl > 0) {
      // TF32 x TF32 -> F32: c_format = 1 [4,6), a/b format = 2 [7,10) [10,13), N >> 3 [17,23),
      // M >> 4 [24,29), both K-major
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
                             ((uint32_t)(kTfM >> 4) << 24);
      if (ARES) wait(bar_aready, 0);
      int it = 0;
      for (int i = 0; i < ntl; ++i) {
        const int acc = i & 1;
        if (i >= 2) wait(bar_empty(acc), (uint32_t)(((i >> 1) - 1) & 1));
        tc_fence_after();
        for (int c = 0; c < nch; ++c, ++it) {
          const int st = it % S;
          wait(bar_full(st), (uint32_t)((it / S) & 1));
          tc_fence_after();
          const int cw = dpad - 32 * c < 32 ? dpad - 32 * c : 32;
          const uint32_t sbo = (uint32_t)(32 * cw);
          const uint32_t bb = smem_u32(sB + (size_t)st * N * kTfKC * 4);
          // descriptors are linear in the start address (bits [0,14) hold addr >> 4, no carry
          // below 256 KB): a K = 8 step adds 256 B = 16 units
          const uint64_t bd0 = umma_desc(bb, 128, sbo);
#pragma unroll
          for (int t = 0; t < QT; ++t) {
            const uint32_t ab = ARES ? smem_u32(sA + t * qblk_bytes + (size_t)c * kTfChunkBytes)
                                     : smem_u32(sA + ((size_t)st * QT + t) * kTfChunkBytes);
            const uint32_t dt = tmem + (uint32_t)((acc * QT + t) * N);
            const uint64_t ad0 = umma_desc(ab, 128, sbo);
            if (cw == 32) {
#pragma unroll
              for (int s = 0; s < 4; ++s)
                asm volatile(
                    "{\n\t.reg .pred p;\n\t"
                    "setp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dt),
                    "l"(ad0 + 16u * s), "l"(bd0 + 16u * s), "r"(idesc), "r"((c | s) != 0 ? 1u : 0u));
            } else {
              for (int s = 0; s < cw / 8; ++s)
                asm volatile(
                    "{\n\t.reg .pred p;\n\t"
                    "setp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dt),
                    "l"(ad0 + 16u * s), "l"(bd0 + 16u * s), "r"(idesc), "r"((c | s) != 0 ? 1u : 0u));
            }
          }
          mma_commit(bar_sfree(st));  // the stage is free once these MMAs complete
        }
        mma_commit(bar_accf(acc));
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue ----------------
    const int lg = warp_id() & 3;                 // TMEM lane group
    const int u = warp_id() >> 2;
    const int qt = u / PPQ;                       // query tile
    const int part = u % PPQ;                     // column part
    const int row = lg * 32 + lane_id();
    const int qrow = qt * kTfM + row;             // query within the CTA's block
    const int64_t my_q = (int64_t)blockIdx.x * QT * kTfM + qrow;
    const bool qok = my_q < a.q;
    const float nq_s = qok ? a.nqs[my_q] : 0.f;
    const float nq_u = qok ? a.nqu[my_q] : 0.f;
    const float ia = __double2float_ru(1.0 / a.alpha);
    const int kk = a.kk;
    // min(own list tail, partners', global); starts from the seed pass's bound
    float t2_eff = qok ? fminf(FLT_MAX, __int_as_float(a.gthr[my_q])) : FLT_MAX;
    float own_t2 = FLT_MAX;     // this thread's kk-th smallest upper key
    float rl[KR > 0 ? KR : 1];  // KR > 0: the list in registers, -FLT_MAX in its first KR - kk
#pragma unroll
    for (int j = 0; j < (KR > 0 ? KR : 1); ++j) rl[j] = j < (KR > 0 ? KR : 1) - kk ? -FLT_MAX : FLT_MAX;
    int last_code = -2;
    float f2 = 1.f, inv_f2 = 1.f, thr_h = -FLT_MAX;
    // y = 2 z >= thr  <=>  lo = nqs - y <= T2 / f^2 (conservatively rounded); thr_h = thr / 2
    auto set_thr = [&]() {
      const float t = t2_eff * inv_f2 * 1.00002f;
      thr_h = t >= FLT_MAX ? -FLT_MAX : 0.5f * (nq_s - t);
    };
    const int32_t* s_at = nullptr;  // the current tile's node attributes
    // f^2 of a node's attribute tuple for this query (f = 1 + s_a / alpha, fp32, rounded up)
    auto attr_f2 = [&](int col) {
      int sa = 0;
      for (int w = 0; w < l; ++w) sa += abs(s_at[col * l + w] - s_qa[qrow * l + w]) * s_qm[qrow * l + w];
      const float f = fmaf((float)sa, ia, 1.0f);
      return f * f;
    };
    const uint32_t lane_base = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(qt * N + part * cols);
    // this thread's private candidate segment (no atomics on the emission path)
    const size_t seg = ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * EPI + tid;
    uint64_t* my_cand = qok ? a.cand + seg * a.cap : nullptr;
    uint32_t emitted = 0;

    float gnext = FLT_MAX;
    for (int i = 0; i < ntl; ++i) {
      const int s = i & 1;
      const int ms = i % kTfMetaStages;
      const char* meta = sM + ms * meta_bytes;
      const float* s_nxd = reinterpret_cast<const float*>(meta);
      const int32_t* s_code = reinterpret_cast<const int32_t*>(meta + N * 4);
      const int32_t* s_orig = reinterpret_cast<const int32_t*>(meta + N * 8);
      const int32_t* s_run = reinterpret_cast<const int32_t*>(meta + N * 12);
      s_at = reinterpret_cast<const int32_t*>(meta + N * 16);
      const int64_t vb = ((int64_t)i * tstride + tile0) * (int64_t)N;
      const int nvalid = (int)(a.n - vb < N ? a.n - vb : N);
      // the query's tightest bound published by any CTA: the value loaded one tile ago (its
      // latency hides behind a whole tile), and the load for the next tile issued now
      const float gpre = gnext;
      gnext = qok ? __int_as_float(*reinterpret_cast<volatile int*>(a.gthr + my_q)) : FLT_MAX;
      wait(bar_fullM(ms), (uint32_t)((i / kTfMetaStages) & 1));
      wait(bar_accf(s), (uint32_t)((i >> 1) & 1));
      tc_fence_after();
      // one filter survivor: emission (lower key), this thread's upper-key list
      auto process = [&](int col, float zj, float fsq) {
        const float yj = 2.0f * zj;
        const float lo = fmaxf(nq_s - yj, 0.f) * fsq * 0.99998f;
        if (lo > t2_eff) return;
        if (!a.seed && !a.bound_only) {  // a possible member of the exact top k
          const uint64_t e = ((uint64_t)__float_as_uint(lo) << 32) | (uint32_t)s_orig[col];
          if (emitted < (uint32_t)a.cap) {
            my_cand[emitted++] = e;
          } else {  // segment full: the query's shared overflow area
            const uint32_t slot = atomicAdd(a.ocnt + my_q, 1u);
            if (slot < (uint32_t)a.ocap) a.ocand[(size_t)my_q * a.ocap + slot] = e;
          }
        }
        // upper key (nqu + nxu - 2 dot = nq_u - y + nxd) into this thread's kk smallest
        const float hi = fmaxf(nq_u - yj + s_nxd[col], 0.f) * fsq * 1.00002f;
        if (a.fixed || !(hi < own_t2)) return;
        if (KR > 0) {  // sorted register list: one branch-free pass, no memory chain
#pragma unroll
          for (int j = KR - 1; j > 0; --j) rl[j] = hi < rl[j - 1] ? rl[j - 1] : fminf(hi, rl[j]);
          rl[0] = fminf(rl[0], hi);
          own_t2 = rl[KR - 1];
        } else {
          int pos = kk - 1;
          while (pos > 0) {
            const float pv = ul[(pos - 1) * EPI + tid];
            if (!(hi < pv)) break;
            ul[pos * EPI + tid] = pv;
            --pos;
          }
          ul[pos * EPI + tid] = hi;
          own_t2 = ul[(kk - 1) * EPI + tid];
        }
        if (own_t2 < t2_eff) {
          t2_eff = own_t2;
          set_thr();
          // (bound-only pass: a thread's KR-th key bounds only the KR-th of the query, not the
          // k-th the two-pass scheme needs, so it filters this thread's own list and nothing else)
          if (!a.bound_only) atomicMin(a.gthr + my_q, __float_as_int(own_t2));  // non-negative floats order as ints
        }
      };
      // scan: the fast filter over the accumulator.  All lanes of a warp see the same columns
      // (nodes) for different queries, so the chunk / run structure is warp-uniform; survivors
      // are processed in rounds, one per lane per round, so lanes with work run in parallel.
#pragma unroll 1
      for (int c = 0; c < cols / CW; ++c) {
        uint32_t r[CW];
        if constexpr (CW == 32) tmem_ld32(lane_base + (uint32_t)(s * QT * N + c * CW), r);
        else tmem_ld16(lane_base + (uint32_t)(s * QT * N + c * CW), r);
        const int c0 = part * cols + c * CW;
        // the accumulator holds z = y / 2 with y = 2 x.q - nxs: one max decides the chunk
        // tree of 3-input maxima: depth 4 instead of a 16-long chain
        float mx;
        if constexpr (CW == 32) {
          float t9[11];
#pragma unroll
          for (int j = 0; j < 10; ++j)
            t9[j] = fmaxf(fmaxf(__uint_as_float(r[3 * j]), __uint_as_float(r[3 * j + 1])), __uint_as_float(r[3 * j + 2]));
          t9[10] = fmaxf(__uint_as_float(r[30]), __uint_as_float(r[31]));
          const float u0 = fmaxf(fmaxf(t9[0], t9[1]), t9[2]), u1 = fmaxf(fmaxf(t9[3], t9[4]), t9[5]);
          const float u2 = fmaxf(fmaxf(t9[6], t9[7]), t9[8]), u3 = fmaxf(t9[9], t9[10]);
          mx = fmaxf(fmaxf(u0, u1), fmaxf(u2, u3));
        } else {
          float t5[6];
#pragma unroll
          for (int j = 0; j < 5; ++j)
            t5[j] = fmaxf(fmaxf(__uint_as_float(r[3 * j]), __uint_as_float(r[3 * j + 1])), __uint_as_float(r[3 * j + 2]));
          t5[5] = __uint_as_float(r[15]);
          mx = fmaxf(fmaxf(fmaxf(t5[0], t5[1]), t5[2]), fmaxf(fmaxf(t5[3], t5[4]), t5[5]));
        }
        const bool uniform = s_code[c0] == last_code && s_code[c0 + CW - 1] == last_code;  // warp-uniform
        const bool act = qok && !(uniform && mx < thr_h);
        if (!__any_sync(0xffffffffu, act)) continue;
        const int jend = nvalid - c0 < CW ? nvalid - c0 : CW;
        // runs of equal codes inside the chunk: one factor (and threshold) per run
        for (int j0 = 0; j0 < jend;) {
          int j1 = jend;
          if (!uniform) {
            const int col0 = c0 + j0;
            const int code = s_code[col0];
            const int e = (int)((int64_t)s_run[col0] - vb) - c0;
            j1 = e < jend ? e : jend;
            if (code != last_code) {
              last_code = code;
              f2 = attr_f2(col0);
              inv_f2 = __frcp_ru(f2);
              set_thr();
            }
          }
          unsigned cand = 0;
#pragma unroll
          for (int j = 0; j < CW; ++j)
            cand |= (j >= j0 && j < j1 && __uint_as_float(r[j]) >= thr_h ? 1u : 0u) << j;
          if (!act) cand = 0;
          j0 = j1;
          while (__any_sync(0xffffffffu, cand != 0)) {
            if (cand) {
              const int j = __ffs(cand) - 1;
              cand &= cand - 1u;
              float zj = 0.f;
#pragma unroll
              for (int jj = 0; jj < CW; ++jj)
                if (jj == j) zj = __uint_as_float(r[jj]);
              process(c0 + j, zj, f2);
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(bar_empty(s));
      mbar_arrive(bar_emptyM(ms));
      // share bounds with the query's other epilogue threads and with the other CTAs
      float pt = a.bound_only ? FLT_MAX : gpre;
      if (PPQ > 1 && !a.bound_only) {
        s_t2[tid] = t2_eff;
#pragma unroll
        for (int q2 = 0; q2 < PPQ; ++q2)
          pt = fminf(pt, s_t2[(lg + 4 * (qt * PPQ + q2)) * 32 + lane_id()]);
      }
      if (pt < t2_eff) {
        t2_eff = pt;
        set_thr();
      }
    }
    if (qok && !a.seed && !a.bound_only) a.cnt[seg] = emitted;
    if (KR > 0 && a.lists && qok) {  // this thread's KR smallest upper keys (FLT_MAX if unfilled)
      const int tq = blockIdx.y * PPQ + part;  // thread index within the query: split, column part
      float* dst = a.lists + ((size_t)my_q * gridDim.y * PPQ + tq) * KR;
#pragma unroll
      for (int j = 0; j < KR; ++j) dst[j] = rl[j];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * QT * N));
  }
}

// segment of query g's sg-th epilogue thread (sg = split * ppq + column part); matches the
// kernel's (CTA, thread) numbering
SB_DEV size_t tf_seg(int64_t g, int sg, int splits, int ppq, int qblock, int ew, int64_t q) {
  const int64_t G = (q + qblock - 1) / qblock;
  const int64_t qb = g / qblock;
  const int w = (int)(g % qblock);
  const int sp = sg / ppq, part = sg % ppq;
  const int qt = w / kTfM, row = w % kTfM;
  const int t = ((row >> 5) + 4 * (qt * ppq + part)) * 32 + (row & 31);
  return ((size_t)sp * G + qb) * (32 * ew) + t;
}

// ---- refine: exact top k of each query's survivors (warp per query) -----------------------
__global__ void tf_refine_kernel(const float* __restrict__ F, const int32_t* __restrict__ A, int m, int l,
                                 const double* __restrict__ qf, const int64_t* __restrict__ qa,
                                 const int64_t* __restrict__ qmask, int64_t q, int k, double alpha,
                                 const uint32_t* __restrict__ cnt, const uint64_t* __restrict__ cand,
                                 int splits, int hsegs, int qblock, int ew, int cap,
                                 const uint32_t* __restrict__ ocnt,
                                 const uint64_t* __restrict__ ocand, int ocap, const int* __restrict__ gthr, int scap, int64_t* out_ids,
                                 double* out_d, int* ovf, int* ovf_count,
                                 unsigned long long* emitted_total) {
  extern __shared__ __align__(16) char smem_raw[];
  const int wpb = blockDim.x >> 5;
  const int wid = warp_id(), lane = lane_id();
  double* sd = reinterpret_cast<double*>(smem_raw) + (size_t)wid * scap;
  uint32_t* si = reinterpret_cast<uint32_t*>(reinterpret_cast<double*>(smem_raw) + (size_t)wpb * scap) +
                 (size_t)wid * scap;
  const int64_t g = (int64_t)blockIdx.x * wpb + wid;
  if (g >= q) return;
  const float t2 = __int_as_float(gthr[g]);
  int kept = 0;
  bool bad = false;
  if (lane == 0) {
    unsigned long long tot = 0;
    for (int sg = 0; sg < splits * hsegs; ++sg) tot += cnt[tf_seg(g, sg, splits, hsegs, qblock, ew, q)];
    tot += ocnt[g];
    atomicAdd(emitted_total, tot);
  }
  // the query's segments (one per split and epilogue thread), then its overflow area
  const int segs = splits * hsegs;
  for (int sg = 0; sg <= segs && !bad; ++sg) {
    const size_t sid = sg < segs ? tf_seg(g, sg, splits, hsegs, qblock, ew, q) : 0;
    const uint32_t c = sg < segs ? cnt[sid] : ocnt[g];
    if (sg == segs && c > (uint32_t)ocap) { bad = true; break; }
    const uint64_t* cg = sg < segs ? cand + sid * cap : ocand + (size_t)g * ocap;
    for (uint32_t base = 0; base < c; base += 32) {
      const uint32_t i = base + lane;
      bool ok = false;
      uint32_t id = 0;
      if (i < c) {
        const uint64_t e = cg[i];
        ok = __uint_as_float((uint32_t)(e >> 32)) <= t2;
        id = (uint32_t)e;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, ok);
      if (kept + __popc(bal) > scap) { bad = true; break; }
      if (ok) si[kept + __popc(bal & ((1u << lane) - 1u))] = id;
      kept += __popc(bal);
    }
  }
  if (kept < k) bad = true;  // cannot happen when nothing overflowed; stay safe
  if (bad) {
    if (lane == 0) {
      ovf[g] = 1;
      atomicAdd(ovf_count, 1);
    }
    return;
  }
  __syncwarp();
  const double* qg = qf + g * (int64_t)m;
  for (int t = lane; t < kept; t += 32) {
    const int64_t v = si[t];
    const double sv = np_pairwise_sq(F + v * (int64_t)m, qg, m);
    int64_t sa = 0;
    for (int u = 0; u < l; ++u) {
      int64_t ad = (int64_t)A[v * (int64_t)l + u] - qa[g * l + u];
      ad = ad < 0 ? -ad : ad;
      sa += qmask ? ad * qmask[g * l + u] : ad;
    }
    sd[t] = dmul(sqrt(sv), dadd(1.0, __ddiv_rn((double)sa, alpha)));
  }
  const int np = next_pow2(kept);
  for (int t = kept + lane; t < np; t += 32) {
    sd[t] = __longlong_as_double(0x7FF0000000000000ll);
    si[t] = 0xFFFFFFFFu;
  }
  __syncwarp();
  warp_bitonic_did(sd, si, np);
  for (int t = lane; t < k; t += 32) {
    out_ids[g * k + t] = (int64_t)si[t];
    out_d[g * k + t] = sd[t];
  }
}

// ---- large k: the bound from every thread's list ------------------------------------------
// lists: q x nl upper keys (each a genuine upper key of a distinct node, or FLT_MAX).  Any k of
// them bound U_k^2 from above, so the k-th smallest is a valid emission bound for the query
// (and close to the exact k-th when the threads' lists cover the query's top k); the query's
// bound becomes the smaller of it and the current one.  CTA per query: bitonic sort of the
// (non-negative, int-ordered) keys in shared memory.
__global__ void tf_select_kernel(const float* __restrict__ lists, int nl, int k, int* gthr) {
  extern __shared__ int sk[];
  const int64_t g = blockIdx.x;
  const int np = next_pow2(nl);
  for (int i = threadIdx.x; i < np; i += blockDim.x)
    sk[i] = i < nl ? __float_as_int(lists[g * nl + i]) : __float_as_int(FLT_MAX);
  __syncthreads();
  for (int size = 2; size <= np; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < np; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          const int x = sk[i], y = sk[j];
          if ((x > y) == up) { sk[i] = y; sk[j] = x; }
        }
      }
      __syncthreads();
    }
  if (threadIdx.x == 0) gthr[g] = min(gthr[g], sk[k - 1]);  // (a bound from an earlier pass may be tighter)
}

int launch_tf_select(const float* lists, int64_t q, int nl, int k, int* gthr, cudaStream_t st) {
  const size_t smem = sizeof(int) * (size_t)next_pow2(nl);
  cudaError_t e = cudaFuncSetAttribute(tf_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  tf_select_kernel<<<(unsigned)q, 256, smem, st>>>(lists, nl, k, gthr);
  return (int)cudaGetLastError();
}

// ---- large k: an exact seed bound from each query's own attribute-code run -------------------
// The nodes are sorted by attribute tuple code (node_order).  For a query whose tuple code is
// c, the M nodes starting at c's run (or the nearest codes when the run is short) get their
// U^2 = S f^2 computed in fp64 (sum order free: any k genuine values bound the k-th from
// above once rounded up), and the k-th smallest, rounded up, becomes the query's starting
// bound.  The strided seed tiles of the tensor-core pass sample popular codes well and rare
// codes badly; this run sample is the other way round, and the smaller of the two is kept.
struct TfCodeSeed {
  int32_t lo[8];
  int64_t stride[8];
};
__global__ void tf_code_seed_kernel(const float* __restrict__ F, const int32_t* __restrict__ A,
                                    const int32_t* __restrict__ s_code, const int32_t* __restrict__ s_orig,
                                    int64_t n, int m, int l, const double* __restrict__ qf,
                                    const int64_t* __restrict__ qa, const int64_t* __restrict__ qmask,
                                    int64_t q, int k, int M, double alpha, TfCodeSeed cs, int* gthr) {
  extern __shared__ uint64_t ks[];
  const int wpb = blockDim.x >> 5;
  const int64_t g = (int64_t)blockIdx.x * wpb + warp_id();
  if (g >= q) return;
  uint64_t* key = ks + (size_t)warp_id() * M;
  const int lane = lane_id();
  int64_t code = 0;
  for (int u = 0; u < l; ++u) code += ((int64_t)qa[g * l + u] - cs.lo[u]) * cs.stride[u];
  int64_t lo = 0, hi = n;  // first sorted position with s_code >= code
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)s_code[mid] < code) lo = mid + 1; else hi = mid;
  }
  int64_t s0 = lo - M / 8;
  if (s0 > n - M) s0 = n - M;
  if (s0 < 0) s0 = 0;
  const double* qv = qf + g * m;
  for (int j = lane; j < M; j += 32) {
    const int64_t v = s_orig[s0 + j];
    const float* x = F + v * m;
    double sv = 0.0;
    for (int t = 0; t < m; ++t) {
      const double d = (double)x[t] - qv[t];
      sv = fma(d, d, sv);
    }
    double sa = 0.0;
    for (int u = 0; u < l; ++u)
      sa += (qmask ? (double)qmask[g * l + u] : 1.0) * fabs((double)A[v * l + u] - (double)qa[g * l + u]);
    const double f = 1.0 + sa / alpha;
    const float u2 = __double2float_ru(sv * f * f * (1.0 + 1e-9));
    key[j] = ((uint64_t)__float_as_uint(u2) << 32) | (uint32_t)j;
  }
  __syncwarp();
  warp_bitonic_u64(key, M);
  if (lane == 0) atomicMin(gthr + g, (int)(key[k - 1] >> 32));
}

int launch_tf_code_seed(const float* F, const int32_t* A, const int32_t* s_code, const int32_t* s_orig,
                        int64_t n, int m, int l, const double* qf, const int64_t* qa,
                        const int64_t* qmask, int64_t q, int k, double alpha, const int32_t* lo8,
                        const int64_t* stride8, int* gthr, cudaStream_t st) {
  int M = 256;
  while (M < 2 * k && M < 2048) M <<= 1;
  if (M > n || k > M) return 0;  // (nothing to seed from)
  TfCodeSeed cs;
  for (int u = 0; u < 8; ++u) { cs.lo[u] = lo8[u]; cs.stride[u] = stride8[u]; }
  const int wpb = 4;
  const size_t smem = sizeof(uint64_t) * (size_t)M * wpb;
  cudaError_t e = cudaFuncSetAttribute(tf_code_seed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  tf_code_seed_kernel<<<(unsigned)((q + wpb - 1) / wpb), 32 * wpb, smem, st>>>(
      F, A, s_code, s_orig, n, m, l, qf, qa, qmask, q, k, M, alpha, cs, gthr);
  return (int)cudaGetLastError();
}

// ---- host side ------------------------------------------------------------------------------
// cE of (1): |S~ - S| <= cE (|x|^2 + |q|^2) for d-dimensional rows (dpad = d rounded up to 8).
//  * operands: |tf32(x) - x| <= 2^-11 |x| (round to nearest), so
//    |sum tf32(x)tf32(q) - x.q| <= (2^-10 + 2^-22) sum |x_t q_t| <= (2^-10 + 2^-22)|x||q|;
//  * accumulation: each of the dpad/8 MMA steps adds at most 16 units of 2^-23 of the sum of
//    magnitudes (a generous allowance for the tensor core's internal alignment and truncation);
//  * fp32 evaluation of |x|^2 + |q|^2 - 2 dot~ and of the keys: a few units of 2^-24 of
//    |x|^2 + |q|^2 (covered by the 2^-19 term);
//  and 2|x||q| <= |x|^2 + |q|^2.  The 1.25 factor is headroom.
double tf_margin(int dpad) {
  const double c_acc = (dpad / 8) * 16.0 * std::ldexp(1.0, -23);
  const double c1 = std::ldexp(1.0, -10) + std::ldexp(1.0, -22) + c_acc * (1.0 + std::ldexp(1.0, -10));
  // + the folded norm column: |hi + lo - (-(1 - cE)|x|^2 / 2)| <= 2^-21 |x|^2
  const double cE = 1.25 * (c1 + std::ldexp(1.0, -21) + std::ldexp(1.0, -20)) + std::ldexp(1.0, -19);
#ifdef SB_TF_MARGIN_SCALE  // tests only: a deliberately wrong margin (tests/test_gpu_tf32.py's
  return cE * SB_TF_MARGIN_SCALE;  // adversarial case must fail with it, see profiles/README.md)
#else
  return cE;
#endif
}

struct TfShape { int N, stages; bool ares; int qt, ew, kr; };

// Tile shape: the first that fits shared memory, in order of preference; wide rows stream both
// operands.  k <= 32 keeps the per-thread lists in registers and runs 16 epilogue warps; larger
// k keeps them in shared memory with 8.
static TfShape tf_shape(int dpad, int l, int kk) {
  if (l > 8 || kk > 256 || dpad > 4096) return {0, 0, false, 0, 0, 0};
  const size_t limit = 227 * 1024;
  int kr = kk <= 16 ? 16 : kk <= 32 ? 32 : 0;
  if (const char* e = getenv("SB_TF_KR")) kr = atoi(e) == 0 ? 0 : kr;  // testing: the smem list
  const int ew = kr > 0 ? 16 : 8;
  if (const char* e = getenv("SB_TF_TILE")) {  // "N,stages,ares,qt" (testing)
    int Nn = 0, st = 0, ar = 0, qt = 1;
    if (sscanf(e, "%d,%d,%d,%d", &Nn, &st, &ar, &qt) == 4 && (Nn == 128 || Nn == 256) && st >= 2 &&
        st <= 8 && (qt == 1 || qt == 2) && 2 * qt * Nn <= 512 &&
        tf_smem_bytes(dpad, l, kk, Nn, st, ar != 0, qt, ew, kr) <= limit)
      return {Nn, st, ar != 0, qt, ew, kr};
  }
  // (N = 256 first: one tf32 MMA instruction moves twice the work of an N = 128 one, and the
  // single issuing thread is the limit for small instructions; measured 9.0 vs 9.9 ms on cfg 3)
  const int pref[][4] = {// N, max stages, min stages, qt (resident query tiles)
                         {256, 6, 3, 1}, {128, 8, 4, 2}, {128, 8, 3, 1}};
  for (auto& pr : pref)
    for (int st = pr[1]; st >= pr[2]; --st)
      if (tf_smem_bytes(dpad, l, kk, pr[0], st, true, pr[3], ew, kr) <= limit)
        return {pr[0], st, true, pr[3], ew, kr};
  const int spref[][2] = {{256, 4}, {256, 3}, {256, 2}, {128, 6}, {128, 4}, {128, 2}};
  for (auto& pr : spref)
    if (tf_smem_bytes(dpad, l, kk, pr[0], pr[1], false, 1, ew, kr) <= limit)
      return {pr[0], pr[1], false, 1, ew, kr};
  return {0, 0, false, 0, 0, 0};
}

int bf_tf_supported(int m, int l, int kk) { return tf_shape(tf_dpad(m), l, kk).N != 0; }
int bf_tf_dpad(int m) { return tf_dpad(m); }

// queries per CTA (query block), epilogue threads per query and epilogue warps of the shape
void bf_tf_layout(int m, int l, int kk, int* qblock, int* ppq, int* ew) {
  const TfShape sh = tf_shape(tf_dpad(m), l, kk);
  *qblock = sh.qt * kTfM;
  *ppq = sh.ew / 4 / sh.qt;
  *ew = sh.ew;
}

int launch_tf_gather(const float* F, const int32_t* A, const int32_t* code_in, const int32_t* orig,
                     int64_t n, int m, int l, double cE, float* Ft, float* nxd, int32_t* code,
                     int32_t* As, cudaStream_t st) {
  const int dpad = tf_dpad(m);
  tf_gather_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(F, A, code_in, orig, n, m, dpad, l, cE,
                                                             Ft, nxd, code, As);
  return (int)cudaGetLastError();
}

int launch_tf_runend(const int32_t* code, int64_t n, int32_t* runend, cudaStream_t st) {
  tf_runend_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(code, n, runend);
  return (int)cudaGetLastError();
}

int launch_tf_prep_queries(const double* qf, int64_t q, int64_t qpad, int m, double cE, double tiny,
                           float* Qt, float* nqs, float* nqu, cudaStream_t st) {
  const int dpad = tf_dpad(m);
  tf_prep_queries_kernel<<<(unsigned)((qpad + 7) / 8), 256, 0, st>>>(qf, q, qpad, m, dpad, cE, tiny,
                                                                     Qt, nqs, nqu);
  return (int)cudaGetLastError();
}

int launch_bf_tf(const float* Ft, const float* nxd, const int32_t* code,
                 const int32_t* orig, const int32_t* runend, const int32_t* As, const float* Qt, const float* nqs,
                 const float* nqu, const int64_t* qa, const int64_t* qmask, int64_t n, int64_t q,
                 int m, int l, int kk, int splits, double alpha, int* gthr, uint32_t* cnt,
                 uint64_t* cand, int cap, uint32_t* ocnt, uint64_t* ocand, int ocap, int seed,
                 int strided, int bound_only, int fixed, float* lists, cudaStream_t st) {
  const int dpad = tf_dpad(m);
  const TfShape sh = tf_shape(dpad, l, kk);
  if (sh.N == 0) return (int)cudaErrorInvalidValue;
  TfArgs a;
  a.Ft = reinterpret_cast<const char*>(Ft); a.nxd = nxd; a.code = code; a.orig = orig;
  a.runend = runend; a.A = As; a.Qt = reinterpret_cast<const char*>(Qt); a.nqs = nqs; a.nqu = nqu; a.qa = qa;
  a.qmask = qmask; a.n = n; a.q = q; a.dpad = dpad; a.l = l; a.kk = kk; a.splits = splits;
  a.stages = sh.stages; a.alpha = alpha; a.gthr = gthr; a.cnt = cnt; a.cand = cand;
  a.cap = cap; a.ocnt = ocnt; a.ocand = ocand; a.ocap = ocap; a.seed = seed;
  a.strided = strided;
  a.bound_only = bound_only; a.fixed = fixed; a.lists = lists;
  const size_t smem = tf_smem_bytes(dpad, l, kk, sh.N, sh.stages, sh.ares, sh.qt, sh.ew, sh.kr);
  void (*kern)(TfArgs) = nullptr;
#define SB_TF_PICK(EW, KR)                                                                          \
  kern = sh.qt == 2 ? bf_tf_kernel<128, true, 2, EW, KR>                                            \
       : sh.N == 256 ? (sh.ares ? bf_tf_kernel<256, true, 1, EW, KR> : bf_tf_kernel<256, false, 1, EW, KR>) \
                     : (sh.ares ? bf_tf_kernel<128, true, 1, EW, KR> : bf_tf_kernel<128, false, 1, EW, KR>)
  if (sh.kr == 16) SB_TF_PICK(16, 16);
  else if (sh.kr == 32) SB_TF_PICK(16, 32);
  else SB_TF_PICK(8, 0);
#undef SB_TF_PICK
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  const int qb = sh.qt * kTfM;
  dim3 grid((unsigned)((q + qb - 1) / qb), (unsigned)splits);
  kern<<<grid, 32 * sh.ew + 64, smem, st>>>(a);
  return (int)cudaGetLastError();
}

int launch_tf_refine(const float* F, const int32_t* A, int m, int l, const double* qf,
                     const int64_t* qa, const int64_t* qmask, int64_t q, int k, double alpha,
                     const uint32_t* cnt, const uint64_t* cand, int splits, int hsegs, int qblock,
                     int ew, int cap,
                     const uint32_t* ocnt, const uint64_t* ocand, int ocap, const int* gthr, int scap, int64_t* out_ids, double* out_d, int* ovf, int* ovf_count,
                     unsigned long long* emitted_total, cudaStream_t st) {
  const int wpb = 4;
  const size_t smem = (size_t)wpb * scap * (sizeof(double) + sizeof(uint32_t));
  cudaError_t e = cudaFuncSetAttribute(tf_refine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  tf_refine_kernel<<<(unsigned)((q + wpb - 1) / wpb), wpb * 32, smem, st>>>(
      F, A, m, l, qf, qa, qmask, q, k, alpha, cnt, cand, splits, hsegs, qblock, ew, cap, ocnt, ocand, ocap, gthr, scap, out_ids, out_d, ovf,
      ovf_count, emitted_total);
  return (int)cudaGetLastError();
}

}  // namespace sb

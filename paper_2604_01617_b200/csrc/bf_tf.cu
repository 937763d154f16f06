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
constexpr int kTfEpi = 256;               // epilogue threads: two per query
constexpr int kTfThreads = kTfEpi + 96;   // + operand loader, MMA and metadata warps
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
  uint32_t* cnt;           // q x segs: candidates each epilogue thread emitted
  uint64_t* cand;          // q x segs x cap: (lower key bits << 32) | original id
  int cap;                 // per segment; segs = splits x (epilogue threads per query per CTA)
  uint32_t* ocnt;          // q: entries in the query's shared overflow area (full segments)
  uint64_t* ocand;         // q x ocap
  int ocap;
  int seed;                // 1: bound-only pass over the first tile of each range (no emission)
  int dbg;                 // timing experiments (SB_TF_DEBUG): 1 = no epilogue work, 2 = no MMAs
};

constexpr int kTfMetaStages = 4;
constexpr int kTfQueue = 8;  // per-thread queue of one tile's filter survivors

SB_HD size_t tf_meta_bytes(int N, int l) { return (size_t)N * (4 + l) * 4; }

// shared layout: [A resident | A stages] | B stages | meta ring | lists | t2 | barriers
SB_HD size_t tf_smem_bytes(int dpad, int l, int kk, int N, int stages, bool ares, int qt) {
  const size_t a = ares ? (size_t)qt * kTfM * dpad * 4 : (size_t)stages * qt * kTfChunkBytes;
  return 1024 + a + (size_t)stages * N * kTfKC * 4 + kTfMetaStages * tf_meta_bytes(N, l) +
         sizeof(float) * (size_t)kk * kTfEpi + sizeof(float) * kTfEpi +
         sizeof(uint64_t) * kTfQueue * kTfEpi + 8 * 32 + 16;
}

// N = nodes per tile, ARES = query tiles resident in shared memory, QT = query tiles (of 128)
// per CTA.  TMEM: 2 buffers x QT x N fp32 columns.  Epilogue warp w reads TMEM lane group w % 4;
// with QT = 2 warps 0..3 own query tile 0 and warps 4..7 tile 1 (all N columns each); with
// QT = 1 they own the two column halves of the one query tile.
template <int N, bool ARES, int QT>
__global__ void __launch_bounds__(kTfThreads, 1) bf_tf_kernel(TfArgs a) {
  constexpr int H = QT == 1 ? 2 : 1;       // epilogue threads per query
  constexpr int cols = N / H;              // columns per epilogue thread and tile
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
  float* ul = reinterpret_cast<float*>(p); p += sizeof(float) * (size_t)a.kk * kTfEpi;
  volatile float* s_t2 = reinterpret_cast<float*>(p); p += sizeof(float) * kTfEpi;
  uint64_t* s_q = reinterpret_cast<uint64_t*>(p); p += sizeof(uint64_t) * kTfQueue * kTfEpi;
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

  const int64_t tiles = (a.n + N - 1) / N;
  const int64_t per = (tiles + a.splits - 1) / a.splits;
  const int64_t t_begin = per * blockIdx.y;
  const int64_t t_end = t_begin + per < tiles ? t_begin + per : tiles;
  int ntl = t_end > t_begin ? (int)(t_end - t_begin) : 0;
  if (a.seed && ntl > 1) ntl = 1;

  if (warp_id() == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(2 * QT * N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == kTfEpi) {
    for (int s = 0; s < S; ++s) {
      mbar_init(bar_full(s), 1);
      mbar_init(bar_sfree(s), 1);
    }
    for (int s = 0; s < kTfMetaStages; ++s) {
      mbar_init(bar_fullM(s), 1);
      mbar_init(bar_emptyM(s), kTfEpi);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar_accf(s), 1);
      mbar_init(bar_empty(s), kTfEpi);
    }
    mbar_init(bar_aready, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < kTfEpi) {
    for (int i = 0; i < a.kk; ++i) ul[i * kTfEpi + tid] = FLT_MAX;
    s_t2[tid] = FLT_MAX;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const char* qblk = a.Qt + (size_t)blockIdx.x * QT * qblk_bytes;

  if (warp_id() == kTfEpi / 32) {
    // ---------------- operand loader ----------------
    if (lane_id() == 0 && ntl > 0) {
      if (ARES) {
        const uint32_t ab = (uint32_t)(QT * qblk_bytes);
        mbar_expect_tx(bar_aready, ab);
        bulk_g2s(smem_u32(sA), qblk, ab, bar_aready);
      }
      int it = 0;
      for (int i = 0; i < ntl; ++i) {
        const int64_t v0 = (t_begin + i) * (int64_t)N;
        for (int c = 0; c < nch; ++c, ++it) {
          const int st = it % S;
          const int use = it / S;
          if (use >= 1) mbar_wait(bar_sfree(st), (uint32_t)((use - 1) & 1));
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
    }
    __syncwarp();
  } else if (warp_id() == kTfEpi / 32 + 2) {
    // ---------------- metadata loader (its own ring, ahead of the accumulators) -------------
    if (lane_id() == 0) {
      for (int i = 0; i < ntl; ++i) {
        const int ms = i % kTfMetaStages;
        const int use = i / kTfMetaStages;
        if (use >= 1) mbar_wait(bar_emptyM(ms), (uint32_t)((use - 1) & 1));
        const int64_t v0 = (t_begin + i) * (int64_t)N;
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
  } else if (warp_id() == kTfEpi / 32 + 1) {
    // ---------------- MMA issuer ----------------
    if (lane_id() == 0 && ntl > 0) {
      // TF32 x TF32 -> F32: c_format = 1 [4,6), a/b format = 2 [7,10) [10,13), N >> 3 [17,23),
      // M >> 4 [24,29), both K-major
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
                             ((uint32_t)(kTfM >> 4) << 24);
      if (ARES) mbar_wait(bar_aready, 0);
      int it = 0;
      for (int i = 0; i < ntl; ++i) {
        const int acc = i & 1;
        if (i >= 2) mbar_wait(bar_empty(acc), (uint32_t)(((i >> 1) - 1) & 1));
        tc_fence_after();
        for (int c = 0; c < nch; ++c, ++it) {
          const int st = it % S;
          mbar_wait(bar_full(st), (uint32_t)((it / S) & 1));
          tc_fence_after();
          const int cw = dpad - 32 * c < 32 ? dpad - 32 * c : 32;
          const uint32_t sbo = (uint32_t)(32 * cw);
          const uint32_t bb = smem_u32(sB + (size_t)st * N * kTfKC * 4);
#pragma unroll
          for (int t = 0; t < QT; ++t) {
            const uint32_t ab = ARES ? smem_u32(sA + t * qblk_bytes + (size_t)c * kTfChunkBytes)
                                     : smem_u32(sA + ((size_t)st * QT + t) * kTfChunkBytes);
            const uint32_t dt = tmem + (uint32_t)((acc * QT + t) * N);
            for (int s = 0; s < cw / 8 && !(a.dbg & 2); ++s) {
              const uint64_t ad = umma_desc(ab + (uint32_t)s * 256, 128, sbo);
              const uint64_t bd = umma_desc(bb + (uint32_t)s * 256, 128, sbo);
              asm volatile(
                  "{\n\t.reg .pred p;\n\t"
                  "setp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dt),
                  "l"(ad), "l"(bd), "r"(idesc), "r"((c | s) != 0 ? 1u : 0u));
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
    const int slot = warp_id() >> 2;
    const int qt = QT == 2 ? slot : 0;            // query tile
    const int half = QT == 1 ? slot : 0;          // column half (QT == 1)
    const int row = lg * 32 + lane_id();
    const int64_t my_q = ((int64_t)blockIdx.x * QT + qt) * kTfM + row;
    const bool qok = my_q < a.q;
    const float nq_s = qok ? a.nqs[my_q] : 0.f;
    const float nq_u = qok ? a.nqu[my_q] : 0.f;
    int32_t qa_row[8];
    int32_t qm_row[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      qa_row[u] = (qok && u < l) ? (int32_t)a.qa[my_q * l + u] : 0;
      qm_row[u] = (qok && u < l) ? (int32_t)(a.qmask ? a.qmask[my_q * l + u] : 1) : 0;
    }
    const float ia = __double2float_ru(1.0 / a.alpha);
    const int kk = a.kk;
    // min(own list tail, partner's, global); starts from the seed pass's bound
    float t2_eff = qok ? fminf(FLT_MAX, __int_as_float(a.gthr[my_q])) : FLT_MAX;
    int last_code = -2;
    float f2 = 1.f, inv_f2 = 1.f, thr_h = -FLT_MAX;
    // y = 2 z >= thr  <=>  lo = nqs - y <= T2 / f^2 (conservatively rounded); thr_h = thr / 2
    auto set_thr = [&]() {
      const float t = t2_eff * inv_f2 * 1.00002f;
      thr_h = t >= FLT_MAX ? -FLT_MAX : 0.5f * (nq_s - t);
    };
    // f^2 of a node's attribute tuple for this query (f = 1 + s_a / alpha, fp32, rounded up)
    const int32_t* s_at_cur = nullptr;
    auto attr_f2 = [&](int col) {
      int sa = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (u < l) sa += abs(s_at_cur[col * l + u] - qa_row[u]) * qm_row[u];
      const float f = fmaf((float)sa, ia, 1.0f);
      return f * f;
    };
    int p_code = -2;   // factor state of the queue processing
    float p_f2 = 1.f;
    const uint32_t lane_base = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(qt * N + half * cols);
    // this thread's private candidate segment: no atomics on the emission path
    const int segs = H * a.splits;
    const size_t seg = (size_t)my_q * segs + H * blockIdx.y + half;
    uint64_t* my_cand = qok ? a.cand + seg * a.cap : nullptr;
    uint32_t emitted = 0;
    for (int i = 0; i < ntl; ++i) {
      const int s = i & 1;
      const uint32_t ph = (uint32_t)((i >> 1) & 1);
      const int ms = i % kTfMetaStages;
      const char* meta = sM + ms * meta_bytes;
      const float* s_nxd = reinterpret_cast<const float*>(meta);
      const int32_t* s_code = reinterpret_cast<const int32_t*>(meta + N * 4);
      const int32_t* s_orig = reinterpret_cast<const int32_t*>(meta + N * 8);
      const int32_t* s_run = reinterpret_cast<const int32_t*>(meta + N * 12);
      s_at_cur = reinterpret_cast<const int32_t*>(meta + N * 16);
      const int64_t vb = (t_begin + i) * (int64_t)N;
      const int nvalid = (int)(a.n - vb < N ? a.n - vb : N);
      const float gpre = qok ? __int_as_float(*reinterpret_cast<volatile int*>(a.gthr + my_q)) : FLT_MAX;
      mbar_wait(bar_fullM(ms), (uint32_t)((i / kTfMetaStages) & 1));
      mbar_wait(bar_accf(s), ph);
      tc_fence_after();
      // one filter survivor: exact-order keys, emission, this thread's upper-key list
      auto process = [&](int col, float zj, float fsq) {
        const float yj = 2.0f * zj;
        const float lo = fmaxf(nq_s - yj, 0.f) * fsq * 0.99998f;
        if (lo > t2_eff) return;
        if (a.dbg & 8) atomicAdd(a.cnt + (size_t)a.q * H * a.splits + 2, 1u);
        // emit: a possible member of the exact top k
        if (!a.seed && !(a.dbg & 16)) {
          const uint64_t e = ((uint64_t)__float_as_uint(lo) << 32) | (uint32_t)s_orig[col];
          if (emitted < (uint32_t)a.cap) {
            my_cand[emitted++] = e;
          } else {  // segment full: the query's shared overflow area
            const uint32_t slot2 = atomicAdd(a.ocnt + my_q, 1u);
            if (slot2 < (uint32_t)a.ocap) a.ocand[(size_t)my_q * a.ocap + slot2] = e;
          }
        }
        // upper key (nqu + nxu - 2 dot = nq_u - y + nxd) into this thread's k smallest
        const float hi = fmaxf(nq_u - yj + s_nxd[col], 0.f) * fsq * 1.00002f;
        if ((a.dbg & 32) || !(hi < ul[(kk - 1) * kTfEpi + tid])) return;
        int pos = kk - 1;
        while (pos > 0) {
          const float pv = ul[(pos - 1) * kTfEpi + tid];
          if (!(hi < pv)) break;
          ul[pos * kTfEpi + tid] = pv;
          --pos;
        }
        ul[pos * kTfEpi + tid] = hi;
        if (a.dbg & 8) atomicAdd(a.cnt + (size_t)a.q * H * a.splits + 3, 1u);
        const float t2 = ul[(kk - 1) * kTfEpi + tid];
        if (t2 < t2_eff) {
          t2_eff = t2;
          set_thr();
          if (!(a.dbg & 64)) atomicMin(a.gthr + my_q, __float_as_int(t2));  // floats >= 0 order as ints
        }
      };
      // scan: the fast filter over the accumulator; survivors wait in a small queue so that
      // the accumulator goes back to the MMA warp as soon as the scan ends
      int qn = 0;
#pragma unroll 1
      for (int c = 0; c < cols / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(lane_base + (uint32_t)(s * QT * N + c * 32), r);
        if (!qok || (a.dbg & 1)) continue;
        const int c0 = half * cols + c * 32;
        // the accumulator holds z = y / 2 with y = 2 x.q - nxs: one max decides the chunk
        float m0 = fmaxf(__uint_as_float(r[0]), __uint_as_float(r[1]));
        float m1 = fmaxf(__uint_as_float(r[2]), __uint_as_float(r[3]));
#pragma unroll
        for (int j = 4; j < 32; j += 2) {
          m0 = fmaxf(m0, __uint_as_float(r[j]));
          m1 = fmaxf(m1, __uint_as_float(r[j + 1]));
        }
        const float mx = fmaxf(m0, m1);
        const bool uniform = s_code[c0] == last_code && s_code[c0 + 31] == last_code;
        if (uniform && mx < thr_h) continue;
        if (a.dbg & 8) atomicAdd(a.cnt + (size_t)a.q * H * a.splits, 1u);
        const int jend = nvalid - c0 < 32 ? nvalid - c0 : 32;
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
          for (int j = 0; j < 32; ++j)
            cand |= (j >= j0 && j < j1 && __uint_as_float(r[j]) >= thr_h ? 1u : 0u) << j;
          j0 = j1;
          if (a.dbg & 8) atomicAdd(a.cnt + (size_t)a.q * H * a.splits + 1, (unsigned)__popc(cand));
          if (a.dbg & 4) continue;
          while (cand) {
            const int j = __ffs(cand) - 1;
            cand &= cand - 1u;
            float zj = 0.f;
#pragma unroll
            for (int jj = 0; jj < 32; ++jj)
              if (jj == j) zj = __uint_as_float(r[jj]);
            if (qn < kTfQueue) {
              s_q[qn * kTfEpi + tid] = ((uint64_t)__float_as_uint(zj) << 32) | (uint32_t)(c0 + j);
              ++qn;
            } else {
              process(c0 + j, zj, f2);  // queue full: now (the scan's factor is this column's)
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(bar_empty(s));
      // the queued survivors, in column order (their codes ascend)
      for (int e = 0; e < qn; ++e) {
        const uint64_t v = s_q[e * kTfEpi + tid];
        const int col = (int)(uint32_t)v;
        const int code = s_code[col];
        if (code != p_code) {
          p_code = code;
          p_f2 = attr_f2(col);
        }
        process(col, __uint_as_float((uint32_t)(v >> 32)), p_f2);
      }
      mbar_arrive(bar_emptyM(ms));
      // share bounds with the other column half (QT == 1) and with the other CTAs
      float pt = gpre;
      if (H == 2) {
        s_t2[tid] = t2_eff;
        pt = fminf(pt, s_t2[tid ^ kTfM]);
      }
      if (pt < t2_eff) {
        t2_eff = pt;
        set_thr();
      }
    }
    if (qok && !a.seed) a.cnt[seg] = emitted;
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * QT * N));
  }
}

// ---- refine: exact top k of each query's survivors (warp per query) -----------------------
__global__ void tf_refine_kernel(const float* __restrict__ F, const int32_t* __restrict__ A, int m, int l,
                                 const double* __restrict__ qf, const int64_t* __restrict__ qa,
                                 const int64_t* __restrict__ qmask, int64_t q, int k, double alpha,
                                 const uint32_t* __restrict__ cnt, const uint64_t* __restrict__ cand,
                                 int segs, int cap, const uint32_t* __restrict__ ocnt,
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
    for (int sg = 0; sg < segs; ++sg) tot += cnt[(size_t)g * segs + sg];
    tot += ocnt[g];
    atomicAdd(emitted_total, tot);
  }
  // segments 0..segs-1, then the overflow area
  for (int sg = 0; sg <= segs && !bad; ++sg) {
    const uint32_t c = sg < segs ? cnt[(size_t)g * segs + sg] : ocnt[g];
    if (sg == segs && c > (uint32_t)ocap) { bad = true; break; }
    const uint64_t* cg = sg < segs ? cand + ((size_t)g * segs + sg) * cap : ocand + (size_t)g * ocap;
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
  return 1.25 * (c1 + std::ldexp(1.0, -21) + std::ldexp(1.0, -20)) + std::ldexp(1.0, -19);
}

struct TfShape { int N, stages; bool ares; int qt; };

// Tile shape: the first that fits shared memory, in order of preference.  Two resident query
// tiles against 128-node tiles halve the node-operand traffic per MMA (L2 -> SM bandwidth is
// the limit of one 128 x 256 TF32 tile per SM); wide rows stream both operands.
static TfShape tf_shape(int dpad, int l, int kk) {
  if (l > 8 || kk > 256 || dpad > 4096) return {0, 0, false, 0};
  const size_t limit = 227 * 1024;
  if (const char* e = getenv("SB_TF_TILE")) {  // "N,stages,ares,qt" (testing)
    int Nn = 0, st = 0, ar = 0, qt = 1;
    if (sscanf(e, "%d,%d,%d,%d", &Nn, &st, &ar, &qt) == 4 && (Nn == 128 || Nn == 256) && st >= 2 &&
        st <= 8 && (qt == 1 || qt == 2) && 2 * qt * Nn <= 512 &&
        tf_smem_bytes(dpad, l, kk, Nn, st, ar != 0, qt) <= limit)
      return {Nn, st, ar != 0, qt};
  }
  const int pref[][4] = {// N, max stages, min stages, qt (resident query tiles)
                         {128, 8, 4, 2}, {256, 6, 3, 1}, {128, 8, 3, 1}};
  for (auto& pr : pref)
    for (int st = pr[1]; st >= pr[2]; --st)
      if (tf_smem_bytes(dpad, l, kk, pr[0], st, true, pr[3]) <= limit) return {pr[0], st, true, pr[3]};
  const int spref[][2] = {{256, 4}, {256, 3}, {256, 2}, {128, 6}, {128, 4}, {128, 2}};
  for (auto& pr : spref)
    if (tf_smem_bytes(dpad, l, kk, pr[0], pr[1], false, 1) <= limit) return {pr[0], pr[1], false, 1};
  return {0, 0, false, 0};
}

int bf_tf_supported(int m, int l, int kk) { return tf_shape(tf_dpad(m), l, kk).N != 0; }
int bf_tf_dpad(int m) { return tf_dpad(m); }

// queries per CTA (query block) and epilogue threads per query of the chosen shape
void bf_tf_layout(int m, int l, int kk, int* qblock, int* hsegs) {
  const TfShape sh = tf_shape(tf_dpad(m), l, kk);
  *qblock = sh.qt * kTfM;
  *hsegs = sh.qt == 1 ? 2 : 1;
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
                 cudaStream_t st) {
  const int dpad = tf_dpad(m);
  const TfShape sh = tf_shape(dpad, l, kk);
  if (sh.N == 0) return (int)cudaErrorInvalidValue;
  TfArgs a;
  a.Ft = reinterpret_cast<const char*>(Ft); a.nxd = nxd; a.code = code; a.orig = orig;
  a.runend = runend; a.A = As; a.Qt = reinterpret_cast<const char*>(Qt); a.nqs = nqs; a.nqu = nqu; a.qa = qa;
  a.qmask = qmask; a.n = n; a.q = q; a.dpad = dpad; a.l = l; a.kk = kk; a.splits = splits;
  a.stages = sh.stages; a.alpha = alpha; a.gthr = gthr; a.cnt = cnt; a.cand = cand;
  a.cap = cap; a.ocnt = ocnt; a.ocand = ocand; a.ocap = ocap; a.seed = seed;
  a.dbg = 0;
  if (const char* e = getenv("SB_TF_DEBUG")) a.dbg = atoi(e);
  const size_t smem = tf_smem_bytes(dpad, l, kk, sh.N, sh.stages, sh.ares, sh.qt);
  void (*kern)(TfArgs) = sh.qt == 2 ? bf_tf_kernel<128, true, 2>
                       : sh.N == 256 ? (sh.ares ? bf_tf_kernel<256, true, 1> : bf_tf_kernel<256, false, 1>)
                                     : (sh.ares ? bf_tf_kernel<128, true, 1> : bf_tf_kernel<128, false, 1>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  const int qb = sh.qt * kTfM;
  dim3 grid((unsigned)((q + qb - 1) / qb), (unsigned)splits);
  kern<<<grid, kTfThreads, smem, st>>>(a);
  return (int)cudaGetLastError();
}

int launch_tf_refine(const float* F, const int32_t* A, int m, int l, const double* qf,
                     const int64_t* qa, const int64_t* qmask, int64_t q, int k, double alpha,
                     const uint32_t* cnt, const uint64_t* cand, int segs, int cap,
                     const uint32_t* ocnt, const uint64_t* ocand, int ocap, const int* gthr, int scap, int64_t* out_ids, double* out_d, int* ovf, int* ovf_count,
                     unsigned long long* emitted_total, cudaStream_t st) {
  const int wpb = 4;
  const size_t smem = (size_t)wpb * scap * (sizeof(double) + sizeof(uint32_t));
  cudaError_t e = cudaFuncSetAttribute(tf_refine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  tf_refine_kernel<<<(unsigned)((q + wpb - 1) / wpb), wpb * 32, smem, st>>>(
      F, A, m, l, qf, qa, qmask, q, k, alpha, cnt, cand, segs, cap, ocnt, ocand, ocap, gthr, scap, out_ids, out_d, ovf,
      ovf_count, emitted_total);
  return (int)cudaGetLastError();
}

}  // namespace sb

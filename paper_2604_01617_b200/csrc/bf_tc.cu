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
// CTA = 128 queries (one per TMEM lane / epilogue thread) x a node range.  Per tile of 256
// nodes: the bf16 node rows are copied into shared memory in the canonical K-major
// no-swizzle core-matrix layout (8 rows x 16 B per core matrix), one elected thread issues
// d/16 tcgen05.mma (M=128, N=256, K=16, BF16 -> F32) into TMEM and commits to an mbarrier;
// each thread then reads its query's 256 dot products with tcgen05.ld and keeps a private
// top-kk list.  A node can enter the list only if sqrt(S) <= T (the factor is >= 1), so the
// epilogue mostly costs one integer compare per (query, node).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "sb_internal.h"

namespace sb {

constexpr int kTcM = 128;       // queries per CTA (UMMA M)
constexpr int kTcN = 256;       // nodes per tile (UMMA N)
constexpr int kTcThreads = 256;  // two threads per query row, each owning half the columns
constexpr int kTcMaxKK = 32;    // per-thread list length limit

// ---- PTX wrappers --------------------------------------------------------------------
SB_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

SB_DEV uint64_t umma_desc(uint32_t start, uint32_t lbo, uint32_t sbo) {
  // K-major, SWIZZLE_NONE canonical layout ((8,n),2):((1,SBO),LBO) in 16-byte units;
  // bits: start[0,14) lbo[16,30) sbo[32,46) version=1 [46,48) layout=0 [61,64)
  uint64_t d = 0;
  d |= (uint64_t)((start >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// BF16 x BF16 -> F32, both K-major, M = 128, N = 256
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kTcN >> 3) << 17) |
                            ((uint32_t)(kTcM >> 4) << 24);

SB_DEV void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate));
}

SB_DEV void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

SB_DEV void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

SB_DEV void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

SB_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
SB_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
SB_DEV void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

SB_DEV void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

SB_DEV void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
SB_DEV void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// byte offset of (row, 16-byte k-chunk) in the core-matrix layout of an R-row tile
SB_DEV uint32_t cm_off(int row, int kc, int R) {
  return (uint32_t)(((kc * (R >> 3) + (row >> 3)) << 7) + ((row & 7) << 4));
}

// ---- prep kernels ----------------------------------------------------------------------
__global__ void tc_prep_queries_kernel(const double* qf, int64_t q, int m, __nv_bfloat16* Qb,
                                       int32_t* nq) {
  int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id();
  if (i >= q) return;
  int acc = 0;
  for (int t = lane_id(); t < m; t += 32) {
    double x = qf[i * m + t];
    Qb[i * m + t] = __float2bfloat16_rn((float)x);
    acc += (int)x * (int)x;
  }
  acc = warp_sum(acc);
  if (lane_id() == 0) nq[i] = acc;
}

// ---- main kernel -------------------------------------------------------------------------
struct TcArgs {
  // node arrays in attribute-grouped order (tc_prepare): nodes with one attribute tuple are
  // contiguous, so the epilogue recomputes the attribute factor only when the tuple changes
  const __nv_bfloat16* Fb;  // n x m
  const int32_t* nx;        // n
  const int32_t* A;         // n x l
  const int32_t* code;      // n: attribute-tuple code (equal codes <=> equal tuples)
  const int32_t* orig;      // n: original node id
  const __nv_bfloat16* Qb;  // q x m
  const int32_t* nq;        // q
  const int64_t* qa;        // q x l
  const int64_t* qmask;     // q x l or null
  int64_t n, q;
  int m, l, kk, splits;
  double alpha;
  double* part_d;           // q x splits x kk
  uint32_t* part_i;
};

__global__ void __launch_bounds__(kTcThreads, 1) bf_tc_kernel(TcArgs a) {
  extern __shared__ __align__(1024) char smem[];
  const int tid = threadIdx.x;
  const int m = a.m;
  // shared layout: A tile | B tile | node norms | node attrs | lists | barrier | tmem slot
  char* p = smem;
  char* sA = p; p += (size_t)kTcM * m * 2;
  char* sB = p; p += (size_t)kTcN * m * 2;
  int32_t* s_nx = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * kTcN;
  int32_t* s_at = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * (size_t)kTcN * a.l;
  int32_t* s_code = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * kTcN;
  int32_t* s_orig = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * kTcN;
  double* ld = reinterpret_cast<double*>(p); p += sizeof(double) * (size_t)kTcMaxKK * kTcThreads;
  uint32_t* li = reinterpret_cast<uint32_t*>(p); p += sizeof(uint32_t) * (size_t)kTcMaxKK * kTcThreads;
  float* s_t2 = reinterpret_cast<float*>(p); p += sizeof(float) * kTcThreads;
  uint64_t* bar = reinterpret_cast<uint64_t*>(p); p += 16;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(p);

  const int64_t q0 = (int64_t)blockIdx.x * kTcM;
  const int split = blockIdx.y;
  const int64_t per = ((a.n + a.splits - 1) / a.splits + kTcN - 1) / kTcN * kTcN;
  const int64_t v_begin = per * split;
  const int64_t v_end = v_begin + per < a.n ? v_begin + per : a.n;
  const int row = tid & (kTcM - 1);   // query row = TMEM lane
  const int half = tid >> 7;          // which 128 columns of each tile this thread owns
  const int64_t my_q = q0 + row;
  const bool qok = my_q < a.q;
  const double inf = __longlong_as_double(0x7FF0000000000000ll);

  // TMEM: 256 fp32 columns (one accumulator of 128 x 256)
  if (warp_id() == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(smem_u32(bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // A tile: this CTA's queries (zero rows past q)
  const int kchunks = m / 8;
  for (int e = tid; e < kTcM * kchunks; e += kTcThreads) {
    int r = e / kchunks, kc = e % kchunks;
    uint32_t dst = smem_u32(sA) + cm_off(r, kc, kTcM);
    if (q0 + r < a.q) cp_async16(dst, a.Qb + (q0 + r) * m + kc * 8);
    else *reinterpret_cast<uint4*>(sA + cm_off(r, kc, kTcM)) = make_uint4(0, 0, 0, 0);
  }
  for (int i = 0; i < a.kk; ++i) {
    ld[i * kTcThreads + tid] = inf;
    li[i * kTcThreads + tid] = 0xFFFFFFFFu;
  }
  cp_async_wait_all();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int32_t my_nq = qok ? a.nq[my_q] : 0;
  int32_t qa_row[8];
  int32_t qm_row[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    qa_row[u] = (qok && u < a.l) ? (int32_t)a.qa[my_q * a.l + u] : 0;
    qm_row[u] = (qok && u < a.l) ? (int32_t)(a.qmask ? a.qmask[my_q * a.l + u] : 1) : 0;
  }
  // Conservative fp32 filter: the exact distance is d = sqrt(S) * (1 + sa/alpha), so a node
  // can beat the list tail T only if S * f^2 <= T^2 with f = 1 + sa * ia, ia <= 1/alpha.
  // fp32 rounding (< 1e-6 relative) is covered by the 1e-5 slack; survivors are decided in
  // exact fp64 below.
  const float ia = __double2float_rd(1.0 / a.alpha);
  float t2 = 3.4e38f;      // own list tail bound
  float t2_eff = 3.4e38f;  // min over both halves of this query
  uint32_t phase = 0;
  int last_code = -2, sa = 0;
  float f2 = 1.0f;

  for (int64_t vb = v_begin; vb < v_end; vb += kTcN) {
    // B tile: node rows (zero rows past the range) + norms + attributes
    for (int e = tid; e < kTcN * kchunks; e += kTcThreads) {
      int r = e / kchunks, kc = e % kchunks;
      int64_t v = vb + r;
      uint32_t off = cm_off(r, kc, kTcN);
      if (v < v_end) cp_async16(smem_u32(sB) + off, a.Fb + v * m + kc * 8);
      else *reinterpret_cast<uint4*>(sB + off) = make_uint4(0, 0, 0, 0);
    }
    for (int r = tid; r < kTcN; r += kTcThreads) {
      int64_t v = vb + r;
      s_nx[r] = v < v_end ? a.nx[v] : 0;
      s_code[r] = v < v_end ? a.code[v] : -1;
      s_orig[r] = v < v_end ? a.orig[v] : 0;
      for (int u = 0; u < a.l; ++u) s_at[r * a.l + u] = v < v_end ? a.A[v * a.l + u] : 0;
    }
    cp_async_wait_all();
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
      for (int s = 0; s < m / 16; ++s) {
        uint64_t ad = umma_desc(a0 + (uint32_t)s * 2 * (kTcM / 8) * 128, (kTcM / 8) * 128, 128);
        uint64_t bd = umma_desc(b0 + (uint32_t)s * 2 * (kTcN / 8) * 128, (kTcN / 8) * 128, 128);
        mma_bf16(tmem, ad, bd, s > 0 ? 1u : 0u);
      }
      mma_commit(smem_u32(bar));
    }
    __syncwarp();
    mbar_wait(smem_u32(bar), phase);
    phase ^= 1u;
    tc_fence_after();
    // epilogue: TMEM lanes 32 * (warp % 4) .. + 31, columns [half * 128, half * 128 + 128)
    const uint32_t lane_base = tmem + ((uint32_t)((warp_id() & 3) * 32) << 16) + (uint32_t)(half * 128);
    const int nvalid = (int)(v_end - vb < kTcN ? v_end - vb : kTcN);
    for (int c = 0; c < 8; ++c) {
      uint32_t r[16];
      tmem_ld16(lane_base + (uint32_t)(c * 16), r);
      if (!qok) continue;
      const int c0 = half * 128 + c * 16;
      // columns are in attribute-grouped order: if both ends of the chunk carry the current
      // tuple, the whole chunk does, and the factor f2 holds for all 16 columns
      unsigned cand = 0;
      if (s_code[c0] == last_code && s_code[c0 + 15] == last_code) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          // S = |x|^2 + |q|^2 - 2 x.q, exact in fp32 (an integer below 2^24)
          const float Sf = fmaf(-2.0f, __uint_as_float(r[j]), (float)(s_nx[c0 + j] + my_nq));
          cand |= (Sf * f2 <= t2_eff ? 1u : 0u) << j;
        }
      } else {
        cand = 0xFFFFu;  // mixed chunk: decide column by column below
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
            if (u < a.l) s2 += abs(s_at[col * a.l + u] - qa_row[u]) * qm_row[u];
          sa = s2;
          const float f = fmaf((float)sa, ia, 1.0f);
          f2 = f * f;
        }
        float rj = 0.f;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj)
          if (jj == j) rj = __uint_as_float(r[jj]);
        const float Sf = fmaf(-2.0f, rj, (float)(s_nx[col] + my_nq));
        if (Sf * f2 > t2_eff) continue;
        // exact fp64 decision (evaluate.py:48-53), ties by original id
        const int S = (int)Sf;
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
          t2_eff = fminf(t2_eff, t2);
        }
      }
    }
    // share list tails between the two threads of a query: a node beyond the other half's
    // kk-th cannot enter the merged top-kk either, so the tighter bound filters both
    s_t2[tid] = t2;
    tc_fence_before();
    __syncthreads();
    t2_eff = fminf(t2, s_t2[tid ^ kTcM]);
  }
  // partial lists out: split index 2 * split + half
  if (qok) {
    const int sp = 2 * split + half;
    size_t o = ((size_t)my_q * (2 * a.splits) + sp) * a.kk;
    for (int i = 0; i < a.kk; ++i) {
      a.part_d[o + i] = ld[i * kTcThreads + tid];
      a.part_i[o + i] = li[i * kTcThreads + tid];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
}

size_t bf_tc_smem(int m, int l) {
  return (size_t)kTcM * m * 2 + (size_t)kTcN * m * 2 + sizeof(int32_t) * kTcN * 3 +
         sizeof(int32_t) * (size_t)kTcN * l + (sizeof(double) + sizeof(uint32_t)) * kTcMaxKK * kTcThreads +
         sizeof(float) * kTcThreads + 64;
}

int bf_tc_supported(int m, int l, int kk) {
  return (m % 16 == 0) && m <= 256 && l <= 8 && kk <= kTcMaxKK && bf_tc_smem(m, l) <= 227 * 1024;
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

// sorted copies: bf16 rows, exact squared norms, codes, attributes (warp per node)
__global__ void tc_gather_kernel(const float* F, const int32_t* A, const int32_t* code_in,
                                 const int32_t* orig, int64_t n, int m, int l,
                                 __nv_bfloat16* Fb, int32_t* nx, int32_t* code, int32_t* As) {
  int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id();
  if (p >= n) return;
  const int64_t v = orig[p];
  int acc = 0;
  for (int t = lane_id(); t < m; t += 32) {
    float x = F[v * m + t];
    Fb[p * m + t] = __float2bfloat16_rn(x);
    acc += (int)x * (int)x;
  }
  acc = warp_sum(acc);
  if (lane_id() == 0) {
    nx[p] = acc;
    code[p] = code_in[v];
  }
  for (int u = lane_id(); u < l; u += 32) As[p * l + u] = A[v * l + u];
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
                     int64_t n, int m, int l, void* Fb, int32_t* nx, int32_t* code, int32_t* As,
                     cudaStream_t st) {
  tc_gather_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(F, A, code_in, orig, n, m, l,
                                                             (__nv_bfloat16*)Fb, nx, code, As);
  return (int)cudaGetLastError();
}

int launch_bf_tc_prep_queries(const double* qf, int64_t q, int m, void* Qb, int32_t* nq,
                              cudaStream_t st) {
  tc_prep_queries_kernel<<<(unsigned)((q + 7) / 8), 256, 0, st>>>(qf, q, m, (__nv_bfloat16*)Qb, nq);
  return (int)cudaGetLastError();
}

int launch_bf_tc(const void* Fb, const int32_t* nx, const int32_t* A, const int32_t* code,
                 const int32_t* orig, const void* Qb, const int32_t* nq, const int64_t* qa,
                 const int64_t* qmask, int64_t n, int64_t q, int m, int l, int kk, int splits,
                 double alpha, double* part_d, uint32_t* part_i, cudaStream_t st) {
  TcArgs a;
  a.Fb = (const __nv_bfloat16*)Fb; a.nx = nx; a.A = A; a.code = code; a.orig = orig;
  a.Qb = (const __nv_bfloat16*)Qb;
  a.nq = nq; a.qa = qa; a.qmask = qmask; a.n = n; a.q = q; a.m = m; a.l = l; a.kk = kk;
  a.splits = splits; a.alpha = alpha; a.part_d = part_d; a.part_i = part_i;
  size_t smem = bf_tc_smem(m, l);
  cudaError_t e = cudaFuncSetAttribute(bf_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  dim3 grid((unsigned)((q + kTcM - 1) / kTcM), (unsigned)splits);
  bf_tc_kernel<<<grid, kTcThreads, smem, st>>>(a);
  return (int)cudaGetLastError();
}

}  // namespace sb

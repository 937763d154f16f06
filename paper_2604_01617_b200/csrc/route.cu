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
// * Entries and expansions share one candidate buffer and one evaluation site, so the whole
//   walk is a single inlined loop (no call-frame spills).
// * Distances, two exact paths:
//     fp64 path (any data): one row per lane, fp64, ascending dimension order, explicitly
//       rounded operations — bit-identical to _query_dist (_kernels.py:26-35).
//     fp32 path (integer data): when features and query are integers and
//       max|x - q|^2 * m < 2^24, every partial sum of squares is an integer below 2^24, so
//       fp32 arithmetic in any order is exact and equals the reference's fp64 sum; lanes then
//       split each row (coalesced 128-bit loads, 8 rows in flight) and reduce with shuffles.
//     The attribute term and the final sqrt(s_v) * (1 + s_a * inv_alpha) are fp64 as in the
//     reference in both paths.
// * Visited set: exact, one bitset of ceil(n/32) words per warp slot in HBM, set with
//   atomicOr (test-and-set); cleared after each query from a per-slot log of visited ids
//   (a full clear when the log overflows).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "rng.cuh"
#include "sb_internal.h"
#include "tc_ptx.cuh"

#include <cub/device/device_radix_sort.cuh>

namespace sb {

constexpr uint32_t kChkR = 0x80000000u;   // phase-2 checked
constexpr uint32_t kChkP = 0x40000000u;   // phase-1 (pioneer) checked
constexpr uint32_t kIdMask = 0x3FFFFFFFu;
constexpr int kRows = 8;                   // rows per lane group in flight (fp32 path)
#ifndef ROUTE_F32_CHUNK
#define ROUTE_F32_CHUNK 8                  // float4 loads in flight per lane (fp32 lane path)
#endif

#ifndef ROUTE_DEEP_SLOTS
#define ROUTE_DEEP_SLOTS 8  // 4-float4 slots in flight per lane in the kModeF64Deep instance
#endif
constexpr int kLazyB = 64;  // insertion buffer of the large-K kernel instances
constexpr int kLazyK = 1024; // K from which routing uses the insertion buffer
constexpr int kLazyW = kLazyB + 2;  // cached window of R below a rank bound (kLazyB + 1 entries used)
#ifndef ROUTE_FAST_MERGE
#define ROUTE_FAST_MERGE 1
#endif
constexpr bool kFastMerge = ROUTE_FAST_MERGE != 0;  // warp_merge_lanes for batches of <= 32

struct WarpSmem {
  double* bd;     // kLazyB (large-K instances)
  uint32_t* bid;  // kLazyB
  double* wd;     // 2 x kLazyW: R[hi - 1 - j], j = 0..kLazyB, for hi = K and hi = P (large-K instances)
  uint32_t* wi;   // 2 x kLazyW
  double* rd;     // Kpad
  double* cd;     // Cpad
  double* qs;     // m
  double* qas;    // l
  double* qms;    // l
  float* qs32;    // m (fp32 copy of the query, integer path)
  uint32_t* rid;  // Kpad
  uint32_t* cid;  // Cpad
  int* cpos;      // Cpad
  char* ring;     // kModeF64Deep: ring_slots x kRingSlotB row-line staging
};

constexpr int kRingSlotB = 144;  // one 128-byte row line + 16 bytes: conflict-free lane-per-row reads
constexpr int kRingStages = 4;   // cp.async groups in flight per round (kModeF64Deep)
SB_HD size_t route_warp_smem_bytes_full(int Kpad, int Cpad, int m, int l, bool lazy,
                                         bool rglobal = false, int ring_slots = 0) {
  if (rglobal) Kpad = 0;  // R lives in global memory
  size_t b = (size_t)((m + 3) & ~3) * 4;  // fp32 query first: 16-byte aligned float4 reads
  if (lazy) b += (size_t)(kLazyB + 2 * kLazyW) * 12;
  // the fp64 query is padded with zeros to whole 32-dimension lines (staged evaluation)
  b += (size_t)Kpad * 8 + (size_t)Cpad * 8 + (size_t)((m + 31) & ~31) * 8 + (size_t)l * 16;
  b += (size_t)Kpad * 4 + (size_t)Cpad * 8;
  b = (b + 15) & ~(size_t)15;
  return b + (ring_slots ? (size_t)ring_slots * kRingSlotB + 256 : 0);  // + 32 row pointers
}

template <bool LAZY>
SB_DEV WarpSmem carve(char* base, const RouteArgs& a, int64_t slot) {
  const bool rg = LAZY && a.gr_d != nullptr;  // global lists only in the large-K instance
  WarpSmem w;
  w.qs32 = reinterpret_cast<float*>(base);
  double* dp = reinterpret_cast<double*>(base + (size_t)((a.m + 3) & ~3) * 4);
  w.qs = dp; dp += (a.m + 31) & ~31;  // 16-byte aligned (double2 reads), zero-padded to lines
  w.bd = nullptr;
  w.bid = nullptr;
  w.wd = nullptr;
  w.wi = nullptr;
  if (LAZY) {
    w.bd = dp;
    dp += kLazyB;
    w.wd = dp;
    dp += 2 * kLazyW;
    w.bid = reinterpret_cast<uint32_t*>(dp);
    w.wi = w.bid + kLazyB;
    dp = reinterpret_cast<double*>(w.wi + 2 * kLazyW);
  }
  if (rg) {
    w.rd = a.gr_d + slot * a.Kpad;
  } else {
    w.rd = dp;
    dp += a.Kpad;
  }
  w.cd = dp; dp += a.Cpad;
  w.qas = dp; dp += a.l;
  w.qms = dp; dp += a.l;
  uint32_t* up = reinterpret_cast<uint32_t*>(dp);
  if (rg) {
    w.rid = a.gr_i + slot * a.Kpad;
  } else {
    w.rid = up;
    up += a.Kpad;
  }
  w.cid = up; up += a.Cpad;
  w.cpos = reinterpret_cast<int*>(up);
  w.ring = base + route_warp_smem_bytes_full(a.Kpad, a.Cpad, a.m, a.l, LAZY, rg, 0);
  return w;
}

// attribute term + final fp64 AUTO combination, exactly _query_dist's tail (_kernels.py:32-35)
SB_DEV double finish_row(const RouteArgs& a, const WarpSmem& w, uint32_t v, double s_v) {
  const int32_t* av = a.A + (int64_t)v * a.l;
  double sa = 0.0;
  for (int u = 0; u < a.l; ++u)
    sa = dadd(sa, dmul(w.qms[u], fabs(dsub((double)__ldg(av + u), w.qas[u]))));
  return auto_finish(s_v, sa, a.inv_alpha);
}

// attribute codes loaded early (first 4 in registers) so their latency overlaps the row loads
struct AttrPre {
  int32_t v[4];
};
SB_DEV void attr_preload(const RouteArgs& a, uint32_t node, AttrPre& p) {
  const int32_t* av = a.A + (int64_t)node * a.l;
#pragma unroll
  for (int u = 0; u < 4; ++u)
    if (u < a.l) p.v[u] = __ldg(av + u);
}
SB_DEV double finish_pre(const RouteArgs& a, const WarpSmem& w, uint32_t node, const AttrPre& p,
                         double s_v) {
  double sa = 0.0;
#pragma unroll
  for (int u = 0; u < 4; ++u)
    if (u < a.l) sa = dadd(sa, dmul(w.qms[u], fabs(dsub((double)p.v[u], w.qas[u]))));
  const int32_t* av = a.A + (int64_t)node * a.l;
  for (int u = 4; u < a.l; ++u)
    sa = dadd(sa, dmul(w.qms[u], fabs(dsub((double)__ldg(av + u), w.qas[u]))));
  return auto_finish(s_v, sa, a.inv_alpha);
}

// distance path of a route_kernel instance (each instance carries only its own path, plus the
// generic fp64 path as the per-query fallback of the integer paths)
enum RouteMode { kModeF64x4 = 0, kModeF32Lane = 1, kModeF32Split = 2, kModeGeneric = 3, kModeU8 = 4,
                 kModeF64Filt = 5, kModeF64Deep = 6 };

// 16-byte read-only loads of a row with an L2 prefetch-size hint: a miss brings the whole
// 128-byte line in one DRAM access instead of one access per 32-byte sector (ROUTE_L2PF: 0 = plain
// __ldg, 128 / 256 = hint size)
#ifndef ROUTE_L2PF
#define ROUTE_L2PF 128
#endif
SB_DEV uint4 ldg_row(const uint4* p) {
#if ROUTE_L2PF == 128
  uint4 v;
  asm("ld.global.nc.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
#elif ROUTE_L2PF == 256
  uint4 v;
  asm("ld.global.nc.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}
SB_DEV float4 ldg_row(const float4* p) {
  const uint4 v = ldg_row(reinterpret_cast<const uint4*>(p));
  return make_float4(__uint_as_float(v.x), __uint_as_float(v.y), __uint_as_float(v.z), __uint_as_float(v.w));
}

// fp32 -> fp64 without the conversion unit (F2F runs at a quarter of the fp64 rate and was the
// busiest pipe of the real-valued walk): the float's fields dropped into a double's give
// X = x * 2^-896 exactly (zero and subnormal floats land on subnormal doubles, which fp64
// handles at full speed), so fma(X, 2^896, -q) is the correctly rounded x - q: the same value
// as __dsub_rn((double)x, q) for every finite x.
SB_DEV double f2d_scaled(float x) {
  const int xi = __float_as_int(x);
  return __hiloint2double((xi >> 3) & (int)0x8FFFFFFF, xi << 29);
}
SB_DEV double sq_diff(float x, double q) {
  const double d = __fma_rn(f2d_scaled(x), 0x1p896, -q);
  return dmul(d, d);
}

SB_DEV void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
SB_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
SB_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// kModeF64Deep: exact distances of rows cid[0..c) -> cd[0..c), _query_dist's sequential fp64 sum
// (bit-identical: the order of the additions is the reference's; padded dimensions add +0.0).
//  * Loads: the warp copies the rows into a shared-memory ring one 128-byte line per row at a
//    time with cp.async, 8 lanes per line (whole-line requests: one row per lane with 16-byte
//    loads is bounded by the single-sector request rate, tools/probes/rowwalk_bw.cu), four
//    groups of lines in flight, the ring as deep as its slots allow for the round's rows.
//  * Chain: lane r walks row r out of the ring; the squares (x - q)^2 of the next 16
//    dimensions are computed between the dependent adds of the current 16, so the chain
//    advances at the latency of one fp64 add, and the loop body is small (no unrolled row).
SB_DEV void eval_rows_staged(const RouteArgs& a, WarpSmem& w, int c) {
  const int lane = lane_id();
  const int rowb = a.m * 4;
  const int nln = (rowb + 127) >> 7;  // 128-byte lines per row
  const uint32_t ring = smem_u32(w.ring);
  const int sub = lane & 7, grp = lane >> 3;
  const double2* q2 = reinterpret_cast<const double2*>(w.qs);
  // row pointers of the round, behind the ring (one per row: the copies read them back)
  const char** rowptr = reinterpret_cast<const char**>(w.ring + (size_t)a.ring_slots * kRingSlotB);
  const int cr_max = a.ring_slots / kRingStages < 32 ? a.ring_slots / kRingStages : 32;
  for (int base = 0; base < c; base += cr_max) {
    const int cr = c - base < cr_max ? c - base : cr_max;
    int lps = a.ring_slots / (cr * kRingStages);  // lines per row per group
    if (lps > 8) lps = 8;
    const int nlr = lps * kRingStages;             // lines per row the ring holds
    const int ngr = (cr + 3) >> 2;
    const int my = lane < cr ? lane : cr - 1;      // idle lanes shadow the last row (no divergence)
    const uint32_t v = w.cid[base + my];
    if (lane < cr) rowptr[lane] = reinterpret_cast<const char*>(a.F) + (int64_t)v * rowb;
    AttrPre pre;
    attr_preload(a, v, pre);
    __syncwarp();
    int issue_ln = 0, issue_pos = 0;
    // one group: the next `lps` lines of every row of the round; 8 lanes copy one line, so a
    // warp instruction moves four rows' lines: rows grp, grp + 4, ... of this lane's group (the
    // first four pointers in registers, any further row through the shared-memory table)
    const char* rp[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) rp[i] = rowptr[grp + 4 * i < cr ? grp + 4 * i : my] + sub * 16;
    const uint32_t dst0 = ring + (uint32_t)(grp * kRingSlotB + sub * 16);
    const uint32_t line_b = (uint32_t)(cr * kRingSlotB);
    auto issue_group = [&]() {
      for (int k = 0; k < lps; ++k) {
        if (issue_ln < nln) {
          const int off = issue_ln * 128;
          const int sz = off + sub * 16 < rowb ? 16 : 0;  // past the row's end: zero fill
          const int so = sz ? off : 0;
          const uint32_t dst = dst0 + (uint32_t)issue_pos * line_b;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (grp + 4 * i < cr) cp_async16(dst + (uint32_t)(4 * i * kRingSlotB), rp[i] + so, sz);
          for (int r = grp + 16; r < cr; r += 4)
            cp_async16(dst + (uint32_t)((r - grp) * kRingSlotB), rowptr[r] + sub * 16 + so, sz);
        }
        ++issue_ln;
        issue_pos = issue_pos + 1 == nlr ? 0 : issue_pos + 1;
      }
      cp_async_commit();
    };
#pragma unroll
    for (int g = 0; g < kRingStages; ++g) issue_group();
    cp_async_wait<kRingStages - 1>();
    __syncwarp();
    // Software pipeline over half lines (16 dimensions): at the top of a step, t holds the
    // squares of the current half line and (x, q) the raw inputs of the next one, read from
    // shared memory a step ahead, so the squares never wait for their loads and can sit between
    // the dependent adds.
    double s = 0.0;
    double t[16];
    float4 x[4];
    double2 q[8];
    auto fetch = [&](int pos, int h, int e) {
      const float4* x4 = reinterpret_cast<const float4*>(w.ring + (size_t)(pos * cr + my) * kRingSlotB + h * 64);
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = x4[u];
#pragma unroll
      for (int u = 0; u < 8; ++u) q[u] = q2[(e >> 1) + u];
    };
    auto square = [&](int u4, bool accumulate) {  // dimensions 4 u4 .. 4 u4 + 3 of the half line
      if (accumulate) s = dadd(s, t[4 * u4 + 0]);
      t[4 * u4 + 0] = sq_diff(x[u4].x, q[2 * u4].x);
      if (accumulate) s = dadd(s, t[4 * u4 + 1]);
      t[4 * u4 + 1] = sq_diff(x[u4].y, q[2 * u4].y);
      if (accumulate) s = dadd(s, t[4 * u4 + 2]);
      t[4 * u4 + 2] = sq_diff(x[u4].z, q[2 * u4 + 1].x);
      if (accumulate) s = dadd(s, t[4 * u4 + 3]);
      t[4 * u4 + 3] = sq_diff(x[u4].w, q[2 * u4 + 1].y);
    };
    // step: s += t; t <- squares of (x, q); (x, q) <- the half line at (pos, h) when `more`
    auto step = [&](bool more, int pos, int h, int e) {
      float4 xn[4];
      double2 qn[8];
      if (more) {
        const float4* x4 = reinterpret_cast<const float4*>(w.ring + (size_t)(pos * cr + my) * kRingSlotB + h * 64);
#pragma unroll
        for (int u = 0; u < 4; ++u) xn[u] = x4[u];
#pragma unroll
        for (int u = 0; u < 8; ++u) qn[u] = q2[(e >> 1) + u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) square(u, true);
      if (more) {
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = xn[u];
#pragma unroll
        for (int u = 0; u < 8; ++u) q[u] = qn[u];
      }
    };
    fetch(0, 0, 0);
#pragma unroll
    for (int u = 0; u < 4; ++u) square(u, false);
    fetch(0, 1, 16);
    int pos = 0, in_group = 0;
    for (int ln = 0; ln < nln; ++ln) {
      // t: squares of (ln, 0); (x, q): inputs of (ln, 1).  Line ln + 1 is read during this
      // iteration: when it opens a new group that group must have landed, and the group before
      // the current one (every lane has it in registers: the __syncwarp) is refilled.
      if (++in_group == lps) {
        in_group = 0;
        cp_async_wait<kRingStages - 2>();
        __syncwarp();
        issue_group();
      }
      const int npos = pos + 1 == nlr ? 0 : pos + 1;
      const bool more = ln + 1 < nln;
      step(more, npos, 0, ln * 32 + 32);  // adds (ln, 0), squares (ln, 1), reads (ln + 1, 0)
      if (more) {
        step(true, npos, 1, ln * 32 + 48);  // adds (ln, 1), squares (ln + 1, 0), reads (ln + 1, 1)
      } else {
#pragma unroll
        for (int u = 0; u < 16; ++u) s = dadd(s, t[u]);
      }
      pos = npos;
    }
    cp_async_wait<0>();
    if (lane < cr) w.cd[base + lane] = finish_pre(a, w, v, pre, s);
    __syncwarp();  // the ring and the row pointers are free for the next round
  }
}

// attribute factor of _query_dist's finish: 1 + s_a * inv_alpha, computed exactly as
// finish_row does (_kernels.py:32-35)
SB_DEV double attr_factor(const RouteArgs& a, const WarpSmem& w, uint32_t v) {
  const int32_t* av = a.A + (int64_t)v * a.l;
  double sa = 0.0;
  for (int u = 0; u < a.l; ++u)
    sa = dadd(sa, dmul(w.qms[u], fabs(dsub((double)__ldg(av + u), w.qas[u]))));
  return dadd(1.0, dmul(sa, a.inv_alpha));
}

// Exact distances of rows cid[0..c) -> cd[0..c).  tau: the admission tail of the result list
// (+inf while the entries fill it); qn: |q| (fp64), both used only by the filtered path.
template <int MODE>
SB_DEV void eval_rows(const RouteArgs& a, WarpSmem& w, int c, bool f32, int nq8, double tau,
                      double qn) {
  const int lane = lane_id();
  if (MODE == kModeU8 && f32) {
    // features and query are integers in [0, 255]: rows are read from the u8 copy and
    // S = |x|^2 + |q|^2 - 2 x.q with x.q from byte dot products (dp4a), exact in int32
    const int n16 = a.m >> 4;
    const uint4* Q = reinterpret_cast<const uint4*>(w.qs32);
    for (int j = lane; j < c; j += 32) {
      const uint32_t v = w.cid[j];
      const uint4* xr = reinterpret_cast<const uint4*>(a.F8 + (int64_t)v * a.m);
      AttrPre pre;
      int nxv;
      if (a.meta16) {  // |x|^2 and up to three attributes in one 16-byte load
        const uint4 mt = __ldg(a.meta16 + v);
        nxv = (int)mt.x;
        pre.v[0] = (int32_t)mt.y; pre.v[1] = (int32_t)mt.z; pre.v[2] = (int32_t)mt.w; pre.v[3] = 0;
      } else {
        attr_preload(a, v, pre);
        nxv = __ldg(a.nx8 + v);
      }
      unsigned acc0 = 0u, acc1 = 0u;
      int k = 0;
      for (; k + 8 <= n16; k += 8) {
        uint4 r[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = ldg_row(xr + k + u);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint4 q = Q[k + u];
          acc0 = __dp4a(r[u].x, q.x, acc0);
          acc1 = __dp4a(r[u].y, q.y, acc1);
          acc0 = __dp4a(r[u].z, q.z, acc0);
          acc1 = __dp4a(r[u].w, q.w, acc1);
        }
      }
      for (; k < n16; ++k) {
        const uint4 r = ldg_row(xr + k);
        const uint4 q = Q[k];
        acc0 = __dp4a(r.x, q.x, acc0);
        acc1 = __dp4a(r.y, q.y, acc1);
        acc0 = __dp4a(r.z, q.z, acc0);
        acc1 = __dp4a(r.w, q.w, acc1);
      }
      const int S = nxv + nq8 - 2 * (int)(acc0 + acc1);
      w.cd[j] = finish_pre(a, w, v, pre, (double)S);
    }
  } else if (MODE == kModeF32Lane && f32) {
    // integer data, one row per lane: fp32 with four independent accumulators (every
    // partial sum is an integer below 2^24, so the order is free and the result exact)
    const int nq = a.m >> 2;
    const float4* Q4 = reinterpret_cast<const float4*>(w.qs32);
    for (int j = lane; j < c; j += 32) {
      const uint32_t v = w.cid[j];
      const float4* vx = reinterpret_cast<const float4*>(a.F) + (int64_t)v * nq;
      AttrPre pre;
      attr_preload(a, v, pre);
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
      auto step = [&](const float4 x, const float4 qv) {
        const float d0 = x.x - qv.x, d1 = x.y - qv.y, d2 = x.z - qv.z, d3 = x.w - qv.w;
        s0 = fmaf(d0, d0, s0);
        s1 = fmaf(d1, d1, s1);
        s2 = fmaf(d2, d2, s2);
        s3 = fmaf(d3, d3, s3);
      };
      int qq = 0;
      for (; qq + ROUTE_F32_CHUNK <= nq; qq += ROUTE_F32_CHUNK) {
        float4 r[ROUTE_F32_CHUNK];
#pragma unroll
        for (int u = 0; u < ROUTE_F32_CHUNK; ++u) r[u] = __ldg(vx + qq + u);
#pragma unroll
        for (int u = 0; u < ROUTE_F32_CHUNK; ++u) step(r[u], Q4[qq + u]);
      }
      for (; qq < nq; ++qq) step(__ldg(vx + qq), Q4[qq]);
      w.cd[j] = finish_pre(a, w, v, pre, (double)((s0 + s1) + (s2 + s3)));
    }
  } else if (MODE == kModeF32Split && f32) {
    const int lpr = a.lpr;
    const int rpp = 32 / lpr;
    const int sub = lane & (lpr - 1);
    const int grp = lane / lpr;
    const int nq = a.m >> 2;
    const float4* F4 = reinterpret_cast<const float4*>(a.F);
    for (int base = 0; base < c; base += rpp * kRows) {
      float acc[kRows];
      uint32_t id[kRows];
#pragma unroll
      for (int g = 0; g < kRows; ++g) {
        int r = base + grp + rpp * g;
        id[g] = r < c ? w.cid[r] : 0xFFFFFFFFu;
        acc[g] = 0.f;
      }
      // lane `sub == g` finishes row g (needs lpr >= kRows); its attributes load now
      uint32_t own = 0xFFFFFFFFu;
#pragma unroll
      for (int g = 0; g < kRows; ++g)
        if (g == sub) own = id[g];
      AttrPre pre;
      if (lpr >= kRows && own != 0xFFFFFFFFu) attr_preload(a, own, pre);
      for (int k = sub; k < nq; k += lpr) {
        float4 x[kRows];
#pragma unroll
        for (int g = 0; g < kRows; ++g)
          if (id[g] != 0xFFFFFFFFu) x[g] = __ldg(F4 + (int64_t)id[g] * nq + k);
        const float4 qv = reinterpret_cast<const float4*>(w.qs32)[k];
#pragma unroll
        for (int g = 0; g < kRows; ++g)
          if (id[g] != 0xFFFFFFFFu) {
            float d0 = x[g].x - qv.x, d1 = x[g].y - qv.y, d2 = x[g].z - qv.z, d3 = x[g].w - qv.w;
            acc[g] = fmaf(d0, d0, acc[g]);
            acc[g] = fmaf(d1, d1, acc[g]);
            acc[g] = fmaf(d2, d2, acc[g]);
            acc[g] = fmaf(d3, d3, acc[g]);
          }
      }
#pragma unroll
      for (int g = 0; g < kRows; ++g)
        for (int o = lpr >> 1; o > 0; o >>= 1) acc[g] += __shfl_xor_sync(0xffffffffu, acc[g], o);
      if (lpr >= kRows) {
        if (own != 0xFFFFFFFFu) {
          float tot = 0.f;
#pragma unroll
          for (int g = 0; g < kRows; ++g)
            if (g == sub) tot = acc[g];
          w.cd[base + grp + rpp * sub] = finish_pre(a, w, own, pre, (double)tot);
        }
      } else if (sub == 0) {
#pragma unroll
        for (int g = 0; g < kRows; ++g)
          if (id[g] != 0xFFFFFFFFu) w.cd[base + grp + rpp * g] = finish_row(a, w, id[g], (double)acc[g]);
      }
    }
  } else if (MODE == kModeF64Deep) {
    eval_rows_staged(a, w, c);
  } else if (MODE == kModeF64x4 || MODE == kModeF64Filt) {
    const int nq = a.m >> 2;
    int ns = c;  // rows that need the exact value: all, or the filter's survivors (w.cpos)
    const bool filt = MODE == kModeF64Filt && tau < __longlong_as_double(0x7FF0000000000000ll);
    if (filt) {
      // (1) Certified lower bound per row from fp32 arithmetic with coalesced loads: lpr lanes
      // split each row (float4 k = sub, sub + lpr, ...), two rows per lane group in flight.
      // With u = 2^-24, e_t = fl32(x_t - fl32(q_t)) and S~ = the fp32 sum of e_t^2:
      //   |q - x| >= sqrt(S~ (1 - (m + 64) u)) (1 - u) - u |q|     (summation error of at most
      //   m + 64 additions per chain, the rounding of x - q and of q to fp32),
      // and the reference's fp64 value U = fl(sqrt(S_seq) * f) >= |q - x| f (1 - (m + 8) 2^-52)
      // with the same attribute factor f.  A row whose bound exceeds tau cannot enter R (nor
      // the pioneer list, a prefix of R), so its exact value is never needed; every other row
      // gets the exact sequential fp64 value below.  Ids, distances and counters are unchanged.
      const int lpr = a.flt_lpr;
      const int G = 32 / lpr;
      const int sub = lane & (lpr - 1), grp = lane / lpr;
      const float4* F4 = reinterpret_cast<const float4*>(a.F);
      const float4* Q4 = reinterpret_cast<const float4*>(w.qs32);
      const double uu = 5.9604644775390625e-08;  // 2^-24
      const double shrink = 1.0 - (a.m + 64) * uu;
      const double fin = 1.0 - (a.m + 8) * 2.220446049250313e-16;
      for (int base = 0; base < c; base += 2 * G) {
        const int r0 = base + grp, r1 = base + G + grp;
        const uint32_t v0 = r0 < c ? w.cid[r0] : 0u, v1 = r1 < c ? w.cid[r1] : 0u;
        float s0a = 0.f, s0b = 0.f, s1a = 0.f, s1b = 0.f;
        const float4* x0p = F4 + (int64_t)v0 * nq;
        const float4* x1p = F4 + (int64_t)v1 * nq;
#pragma unroll 4
        for (int k = sub; k < nq; k += lpr) {
          const float4 qv = Q4[k];
          const float4 x0 = r0 < c ? __ldg(x0p + k) : qv;
          const float4 x1 = r1 < c ? __ldg(x1p + k) : qv;
          float d;
          d = x0.x - qv.x; s0a = fmaf(d, d, s0a);
          d = x0.y - qv.y; s0b = fmaf(d, d, s0b);
          d = x0.z - qv.z; s0a = fmaf(d, d, s0a);
          d = x0.w - qv.w; s0b = fmaf(d, d, s0b);
          d = x1.x - qv.x; s1a = fmaf(d, d, s1a);
          d = x1.y - qv.y; s1b = fmaf(d, d, s1b);
          d = x1.z - qv.z; s1a = fmaf(d, d, s1a);
          d = x1.w - qv.w; s1b = fmaf(d, d, s1b);
        }
        float t0 = s0a + s0b, t1 = s1a + s1b;
        for (int o = lpr >> 1; o > 0; o >>= 1) {
          t0 += __shfl_xor_sync(0xffffffffu, t0, o);
          t1 += __shfl_xor_sync(0xffffffffu, t1, o);
        }
        if (sub == 0) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = h ? r1 : r0;
            if (r >= c) continue;
            const double S = (double)(h ? t1 : t0);
            double rl = sqrt(S * shrink) * (1.0 - uu) - uu * qn;
            rl = rl > 0.0 ? rl : 0.0;
            const double lo = rl * attr_factor(a, w, h ? v1 : v0) * fin;
            w.cd[r] = lo > tau ? __longlong_as_double(0x7FF0000000000000ll) : -1.0;
          }
        }
      }
      __syncwarp();
      // survivors -> w.cpos[0..ns)
      ns = 0;
      for (int b = 0; b < c; b += 32) {
        const int j = b + lane;
        const bool need = j < c && w.cd[j] < 0.0;
        const unsigned bal = __ballot_sync(0xffffffffu, need);
        if (need) w.cpos[ns + __popc(bal & ((1u << lane) - 1u))] = j;
        ns += __popc(bal);
      }
      __syncwarp();
    }
    for (int t = lane; t < ns; t += 32) {
      const int j = filt ? w.cpos[t] : t;
      const uint32_t v = w.cid[j];

      const float4* vx = reinterpret_cast<const float4*>(a.F) + (int64_t)v * nq;
      AttrPre pre;
      attr_preload(a, v, pre);
      double s = 0.0;
      auto step = [&](const float4 x, const double* qv) {
        s = sq_step(s, x.x, qv[0]);
        s = sq_step(s, x.y, qv[1]);
        s = sq_step(s, x.z, qv[2]);
        s = sq_step(s, x.w, qv[3]);
      };
      int qq = 0;
      for (; qq + 8 <= nq; qq += 8) {
        float4 r[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = __ldg(vx + qq + u);
#pragma unroll
        for (int u = 0; u < 8; ++u) step(r[u], w.qs + 4 * (qq + u));
      }
      for (; qq < nq; ++qq) step(__ldg(vx + qq), w.qs + 4 * qq);
      w.cd[j] = finish_pre(a, w, v, pre, s);
    }
  } else {
    for (int j = lane; j < c; j += 32) {
      const uint32_t v = w.cid[j];
      const float* x = a.F + (int64_t)v * a.m;
      double s = 0.0;
#pragma unroll 4
      for (int t = 0; t < a.m; ++t) s = sq_step(s, __ldg(x + t), w.qs[t]);
      w.cd[j] = finish_row(a, w, v, s);
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

// first position in [lb, hi) whose id word lacks `bit`, with that entry's distance and id (the
// distances ride along with the flag words: one memory round trip); -1 if none
SB_DEV int first_unchecked_d(const double* rd, const uint32_t* rid, int lb, int hi, uint32_t bit,
                             double* dsel, uint32_t* isel) {
  for (int base = lb; base < hi; base += 32) {
    const int i = base + lane_id();
    const uint32_t wv = i < hi ? rid[i] : bit;
    const double dv = i < hi ? rd[i] : 0.0;
    const unsigned bal = __ballot_sync(0xffffffffu, !(wv & bit));
    if (bal) {
      const int f = __ffs(bal) - 1;
      *dsel = __shfl_sync(0xffffffffu, dv, f);
      *isel = __shfl_sync(0xffffffffu, wv, f);
      return base + f;
    }
  }
  return -1;
}

// warm L2 with the neighbour row of a node we will probably expand next
SB_DEV void prefetch_row(const RouteArgs& a, uint32_t node) {
  const int lane = lane_id();
  const char* p = reinterpret_cast<const char*>(a.nbr_ids + (int64_t)node * a.g);
  if (lane * 128 < a.g * 4) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + lane * 128));
  // and its count (loaded beside the ids: the slower of the two sets the pace)
  if (lane == 31) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.nbr_counts + node));
}

// float ordering key usable with integer atomics (monotone in the float value)
SB_HD uint32_t fkey(float f) {
#ifdef __CUDA_ARCH__
  uint32_t b = __float_as_uint(f);
#else
  uint32_t b;
  memcpy(&b, &f, 4);
#endif
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
SB_HD float fkey_inv(uint32_t k) {
  uint32_t b = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
#ifdef __CUDA_ARCH__
  return __uint_as_float(b);
#else
  float f;
  memcpy(&f, &b, 4);
  return f;
#endif
}

// 256 threads x ROUTE_MIN_CTAS CTAs per SM
#ifndef ROUTE_MIN_CTAS
#define ROUTE_MIN_CTAS 3
#endif
// entries of the sorted (d, id) list x[0..n) ordered before (d, id); ids compared without flags
SB_DEV int count_before(const double* xd, const uint32_t* xi, int n, double d, uint32_t id,
                        const IdOrder& ord) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (ord(xd[mid], xi[mid] & kIdMask, d, id)) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// count_before for a warp-uniform target: a 32-ary search, one ballot per level (n = 4096
// takes 3 levels instead of 12 dependent steps)
SB_DEV int warp_count_before(const double* xd, const uint32_t* xi, int n, double d, uint32_t id,
                             const IdOrder& ord) {
  const int lane = lane_id();
  int lo = 0, len = n;
  while (len > 32) {
    const int step = (len + 31) >> 5;
    const int idx = lo + lane * step;
    const bool p = idx < lo + len && ord(xd[idx], xi[idx] & kIdMask, d, id);
    const int c = __popc(__ballot_sync(0xffffffffu, p));
    if (c == 0) return lo;
    const int nlo = lo + (c - 1) * step + 1;
    const int end = c * step < len ? lo + c * step : lo + len;  // sample c is not before
    len = end - nlo;
    lo = nlo;
  }
  const bool p = lane < len && ord(xd[lo + lane], xi[lo + lane] & kIdMask, d, id);
  return lo + __popc(__ballot_sync(0xffffffffu, p));
}

// LAZY (K >= kLazyK): new candidates collect in a small sorted buffer B next to the result
// list R and are merged into R only when B fills, so the O(K) list shift is paid once per
// ~kLazyB candidates instead of once per expansion.  R ∪ B holds the walk's results; an entry
// whose rank in R ∪ B is >= K is evicted in the reference and can never return (ranks only
// grow), so it simply stays unselectable until the next merge drops it.  Selection takes the
// first unchecked entry of R ∪ B by rank; the admission tail is the union's K-th entry.
// warp_merge_topk into R: lists in global memory (large-K instance) move 8 chunks per round
// trip; the small-K instance keeps one code path (its hot loop must stay compact)
template <bool LAZY, class L>
SB_DEV int merge_into_r(const RouteArgs& a, double* rd, uint32_t* rid, int K, double* cd,
                        uint32_t* cid, int* cpos, int c, L lt, bool presorted = false) {
  if (LAZY && a.gr_d) return warp_merge_topk<L, 8>(rd, rid, K, cd, cid, cpos, c, kIdMask, lt, presorted);
  return warp_merge_topk<L, 1>(rd, rid, K, cd, cid, cpos, c, kIdMask, lt, presorted);
}

template <int MODE, bool LAZY>
__global__ void __launch_bounds__(256, MODE == kModeF64Deep ? 1 : LAZY ? 2 : ROUTE_MIN_CTAS)
route_kernel(RouteArgs a) {
  extern __shared__ __align__(16) char smem_raw[];
  const int lane = lane_id();
  const int wid = warp_id();
  const int nw = blockDim.x >> 5;
  const size_t wbytes = route_warp_smem_bytes_full(a.Kpad, a.Cpad, a.m, a.l, LAZY, LAZY && a.gr_d != nullptr,
                                                   MODE == kModeF64Deep ? a.ring_slots : 0);
  const int64_t slot = (int64_t)blockIdx.x * nw + wid;
  WarpSmem w = carve<LAZY>(smem_raw + wbytes * wid, a, slot);
  uint32_t* vis = a.visited + slot * a.vwords;
  uint32_t* vlog = a.vlog + slot * (int64_t)a.logcap;
  const int K = a.K;
  const int Cap = a.Cpad;
  const IdOrder ord{a.perm, (uint32_t)a.n};  // ties by original id in a relabeled layout

  for (;;) {
    int qi = 0;
    if (lane == 0) qi = atomicAdd(a.counter, 1);
    qi = __shfl_sync(0xffffffffu, qi, 0);
    if (qi >= a.q) break;

    // query -> shared memory; choose the distance path
    bool integral = true;
    float qlo = 3.4e38f, qhi = -3.4e38f;
    for (int t = lane; t < a.m; t += 32) {
      double v = a.qf[(int64_t)qi * a.m + t];
      w.qs[t] = v;
      w.qs32[t] = (float)v;
      integral = integral && v == rint(v) && fabs(v) < 16777216.0;
      qlo = fminf(qlo, (float)v);
      qhi = fmaxf(qhi, (float)v);
    }
    for (int t = a.m + lane; t < ((a.m + 31) & ~31); t += 32) w.qs[t] = 0.0;
    for (int t = lane; t < a.l; t += 32) {
      w.qas[t] = a.qa[(int64_t)qi * a.l + t];
      w.qms[t] = a.qm ? a.qm[(int64_t)qi * a.l + t] : 1.0;
    }
    for (int o = 16; o > 0; o >>= 1) {
      qlo = fminf(qlo, __shfl_xor_sync(0xffffffffu, qlo, o));
      qhi = fmaxf(qhi, __shfl_xor_sync(0xffffffffu, qhi, o));
    }
    integral = __all_sync(0xffffffffu, integral);
    double qn = 0.0;  // |q|, rounded up (the filtered fp64 path's bound)
    if (MODE == kModeF64Filt) {
      for (int t = lane; t < a.m; t += 32) qn += w.qs[t] * w.qs[t];
      qn = sqrt(warp_sum(qn)) * (1.0 + 1e-12);
    }
    bool f32 = false;
    int nq8 = 0;
    if ((MODE == kModeF32Lane || MODE == kModeF32Split) && integral) {
      double dmax = fmax((double)a.fhi - (double)qlo, (double)qhi - (double)a.flo);
      f32 = dmax * dmax * (double)a.m < 16777216.0;  // 2^24
    }
    if (MODE == kModeU8 && integral && qlo >= 0.f && qhi <= 255.f) {
      // u8 query over the fp32 copy (the byte array overlays it: every float is read
      // before this warp's bytes are written, see the __syncwarp)
      f32 = true;
      int acc = 0;
      uint32_t packed[4];
      const int nw = a.m >> 2;  // 32-bit words of bytes
      // lane handles words lane, lane + 32, lane + 64, lane + 96: 4 dims each (m <= 512)
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        const int wd = lane + 32 * it;
        uint32_t b = 0;
        if (wd < nw) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int x = (int)w.qs32[4 * wd + e];
            acc += x * x;
            b |= (uint32_t)x << (8 * e);
          }
        }
        packed[it] = b;
      }
      __syncwarp();
#pragma unroll
      for (int it = 0; it < 4; ++it)
        if (lane + 32 * it < nw) reinterpret_cast<uint32_t*>(w.qs32)[lane + 32 * it] = packed[it];
      nq8 = warp_sum(acc);
    }
    __syncwarp();

    int64_t evals = 0, p1_evals = 0, p1_exp = 0, hops = 0, scanned = 0;
    int logn = 0;
    int lb = 0;    // first position of R that may hold an unchecked entry
    int nbuf = 0;  // LAZY: entries in the insertion buffer B
    const int bcap = Cap < kLazyB ? Cap : kLazyB;
    // LAZY: merge B into R (drops whatever leaves the top K)
    // LAZY: R changes only when B (or an oversized batch) is merged into it, so the entries just
    // below the two rank bounds the walk uses (K: admission and phase-2 selection; P: phase-1
    // selection) are cached in shared memory: window h holds R[hi - 1 - j], j = 0..kLazyB
    // (-inf where R has no such entry).  With R in global memory this takes the admission tail
    // and the rank tests of every expansion off the memory round trips.
    auto refresh_windows = [&]() {
      if (!LAZY) return;
      __syncwarp();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int hi_h = h ? a.P : K;
        for (int j = lane; j <= kLazyB; j += 32) {
          const int idx = hi_h - 1 - j;
          w.wd[h * kLazyW + j] = idx >= 0 ? w.rd[idx] : -__longlong_as_double(0x7FF0000000000000ll);
          w.wi[h * kLazyW + j] = idx >= 0 ? (w.rid[idx] & kIdMask) : 0u;
        }
      }
      __syncwarp();
    };
    // entries of B within the first hi of R ∪ B (a prefix of B: B[j-1] before R[hi-j])
    auto b_in_top = [&](int h) {
      int jt = 0;
      for (int base = 0; base < nbuf; base += 32) {
        const int j = base + lane + 1;
        const bool p = j <= nbuf && ord(w.bd[j - 1], w.bid[j - 1] & kIdMask, w.wd[h * kLazyW + j - 1],
                                        w.wi[h * kLazyW + j - 1]);
        jt += __popc(__ballot_sync(0xffffffffu, p));
      }
      return jt;
    };
    auto flush_b = [&]() {
      if (nbuf > 0) {
        const int ins = merge_into_r<LAZY>(a, w.rd, w.rid, K, w.bd, w.bid, w.cpos, nbuf, ord, true);
        if (ins < lb) lb = ins;
        nbuf = 0;
        refresh_windows();
      }
    };
    // LAZY: admit the batch cd/cid[0..c) against the K-th entry of R ∪ B, then add it to B
    // (or, when it does not fit, flush B and merge the batch into R directly)
    auto lazy_merge = [&](int c) {
      // the union's K-th entry: j = number of B entries within the first K of R ∪ B
      // (B[j-1] before R[K-j] holds for a prefix of j = 1..nbuf: count it by ballots)
      const int jt = b_in_top(0);
      double td = w.wd[jt];       // R[K - 1 - jt]
      uint32_t ti = w.wi[jt];
      if (jt > 0 && ord(td, ti, w.bd[jt - 1], w.bid[jt - 1] & kIdMask)) {
        td = w.bd[jt - 1];
        ti = w.bid[jt - 1] & kIdMask;
      }
      int kept = 0;
      for (int base = 0; base < c; base += 32) {
        const int i = base + lane;
        double d = 0.0;
        uint32_t id = 0;
        bool ok = false;
        if (i < c) {
          d = w.cd[i];
          id = w.cid[i];
          ok = ord(d, id, td, ti);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        __syncwarp();
        if (ok) {
          const int pos = kept + __popc(bal & ((1u << lane) - 1u));
          w.cd[pos] = d;
          w.cid[pos] = id;
        }
        kept += __popc(bal);
        __syncwarp();
      }
      if (kept == 0) return;
      if (nbuf + kept > bcap) flush_b();
      if (kept > bcap) {
        const int ins = merge_into_r<LAZY>(a, w.rd, w.rid, K, w.cd, w.cid, w.cpos, kept, ord);
        if (ins < lb) lb = ins;
        refresh_windows();
        return;
      }
      // B <- B ∪ batch by ranks (distinct ids): B[j] goes to j + #{batch < B[j]}, batch entry
      // x to #{batch < x} + #{B < x}; kept + nbuf <= bcap <= 64 entries, two per lane at most
      double xd[4];
      uint32_t xw[4];
      int xp[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int t = lane + 32 * (h & 1);
        const bool fromb = h < 2;
        xp[h] = -1;
        if (t < (fromb ? nbuf : kept)) {
          xd[h] = fromb ? w.bd[t] : w.cd[t];
          xw[h] = fromb ? w.bid[t] : w.cid[t];
          const uint32_t id = xw[h] & kIdMask;
          int r = fromb ? t : count_before(w.bd, w.bid, nbuf, xd[h], id, ord);
          for (int i = 0; i < kept; ++i) r += ord(w.cd[i], w.cid[i], xd[h], id);
          xp[h] = r;
        }
      }
      __syncwarp();
#pragma unroll
      for (int h = 0; h < 4; ++h)
        if (xp[h] >= 0) {
          w.bd[xp[h]] = xd[h];
          w.bid[xp[h]] = xw[h];
        }
      const int tot = kept + nbuf;
      __syncwarp();
      nbuf = tot;
      __syncwarp();
    };
    // walk state: stage 0 = evaluating entries, 1 = phase 1, 2 = phase 2
    int stage = 0;
    int ent_pos = 0;
    const int64_t* ent = a.entries + (int64_t)qi * K;
    for (;;) {
      int c = 0;
      bool half = false;
      if (stage == 0) {
        // next chunk of entries: mark visited, evaluate (_kernels.py:535-540)
        c = K - ent_pos < Cap ? K - ent_pos : Cap;
        for (int t = lane; t < c; t += 32) {
          uint32_t v = (uint32_t)ent[ent_pos + t];
          if (a.inv) v = (uint32_t)__ldg(a.inv + v);  // original -> layout id
          atomicOr(vis + (v >> 5), 1u << (v & 31));
          if (ent_pos + t < a.logcap) vlog[ent_pos + t] = v >> 5;  // the log holds bitset words
          w.cid[t] = v;
        }
      } else {
        const bool p1 = stage == 1;
        const int hi = p1 ? a.P : K;
        const uint32_t bit = p1 ? kChkP : kChkR;
        int nxt;
        int sel;
        uint32_t node;
        if (LAZY) {
          // first unchecked of R (by position) and of B, each admitted only if its rank in
          // R ∪ B is below hi; the smaller of the two is the reference's selection
          // The first hi of R ∪ B are B[0, jt) and R[0, hi - jt) (jt from the cached window, no
          // access to R): the first unchecked entry of each, the smaller of the two.
          nxt = -1;
          const int jt = b_in_top(p1 ? 1 : 0);
          double dR = 0.0;
          uint32_t idR = 0u;
          int iR = first_unchecked_d(w.rd, w.rid, lb, hi - jt, bit, &dR, &idR);
          int jB = -1;
          for (int base = 0; base < jt && jB < 0; base += 32) {
            const int j = base + lane;
            const unsigned bal = __ballot_sync(0xffffffffu, j < jt && !(w.bid[j] & bit));
            if (bal) jB = base + __ffs(bal) - 1;
          }
          if (iR >= 0 && jB >= 0) {
            if (ord(w.bd[jB], w.bid[jB] & kIdMask, dR, idR & kIdMask)) iR = -1;
            else jB = -1;
          }
          if (iR < 0 && jB < 0) {
            if (!p1) break;
            stage = 2;  // phase 2 starts with all checked flags cleared (_kernels.py:587-588)
            lb = 0;
            for (int t = lane; t < K; t += 32) w.rid[t] &= ~kChkR;
            for (int t = lane; t < nbuf; t += 32) w.bid[t] &= ~kChkR;
            __syncwarp();
            continue;
          }
          sel = iR;
          node = iR >= 0 ? (idR & kIdMask) : (w.bid[jB] & kIdMask);
          __syncwarp();
          if (lane == 0) {
            if (iR >= 0) w.rid[iR] |= bit;
            else w.bid[jB] |= bit;
          }
          __syncwarp();
          if (iR >= 0) lb = iR + 1;
        } else {
          sel = first_unchecked(w.rid, lb, hi, bit, &nxt);
          if (sel < 0) {
            if (!p1) break;
            stage = 2;  // phase 2 starts with all checked flags cleared (_kernels.py:587-588)
            lb = 0;
            for (int t = lane; t < K; t += 32) w.rid[t] &= ~kChkR;
            __syncwarp();
            continue;
          }
          node = w.rid[sel] & kIdMask;
          if (nxt >= 0) prefetch_row(a, w.rid[nxt] & kIdMask);
          __syncwarp();
          if (lane == 0) w.rid[sel] |= bit;
          __syncwarp();
          lb = sel + 1;
        }
        if (p1) ++p1_exp; else ++hops;
        half = p1;
        // expand: count and id row load together; visited test-and-set of the first cnt
        const int32_t* nb = a.nbr_ids + (int64_t)node * a.g;
        const int deg = __ldg(a.nbr_counts + node);
        for (int base = 0; base < a.g; base += 128) {
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
              uint32_t b = 1u << (v[k] & 31);
              uint32_t old = atomicOr(vis + (v[k] >> 5), b);
              fresh[k] = !(old & b);
            }
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            unsigned bal = __ballot_sync(0xffffffffu, fresh[k]);
            if (fresh[k]) {
              int pos = c + __popc(bal & ((1u << lane) - 1u));
              w.cid[pos] = v[k];
              int lp = logn + pos;
              if (lp < a.logcap) vlog[lp] = v[k] >> 5;
            }
            c += __popc(bal);
          }
        }
        scanned += half ? (deg + 1) >> 1 : deg;
        logn += c;
        evals += c;
        if (half) p1_evals += c;
      }
      __syncwarp();
      // L2 prefetch of the batch's rows: for rows of more than 1 KB (one lane walks its row in
      // many dependent chunks: cfg 4, d = 960: 28.9 -> 24.0 ms per 1k queries) whatever the batch
      // size, else when the batch exceeds one row per lane (cfg 5, d = 100: prefetching every
      // batch was 4% slower)
      if (MODE != kModeF64Deep && (c > 32 || (a.m * 4 > 1024 && !(MODE == kModeU8 && f32))) && a.pf_rows) {
        // request every line of the batch's rows at once (L2), so the per-lane row loads
        // below wait for one memory latency instead of one per 128-byte chunk
        const int lines = MODE == kModeU8 && f32 ? (a.m + 127) >> 7 : (a.m * 4 + 127) >> 7;
        const char* fb = (MODE == kModeU8 && f32) ? reinterpret_cast<const char*>(a.F8)
                                                  : reinterpret_cast<const char*>(a.F);
        const int64_t rowb = (MODE == kModeU8 && f32) ? a.m : 4 * (int64_t)a.m;
        if (lines == 1) {  // one 128-byte line per row: no division
          for (int t = lane; t < c; t += 32)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(fb + (int64_t)w.cid[t] * rowb));
        } else if (a.pf_rows == 2 && (rowb & 15) == 0) {
          // one bulk prefetch per row: DRAM sees whole-row bursts instead of the lanes' single
          // 32-byte sectors (the random-sector rate, not bandwidth, bounded the long rows)
          for (int t = lane; t < c; t += 32)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(fb + (int64_t)w.cid[t] * rowb),
                         "r"((uint32_t)rowb));
        } else {
          for (int t = lane; t < c * lines; t += 32) {
            const int r = t / lines;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(fb + (int64_t)w.cid[r] * rowb + (t - r * lines) * 128));
          }
        }
      }
      if (c > 0)
        eval_rows<MODE>(a, w, c, f32, nq8,
                        stage == 0 ? __longlong_as_double(0x7FF0000000000000ll) : w.rd[K - 1], qn);
      if (stage == 0) {
        for (int t = lane; t < c; t += 32) {
          w.rd[ent_pos + t] = w.cd[t];
          w.rid[ent_pos + t] = w.cid[t];
        }
        ent_pos += c;
        if (ent_pos == K) {
          logn = K;
          evals = K;
          for (int t = K + lane; t < a.Kpad; t += 32) {
            w.rd[t] = __longlong_as_double(0x7FF0000000000000ll);
            w.rid[t] = 0xFFFFFFFFu;
          }
          __syncwarp();
          if (a.Kpad > 1) {
            if (LAZY && a.gr_d) warp_bitonic_did_batched(w.rd, w.rid, a.Kpad, ord);
            else warp_bitonic_did(w.rd, w.rid, a.Kpad, ord);
          }
          stage = a.use_coarse ? 1 : 2;
          lb = 0;
          refresh_windows();
        }
        __syncwarp();
      } else if (c > 0) {
        if (LAZY) {
          lazy_merge(c);
        } else {
          int ins;
          if (c <= 32 && kFastMerge) {
            // one candidate per lane: filter against the tail, then the shuffle-ranked merge
            const double wd = w.rd[K - 1];
            const uint32_t wi = w.rid[K - 1] & kIdMask;
            const bool have = lane < c;
            const double d = have ? w.cd[lane] : 0.0;
            const uint32_t id = have ? w.cid[lane] : 0u;
            const bool ok = have && ord(d, id, wd, wi);
            ins = warp_merge_lanes(w.rd, w.rid, K, ok, d, id, kIdMask, w.cpos, ord);
          } else {
            ins = merge_into_r<LAZY>(a, w.rd, w.rid, K, w.cd, w.cid, w.cpos, c, ord);
          }
          if (ins < lb) lb = ins;
        }
      }
    }
    if (LAZY) flush_b();
    // results
    for (int t = lane; t < K; t += 32) {
      const uint32_t id = w.rid[t] & kIdMask;
      a.out_ids[(int64_t)qi * K + t] = (int64_t)(a.perm ? (uint32_t)__ldg(a.perm + id) : id);
      a.out_dists[(int64_t)qi * K + t] = w.rd[t];
    }
    if (a.stats && lane == 0) {
      int64_t* st = a.stats + (int64_t)qi * 5;
      st[0] = evals;
      st[1] = p1_evals;
      st[2] = p1_exp;
      st[3] = hops;
      st[4] = scanned;
    }
    // clear the visited bits this query set
    if (logn <= a.logcap) {
      for (int t = lane; t < logn; t += 32) vis[vlog[t]] = 0u;
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

// The Floyd regime (the usual one: k <= n / 50 or n <= 10,000) with the hash table and the
// output in shared memory as int32 (n < 2^31): every probe and shuffle swap is a shared-memory
// access instead of a dependent global one.  One thread per query, kEpThreads per block.
constexpr int kEpThreads = 32;  // threads per block at most (fewer for large k)
__global__ void entry_points_smem_kernel(int64_t n, int K, uint64_t seed, int64_t qi0, int64_t q,
                                         int64_t* out, int tslots) {
  extern __shared__ int32_t ep_smem[];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= q) return;
  int32_t* table = ep_smem + (size_t)threadIdx.x * (tslots + K);
  int32_t* o = table + tslots;
  sbrng::Pcg64 g;
  sbrng::pcg_from_entropy2(&g, seed, (uint64_t)(qi0 + i));
  sbrng::choice_floyd<int32_t>(&g, n, K, o, table, (uint64_t)tslots - 1);
  int64_t* dst = out + i * K;
  for (int t = 0; t < K; ++t) dst[t] = o[t];
}

// Warp per query (Floyd regime, n < 2^31, n != K): every 32-bit draw of the query's choice()
// comes from a PCG64 output reachable by jump-ahead — draw d is half d % 2 of output d / 2,
// and with no Lemire rejection draw d serves bounded(n - K + d) (Floyd, d < K) or
// bounded(2K - 1 - d) (the shuffle's i = 2K - 1 - d) — so the lanes compute all 2K - 1 bounded values in
// parallel; lane 0 then resolves Floyd's collisions and applies the swaps in shared memory.
// A rejection (probability ~ range / 2^32 per draw) shifts the stream: the warp then redoes
// the query sequentially.  Same ids as NumPy (tests/test_gpu_kernels.py).
__global__ void entry_points_warp_kernel(int64_t n, int K, uint64_t seed, int64_t qi0, int64_t q,
                                         int64_t* out, int tslots) {
  extern __shared__ int32_t ew_smem[];
  const int lane = lane_id();
  const int wpb = blockDim.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * wpb + warp_id();
  if (i >= q) return;
  int32_t* table = ew_smem + (size_t)warp_id() * (tslots + 2 * K);
  int32_t* vals = table + tslots;  // [0, K): Floyd values, then the ids; [K, 2K - 1): swap partners
  sbrng::Pcg64 g;
  sbrng::pcg_from_entropy2(&g, seed, (uint64_t)(qi0 + i));
  for (int t = lane; t < tslots; t += 32) table[t] = -1;
  const int D = 2 * K - 1;
  sbrng::U128 m1, p1, m16, p16;
  sbrng::pcg_jump_params(g.inc, (uint64_t)(lane >> 1) + 1, &m1, &p1);
  sbrng::pcg_jump_params(g.inc, 16, &m16, &p16);
  sbrng::U128 stt = sbrng::add128(sbrng::mul128(m1, g.s), p1);
  bool reject = false;
  for (int d = lane; d < D; d += 32) {
    const uint64_t o = sbrng::pcg_output(stt);
    const uint32_t u = (lane & 1) ? (uint32_t)(o >> 32) : (uint32_t)o;
    const uint32_t range = d < K ? (uint32_t)(n - K + d) : (uint32_t)(2 * K - 1 - d);
    const uint32_t excl = range + 1u;
    const uint64_t mm = (uint64_t)u * excl;
    const uint32_t left = (uint32_t)mm;
    if (left < excl && left < (0xFFFFFFFFu - range) % excl) reject = true;
    vals[d] = (int32_t)(mm >> 32);
    stt = sbrng::add128(sbrng::mul128(m16, stt), p16);
  }
  reject = __any_sync(0xffffffffu, reject);
  __syncwarp();
  if (lane == 0) {
    if (reject) {
      sbrng::choice_floyd<int32_t>(&g, n, K, vals, table, (uint64_t)tslots - 1);
    } else {
      const uint64_t tmask = (uint64_t)tslots - 1;
      for (int t = 0; t < K; ++t) {  // Floyd: value v_j, or j itself when v_j was taken
        const int32_t v = vals[t], j = (int32_t)(n - K + t);
        uint64_t loc = (uint64_t)v & tmask;
        while (table[loc] != -1 && table[loc] != v) loc = (loc + 1) & tmask;
        if (table[loc] == -1) {
          table[loc] = v;
        } else {
          loc = (uint64_t)j & tmask;
          while (table[loc] != -1) loc = (loc + 1) & tmask;
          table[loc] = j;
          vals[t] = j;
        }
      }
      for (int t = K - 1; t > 0; --t) {  // the shuffle
        const int32_t jj = vals[K + (K - 1 - t)];
        const int32_t x = vals[t];
        vals[t] = vals[jj];
        vals[jj] = x;
      }
    }
  }
  __syncwarp();
  int64_t* dst = out + i * K;
  for (int t = lane; t < K; t += 32) dst[t] = vals[t];
}

int launch_entry_points(int64_t n, int K, uint64_t seed, int64_t qi0, int64_t q, int64_t* out,
                        int64_t* scratch, uint64_t scratch_slots, cudaStream_t st) {
  {
    const uint64_t ts = sbrng::choice_table_size(n, K);
    const size_t per = sizeof(int32_t) * (size_t)(ts + 2 * K);
    int wpb = 8;
    while (wpb > 1 && per * wpb > (size_t)100 * 1024) wpb >>= 1;
    static const bool warp_on = [] { const char* e = getenv("SB_EP_WARP"); return !(e && e[0] == '0'); }();
    if (warp_on && !sbrng::choice_uses_tail_shuffle(n, K) && n < (int64_t)0x7FFFFFFF && n != K && K >= 1 &&
        per * wpb <= (size_t)100 * 1024) {
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(entry_points_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        attr = true;
      }
      const int64_t gb = (q + wpb - 1) / wpb;
      if (gb > 0)
        entry_points_warp_kernel<<<(unsigned)gb, 32 * wpb, per * wpb, st>>>(n, K, seed, qi0, q, out, (int)ts);
      return (int)cudaGetLastError();
    }
  }
  const uint64_t ts = sbrng::choice_table_size(n, K);
  const size_t per = sizeof(int32_t) * (size_t)(ts + K);
  int tpb = kEpThreads;
  while (tpb > 1 && per * tpb > (size_t)200 * 1024) tpb >>= 1;
  if (!sbrng::choice_uses_tail_shuffle(n, K) && n < (int64_t)0x7FFFFFFF && per * tpb <= (size_t)200 * 1024) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(entry_points_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = true;
    }
    const int64_t gb = (q + tpb - 1) / tpb;
    if (gb > 0)
      entry_points_smem_kernel<<<(unsigned)gb, tpb, per * tpb, st>>>(n, K, seed, qi0, q, out, (int)ts);
    return (int)cudaGetLastError();
  }
  int bs = 128;
  int64_t gb = (q + bs - 1) / bs;
  if (gb > 0) entry_points_kernel<<<(unsigned)gb, bs, 0, st>>>(n, K, seed, qi0, q, out, scratch,
                                                               scratch_slots);
  return (int)cudaGetLastError();
}

// the insertion-buffer instance for large K (SB_ROUTE_LAZY=0 disables it, for A/B runs)
static bool route_lazy(const RouteArgs& a) {
  static const bool on = [] {
    const char* e = getenv("SB_ROUTE_LAZY");
    return !(e && e[0] == '0');
  }();
  static const int kmin = [] {
    const char* e = getenv("SB_ROUTE_LAZYK");
    return e ? atoi(e) : kLazyK;
  }();
  return on && a.Kpad >= kmin && a.Cpad >= 16;
}

bool route_large_k(const RouteArgs& a) { return route_lazy(a); }

static int route_mode(const RouteArgs& a);
size_t route_smem_per_warp(const RouteArgs& a) {
  const bool lz = route_lazy(a);
  return route_warp_smem_bytes_full(a.Kpad, a.Cpad, a.m, a.l, lz, lz && a.gr_d != nullptr,
                                    route_mode(a) == kModeF64Deep ? a.ring_slots : 0);
}

template <int MODE>
static int launch_route_t(const RouteArgs& a, int warps_per_cta, int ctas, size_t smem,
                          cudaStream_t st) {
  auto kern = route_lazy(a) ? route_kernel<MODE, true> : route_kernel<MODE, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  kern<<<ctas, warps_per_cta * 32, smem, st>>>(a);
  return (int)cudaGetLastError();
}

static int route_mode(const RouteArgs& a) {
  if (a.F8) return kModeU8;
  if (a.f32_ok) return a.lpr == 1 ? kModeF32Lane : kModeF32Split;
  if ((a.m & 3) == 0) return a.flt_lpr > 0 ? kModeF64Filt : a.deep ? kModeF64Deep : kModeF64x4;
  return kModeGeneric;
}

int route_path(const RouteArgs& a) { return route_mode(a); }

int launch_route(const RouteArgs& a, int warps_per_cta, int ctas, cudaStream_t st) {
  size_t smem = route_smem_per_warp(a) * warps_per_cta;
  switch (route_mode(a)) {
    case kModeF64x4: return launch_route_t<kModeF64x4>(a, warps_per_cta, ctas, smem, st);
    case kModeF64Filt: return launch_route_t<kModeF64Filt>(a, warps_per_cta, ctas, smem, st);
    case kModeF64Deep: return launch_route_t<kModeF64Deep>(a, warps_per_cta, ctas, smem, st);
    case kModeF32Lane: return launch_route_t<kModeF32Lane>(a, warps_per_cta, ctas, smem, st);
    case kModeF32Split: return launch_route_t<kModeF32Split>(a, warps_per_cta, ctas, smem, st);
    case kModeU8: return launch_route_t<kModeU8>(a, warps_per_cta, ctas, smem, st);
    default: return launch_route_t<kModeGeneric>(a, warps_per_cta, ctas, smem, st);
  }
}

template <int MODE>
static int route_occupancy_t(int warps_per_cta, size_t smem, int* ctas_per_sm, bool lazy) {
  auto kern = lazy ? route_kernel<MODE, true> : route_kernel<MODE, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, kern, warps_per_cta * 32,
                                                            smem);
}

int route_occupancy(const RouteArgs& a, int warps_per_cta, size_t smem, int* ctas_per_sm) {
  const bool lz = route_lazy(a);
  switch (route_mode(a)) {
    case kModeF64x4: return route_occupancy_t<kModeF64x4>(warps_per_cta, smem, ctas_per_sm, lz);
    case kModeF64Filt: return route_occupancy_t<kModeF64Filt>(warps_per_cta, smem, ctas_per_sm, lz);
    case kModeF64Deep: return route_occupancy_t<kModeF64Deep>(warps_per_cta, smem, ctas_per_sm, lz);
    case kModeF32Lane: return route_occupancy_t<kModeF32Lane>(warps_per_cta, smem, ctas_per_sm, lz);
    case kModeF32Split: return route_occupancy_t<kModeF32Split>(warps_per_cta, smem, ctas_per_sm, lz);
    case kModeU8: return route_occupancy_t<kModeU8>(warps_per_cta, smem, ctas_per_sm, lz);
    default: return route_occupancy_t<kModeGeneric>(warps_per_cta, smem, ctas_per_sm, lz);
  }
}

// u8 copy of integer features in [0, 255] plus exact squared norms (warp per node)
__global__ void pack_u8_kernel(const float* F, int64_t n, int m, uint8_t* F8, int32_t* nx) {
  const int64_t v = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id();
  if (v >= n) return;
  int acc = 0;
  for (int t = lane_id(); t < m; t += 32) {
    const int x = (int)F[v * m + t];
    F8[v * m + t] = (uint8_t)x;
    acc += x * x;
  }
  acc = warp_sum(acc);
  if (lane_id() == 0) nx[v] = acc;
}

// {|x|^2, attrs[0..2]} per node for the u8 routing rows (l <= 3)
__global__ void pack_meta16_kernel(const int32_t* nx, const int32_t* A, int64_t n, int l, uint4* out) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  uint4 r;
  r.x = (uint32_t)nx[v];
  r.y = l > 0 ? (uint32_t)A[v * l] : 0u;
  r.z = l > 1 ? (uint32_t)A[v * l + 1] : 0u;
  r.w = l > 2 ? (uint32_t)A[v * l + 2] : 0u;
  out[v] = r;
}

int launch_pack_meta16(const int32_t* nx, const int32_t* A, int64_t n, int l, void* out, cudaStream_t st) {
  pack_meta16_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(nx, A, n, l, reinterpret_cast<uint4*>(out));
  return (int)cudaGetLastError();
}

int launch_pack_u8(const float* F, int64_t n, int m, uint8_t* F8, int32_t* nx, cudaStream_t st) {
  pack_u8_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(F, n, m, F8, nx);
  return (int)cudaGetLastError();
}

// ---- routing layout: a locality order of the nodes ------------------------------------
// Nodes are renumbered along a Z-order (Morton) curve over kOrdDims random +-1 projections of
// their features, so the nodes one query visits sit close together: their visited bits share
// words and sectors, and their rows, attributes and adjacency share DRAM pages.  Any order is
// exact (ties still compare original ids); this one only changes speed.
#ifndef ROUTE_ORD_RADEMACHER
#define ROUTE_ORD_RADEMACHER 1  // +-1 projections (measured equal to Gaussian ones)
#endif
#ifndef ROUTE_ORD_DIMS
#define ROUTE_ORD_DIMS 6
#endif
#ifndef ROUTE_ORD_BITS
#define ROUTE_ORD_BITS 10
#endif
constexpr int kOrdDims = ROUTE_ORD_DIMS, kOrdBits = ROUTE_ORD_BITS;

SB_DEV uint32_t ord_hash(uint32_t x) {
  x *= 0x9E3779B1u;
  x ^= x >> 15;
  x *= 0x85EBCA77u;
  x ^= x >> 13;
  x *= 0xC2B2AE3Du;
  x ^= x >> 16;
  return x;
}

// fixed Gaussian projection matrix entry (Box-Muller from two hashed uniforms)
SB_DEV float proj_coef(int d, int p) {
#if ROUTE_ORD_RADEMACHER
  return (ord_hash((uint32_t)(d * kOrdDims + p)) & 1u) ? 1.f : -1.f;
#else
  const uint32_t k = (uint32_t)(d * kOrdDims + p);
  const float u1 = ((ord_hash(2 * k) >> 8) + 1) * (1.0f / 16777217.0f);
  const float u2 = (ord_hash(2 * k + 1) >> 8) * (1.0f / 16777216.0f);
  return sqrtf(-2.0f * __logf(u1)) * __cosf(6.28318531f * u2);
#endif
}

__global__ void order_project_kernel(const float* F, int64_t n, int m, float* proj, unsigned* lohi) {
  const int64_t v = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id();
  if (v >= n) return;
  float acc[kOrdDims];
#pragma unroll
  for (int p = 0; p < kOrdDims; ++p) acc[p] = 0.f;
  for (int t = lane_id(); t < m; t += 32) {
    const float x = F[v * m + t];
#pragma unroll
    for (int p = 0; p < kOrdDims; ++p) acc[p] += proj_coef(t, p) * x;
  }
#pragma unroll
  for (int p = 0; p < kOrdDims; ++p) {
    const float r = warp_sum(acc[p]);
    if (lane_id() == 0) {
      proj[v * kOrdDims + p] = r;
      atomicMin(lohi + 2 * p, fkey(r));
      atomicMax(lohi + 2 * p + 1, fkey(r));
    }
  }
}

__global__ void order_morton_kernel(const float* proj, int64_t n, const unsigned* lohi,
                                    uint64_t* key, int32_t* val) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  uint32_t qv[kOrdDims];
#pragma unroll
  for (int p = 0; p < kOrdDims; ++p) {
    const float lo = fkey_inv(lohi[2 * p]), hi = fkey_inv(lohi[2 * p + 1]);
    const float t = hi > lo ? (proj[v * kOrdDims + p] - lo) / (hi - lo) : 0.f;
    qv[p] = (uint32_t)fminf(fmaxf(t * (float)((1 << kOrdBits) - 1), 0.f), (float)((1 << kOrdBits) - 1));
  }
  uint64_t k = 0;
  for (int b = kOrdBits - 1; b >= 0; --b)
#pragma unroll
    for (int p = 0; p < kOrdDims; ++p) k = (k << 1) | ((qv[p] >> b) & 1u);
  key[v] = k;
  val[v] = (int32_t)v;
}

__global__ void order_inverse_kernel(const int32_t* perm, int64_t n, int32_t* inv) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) inv[perm[i]] = (int32_t)i;
}

size_t route_order_scratch_bytes(int64_t n) {
  size_t temp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)n);
  return (size_t)n * (2 * sizeof(uint64_t) + sizeof(int32_t) + sizeof(float) * kOrdDims) + temp +
         64 * sizeof(unsigned) + 1024;
}

int launch_route_order(const float* F, int64_t n, int m, int32_t* perm, int32_t* inv,
                       void* scratch, size_t scratch_bytes, cudaStream_t st) {
  char* p = static_cast<char*>(scratch);
  auto take = [&](size_t b) { char* r = p; p += (b + 255) & ~(size_t)255; return r; };
  uint64_t* k_in = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * n));
  uint64_t* k_out = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * n));
  int32_t* v_in = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * n));
  float* proj = reinterpret_cast<float*>(take(sizeof(float) * n * kOrdDims));
  unsigned* lohi = reinterpret_cast<unsigned*>(take(64 * sizeof(unsigned)));
  size_t temp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp, k_in, k_out, v_in, perm, (int)n);
  void* d_temp = take(temp);
  if ((size_t)(p - static_cast<char*>(scratch)) > scratch_bytes) return (int)cudaErrorInvalidValue;
  unsigned init[2 * kOrdDims];
  for (int i = 0; i < kOrdDims; ++i) { init[2 * i] = 0xFFFFFFFFu; init[2 * i + 1] = 0u; }
  cudaMemcpyAsync(lohi, init, sizeof(init), cudaMemcpyHostToDevice, st);
  order_project_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(F, n, m, proj, lohi);
  order_morton_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(proj, n, lohi, k_in, v_in);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(d_temp, temp, k_in, k_out, v_in, perm, (int)n,
                                                  0, kOrdDims * kOrdBits, st);
  if (e != cudaSuccess) return (int)e;
  order_inverse_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(perm, n, inv);
  // the init copy above must complete before `init` leaves scope
  cudaStreamSynchronize(st);
  return (int)cudaGetLastError();
}

__global__ void permute_rows_f32_kernel(const float* src, int64_t n, int m, const int32_t* perm,
                                        float* dst) {
  const int64_t v = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id();
  if (v >= n) return;
  const float* s = src + (int64_t)perm[v] * m;
  for (int t = lane_id(); t < m; t += 32) dst[v * m + t] = s[t];
}

__global__ void permute_rows_i32_kernel(const int32_t* src, int64_t n, int w, const int32_t* perm,
                                        int32_t* dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * w) return;
  const int64_t v = i / w;
  dst[i] = src[(int64_t)perm[v] * w + (i - v * w)];
}

__global__ void relabel_adjacency_kernel(const int32_t* ids, const int32_t* counts, int64_t n, int g,
                                         const int32_t* perm, const int32_t* inv, int32_t* ids_r,
                                         int32_t* counts_r) {
  const int64_t v = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id();
  if (v >= n) return;
  const int64_t o = perm[v];
  const int c = counts[o];
  for (int t = lane_id(); t < g; t += 32) ids_r[v * g + t] = t < c ? inv[ids[o * g + t]] : 0;
  if (lane_id() == 0) counts_r[v] = c;
}

int launch_permute_rows_f32(const float* src, int64_t n, int m, const int32_t* perm, float* dst,
                            cudaStream_t st) {
  permute_rows_f32_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(src, n, m, perm, dst);
  return (int)cudaGetLastError();
}
int launch_permute_rows_i32(const int32_t* src, int64_t n, int w, const int32_t* perm,
                            int32_t* dst, cudaStream_t st) {
  permute_rows_i32_kernel<<<(unsigned)((n * w + 255) / 256), 256, 0, st>>>(src, n, w, perm, dst);
  return (int)cudaGetLastError();
}
int launch_relabel_adjacency(const int32_t* ids, const int32_t* counts, int64_t n, int g,
                             const int32_t* perm, const int32_t* inv, int32_t* ids_r,
                             int32_t* counts_r, cudaStream_t st) {
  relabel_adjacency_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(ids, counts, n, g, perm, inv,
                                                                   ids_r, counts_r);
  return (int)cudaGetLastError();
}

// index property: are all features integral, and their range (monotone keys in out[1..2])
__global__ void feature_scan_kernel(const float* F, int64_t count, unsigned* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool bad = false;
  float lo = 3.4e38f, hi = -3.4e38f;
  for (; i < count; i += stride) {
    float v = F[i];
    bad = bad || v != rintf(v) || !isfinite(v);
    lo = fminf(lo, v);
    hi = fmaxf(hi, v);
  }
  if (__any_sync(0xffffffffu, bad) && lane_id() == 0) atomicOr(out, 1u);
  for (int o = 16; o > 0; o >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if (lane_id() == 0) {
    atomicMin(out + 1, fkey(lo));
    atomicMax(out + 2, fkey(hi));
  }
}

int launch_feature_scan(const float* F, int64_t count, unsigned* out3, cudaStream_t st) {
  unsigned init[3] = {0u, 0xFFFFFFFFu, 0u};
  cudaMemcpyAsync(out3, init, sizeof(init), cudaMemcpyHostToDevice, st);
  cudaStreamSynchronize(st);
  feature_scan_kernel<<<1184, 256, 0, st>>>(F, count, out3);
  return (int)cudaGetLastError();
}

float feature_key_to_float(unsigned k) { return fkey_inv(k); }

}  // namespace sb

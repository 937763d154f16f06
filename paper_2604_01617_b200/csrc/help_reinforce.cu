// help_reinforce.cu — reinforce_pass (_kernels.py:398-409 with _try_insert_edge 306-395),
// exact, with the sequential part confined to the rows that can overflow.
//
// Facts used (all follow from the reference's sequential semantics):
//  (1) With O = { j : |row_j ∪ rev_j| > gamma } computed on the post-prune graph
//      (rev_j = { s : j in row_s }), rows outside O never become full: every insertion into
//      row j comes from a source s with j in row_s at time s, which is either a static edge
//      (s in rev_j) or a mirror that is already present (a duplicate).
//  (2) Rows outside O never lose entries, so an event s -> j with j outside O is a duplicate
//      iff s was in row_j after pruning; those events commute and are applied in parallel.
//  (3) Every node that can ever sit in an O row j belongs to U_j = row_j ∪ rev_j, so the
//      redundancy relation attrs_equal(p, k) and cos(p - j, k - j) > sigma used by the
//      re-prune can be precomputed for all pairs of U_j, in parallel, as a bit matrix.
//  (4) in_deg[p] at event time (s, .) = post-prune in_deg + insertions of p so far - drops
//      so far; insertions of p happen only while processing row p, so for p outside O they
//      are all "static" and complete once p < s.
// The sequential simulation then visits only sources in O and sources with an O-row entry,
// in ascending order, and performs exact try_insert semantics on O rows with bit lookups.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "sb_internal.h"

namespace sb {

SB_DEV int row_find_key(const int32_t* ids, const float* dists, int cnt, uint64_t key) {
  int lo = 0, hi = cnt;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    uint64_t k = row_key(dists[mid], (uint32_t)ids[mid]);
    if (k < key) lo = mid + 1; else hi = mid;
  }
  return (lo < cnt && row_key(dists[lo], (uint32_t)ids[lo]) == key) ? lo : -1;
}

// K1: mutual flags per edge, non-mutual counts per target
__global__ void rf_mutual_kernel(RfArgs a) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= a.n * a.g) return;
  int64_t s = e / a.g;
  int t = (int)(e % a.g);
  if (t >= a.counts[s]) return;
  int32_t j = a.ids[e];
  uint64_t key = row_key(a.dists[e], (uint32_t)s);
  bool mut = row_find_key(a.ids + (int64_t)j * a.g, a.dists + (int64_t)j * a.g, a.counts[j], key) >= 0;
  a.mutual[e] = mut ? 1 : 0;
  if (!mut) atomicAdd(reinterpret_cast<unsigned long long*>(a.rev_extra + j), 1ull);
}

// K2: overflow flags
__global__ void rf_over_kernel(RfArgs a, int64_t* oflag64) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.n) return;
  bool o = (int64_t)a.counts[j] + a.rev_extra[j] > a.g;
  a.is_o[j] = o ? 1 : 0;
  oflag64[j] = o ? 1 : 0;
}

// K3: O index, U sizes, static insertion counts, relevance; count static non-O inserts per
// target (for the parallel apply) and reverse sources per O target (for U lists)
__global__ void rf_classify_kernel(RfArgs a, const int64_t* oscan) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.n) return;
  const bool so = a.is_o[s];
  if (so) {
    int64_t o = oscan[s];
    a.o_idx[s] = (int32_t)o;
    a.o_nodes[o] = (int32_t)s;
    a.u_size[o] = a.counts[s] + a.rev_extra[s];
  } else {
    a.o_idx[s] = -1;
  }
  int stat = 0;
  bool rel = so;
  for (int t = 0; t < a.counts[s]; ++t) {
    int64_t e = s * a.g + t;
    int32_t j = a.ids[e];
    bool jo = a.is_o[j];
    if (jo) rel = true;
    if (!a.mutual[e]) {
      if (jo) {
        atomicAdd(reinterpret_cast<unsigned long long*>(a.orev_cnt + j), 1ull);
      } else if (!so) {
        ++stat;
        atomicAdd(reinterpret_cast<unsigned long long*>(a.apply_cnt + j), 1ull);
      }
    }
  }
  a.static_ins[s] = so ? 0 : stat;
  a.relevant[s] = rel ? 1 : 0;
}

// K3b: per-edge O index of the target (post-prune rows; static for rows outside O)
__global__ void rf_eo_kernel(RfArgs a) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= a.n * a.g) return;
  const int64_t s = e / a.g;
  const int t = (int)(e - s * a.g);
  a.eo[e] = t < a.counts[s] ? a.o_idx[a.ids[e]] : -2;
}

// K4a: scatter reverse sources of O targets into their U lists (after the row's own ids)
__global__ void rf_u_scatter_kernel(RfArgs a) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= a.n * a.g) return;
  int64_t s = e / a.g;
  int t = (int)(e % a.g);
  if (t >= a.counts[s] || a.mutual[e]) return;
  int32_t j = a.ids[e];
  if (!a.is_o[j]) return;
  int o = a.o_idx[j];
  unsigned long long p = atomicAdd(reinterpret_cast<unsigned long long*>(a.u_cur + o), 1ull);
  a.u_list[a.u_off[o] + a.counts[j] + (int64_t)p] = (int32_t)s;
}

// K4b: U list = row ids + reverse sources, sorted by id (warp per O row, in smem)
__global__ void rf_u_sort_kernel(RfArgs a, int upad_max) {
  extern __shared__ __align__(16) char smem_raw[];
  const int wpb = blockDim.x >> 5;
  uint64_t* buf = reinterpret_cast<uint64_t*>(smem_raw) + (size_t)warp_id() * upad_max;
  int64_t o = (int64_t)blockIdx.x * wpb + warp_id();
  if (o >= a.no) return;
  const int32_t j = a.o_nodes[o];
  const int u = (int)a.u_size[o];
  const int up = next_pow2(u);
  int32_t* U = a.u_list + a.u_off[o];
  for (int t = lane_id(); t < up; t += 32) {
    uint64_t v = kKeyInf;
    if (t < a.counts[j]) v = (uint64_t)(uint32_t)a.ids[(int64_t)j * a.g + t];
    else if (t < u) v = (uint64_t)(uint32_t)U[t];
    buf[t] = v;
  }
  __syncwarp();
  warp_bitonic_u64(buf, up);
  for (int t = lane_id(); t < u; t += 32) U[t] = (int32_t)buf[t];
}

// K5: symmetric redundancy bits over U_j: attrs_equal(p, k) && cos(p - j, k - j) > sigma,
// fp64 in the reference's operation order (_kernels.py:235-253).  CTA per O row,
// 4 x 4 tiles over the lower triangle, features staged in dimension chunks.
constexpr int kRfThreads = 256;
__global__ void __launch_bounds__(kRfThreads) rf_bits_kernel(RfArgs a, int dc_max, int upad4) {
  extern __shared__ __align__(16) char smem_raw[];
  const int64_t o = blockIdx.x;
  const int32_t j = a.o_nodes[o];
  const int u = (int)a.u_size[o];
  const int32_t* U = a.u_list + a.u_off[o];
  const int W = (u + 31) >> 5;
  uint32_t* bits = a.r_bits + a.r_off[o];
  // the float tile goes first: its float4 reads need 16-byte alignment
  char* p = smem_raw;
  float* xr = reinterpret_cast<float*>(p); p += sizeof(float) * (size_t)dc_max * upad4;
  double* xs = reinterpret_cast<double*>(p); p += sizeof(double) * dc_max;
  double* nrm = reinterpret_cast<double*>(p);
  const int tid = threadIdx.x;
  const int up4 = (u + 3) & ~3;
  // dimensions [d0, d0 + dc) of every member of U_j, transposed, by 4-byte asynchronous copies
  // (a warp per member, lanes along the dimensions)
  auto stage_rows = [&](int d0, int dc) {
    const int lane_ = tid & 31, nwarp = blockDim.x >> 5;
    for (int t = tid >> 5; t < u; t += nwarp) {
      const float* src = a.F + (int64_t)U[t] * a.m + d0;
      for (int dd = lane_; dd < dc; dd += 32)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(xr + dd * up4 + t)),
                     "l"(src + dd)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  };
  // norms |p - j|^2 in ascending dimension order; thread tid owns entries tid + 256 r
  constexpr int kMaxPer = 16;  // u <= 4096
  double myn[kMaxPer];
#pragma unroll
  for (int r = 0; r < kMaxPer; ++r) myn[r] = 0.0;
  for (int d0 = 0; d0 < a.m; d0 += dc_max) {
    const int dc = a.m - d0 < dc_max ? a.m - d0 : dc_max;
    __syncthreads();
    for (int t = tid; t < dc; t += blockDim.x) xs[t] = (double)__ldg(a.F + (int64_t)j * a.m + d0 + t);
    stage_rows(d0, dc);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kMaxPer; ++r) {
      const int t = tid + r * kRfThreads;
      if (t < u)
        for (int dd = 0; dd < dc; ++dd) {
          double dp = dsub((double)xr[dd * up4 + t], xs[dd]);
          myn[r] = dadd(myn[r], dmul(dp, dp));
        }
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kMaxPer; ++r)
    if (tid + r * kRfThreads < u) nrm[tid + r * kRfThreads] = myn[r];
  __syncthreads();
  const int nb = (u + 3) / 4;
  const int ntiles = nb * (nb + 1) / 2;
  for (int pass = 0; pass * kRfThreads < ntiles; ++pass) {
    const int ti = pass * kRfThreads + tid;
    const bool have = ti < ntiles;
    int tb = 0, ub = 0;
    if (have) {
      tb = (int)((sqrt(8.0 * ti + 1.0) - 1.0) * 0.5);
      while ((tb + 1) * (tb + 2) / 2 <= ti) ++tb;
      while (tb * (tb + 1) / 2 > ti) --tb;
      ub = ti - tb * (tb + 1) / 2;
    }
    double acc[4][4];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
    for (int d0 = 0; d0 < a.m; d0 += dc_max) {
      const int dc = a.m - d0 < dc_max ? a.m - d0 : dc_max;
      __syncthreads();
      for (int t = tid; t < dc; t += blockDim.x) xs[t] = (double)__ldg(a.F + (int64_t)j * a.m + d0 + t);
      stage_rows(d0, dc);
      __syncthreads();
      if (have) {
        for (int dd = 0; dd < dc; ++dd) {
          const float* row = xr + (size_t)dd * up4;
          const double c = xs[dd];
          float4 tv = *reinterpret_cast<const float4*>(row + tb * 4);
          float4 uv = *reinterpret_cast<const float4*>(row + ub * 4);
          const double dt[4] = {dsub((double)tv.x, c), dsub((double)tv.y, c), dsub((double)tv.z, c), dsub((double)tv.w, c)};
          const double du[4] = {dsub((double)uv.x, c), dsub((double)uv.y, c), dsub((double)uv.z, c), dsub((double)uv.w, c)};
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) acc[x][y] = dadd(acc[x][y], dmul(dt[x], du[y]));
        }
      }
    }
    if (have) {
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) {
          const int t = tb * 4 + x, v = ub * 4 + y;
          if (t >= u || v >= t) continue;
          const int32_t pt = U[t], pv = U[v];
          bool eq = true;
          for (int z = 0; z < a.l; ++z) eq = eq && __ldg(a.A + (int64_t)pt * a.l + z) == __ldg(a.A + (int64_t)pv * a.l + z);
          if (!eq) continue;
          const double np2 = nrm[t], nk2 = nrm[v];
          // cos of (p_t - j, p_v - j); the reference evaluates it with p = later entry,
          // k = earlier kept entry; dot and the norm product are symmetric in (p, k)
          double c = (np2 == 0.0 || nk2 == 0.0) ? 1.0 : __ddiv_rn(acc[x][y], sqrt(dmul(np2, nk2)));
          if (c > a.sigma) {
            atomicOr(bits + (int64_t)t * W + (v >> 5), 1u << (v & 31));
            atomicOr(bits + (int64_t)v * W + (t >> 5), 1u << (t & 31));
          }
        }
    }
  }
}

// ---------------------------------------------------------------------------------------
// K7: the sequential simulation, run by one warp.  Events are processed strictly in the
// reference's order; the warp parallelises the work inside each event (row scans, the
// merged-list build, in-degree and redundancy-row loads) and keeps the greedy re-prune
// sequential over list positions.
constexpr unsigned kFull = 0xFFFFFFFFu;

SB_DEV int u_index(const RfArgs& a, int o, int32_t node) {
  const int32_t* U = a.u_list + a.u_off[o];
  int lo = 0, hi = (int)a.u_size[o];
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (U[mid] < node) lo = mid + 1; else hi = mid;
  }
  return (lo < (int)a.u_size[o] && U[lo] == node) ? lo : -1;
}

// u_index by 32-way search over U (sorted, u entries): each round probes 32 positions
SB_DEV int warp_u_index(const int32_t* U, int u, int32_t node) {
  const int lane = lane_id();
  int lo = 0, hi = u;  // first position with U[pos] >= node lies in [lo, hi]
  while (hi - lo > 32) {
    const int step = (hi - lo + 31) >> 5;
    const int pk = lo + lane * step;
    const bool less = pk < hi && U[pk] < node;
    const int c = __popc(__ballot_sync(kFull, less));
    if (c == 0) {
      hi = lo;
    } else {
      const int last = lo + (c - 1) * step;
      const int nxt = lo + c * step;
      lo = last + 1;
      if (c < 32 && nxt < hi) hi = nxt;
    }
  }
  const bool less = lo + lane < hi && U[lo + lane] < node;
  lo += __popc(__ballot_sync(kFull, less));
  const bool found = lo < u && U[lo] == node;
  return found ? lo : -1;
}

SB_DEV int32_t indeg_read(const RfArgs& a, int32_t p, int64_t s) {
  int32_t v = __ldcg(a.in_deg + p);  // other groups update in-degrees with L2 atomics
  if (p < s && !a.is_o[p]) v += a.static_ins[p];
  return v;
}

// shared scratch of the simulating warp: the merged list of a full row (g + 1 entries) with
// in-degrees, keep flags and redundancy rows
struct SimSmem {
  int32_t* mi;
  float* md;
  int32_t* mu;
  int32_t* midg;
  uint8_t* mkeep;
  uint32_t* Rs;
};

__host__ __device__ size_t rf_simulate_smem(int g, int wmax) {
  const size_t b = (size_t)(g + 1) * (4 * 4 + 1) + 16 + sizeof(uint32_t) * (size_t)(g + 1) * wmax + 64;
  return (b + 15) & ~(size_t)15;  // per-warp slices stay 16-byte aligned
}

// exact _try_insert_edge on O row j (_kernels.py:306-395); returns 1 if inserted
// cycle counters of the simulation (build with -DSB_RF_PROF=1, print with env SB_RF_PROF)
#ifndef SB_RF_PROF
#define SB_RF_PROF 0
#endif
constexpr bool kRfProf = SB_RF_PROF != 0;
__device__ unsigned long long g_rf_prof[16];

// cu_hint: cand's position in U_j when known (precomputed for static edges, recorded for
// mirrors), or -1 to search U_j
SB_DEV int warp_try_insert(RfArgs& a, const SimSmem& S, int32_t j, int o, int32_t cand,
                           float d, int64_t s, int& err, int cu_hint = -1) {
  const int lane = lane_id();
  const long long t_start = clock64();
  const int g = a.g;
  int32_t* ri = a.ids + (int64_t)j * g;
  float* rd = a.dists + (int64_t)j * g;
  int32_t* ru = a.u_pos + (int64_t)o * g;
  // one round of independent loads: the row's count, U bounds and the whole row (rows are
  // allocated gamma wide, so entries past the count are read and masked)
  const int cj = a.counts[j];
  const int64_t uoff = a.u_off[o];
  const int usz = (int)a.u_size[o];
  int32_t vi[8], vu[8];
  float vd[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int t = lane + 32 * k;
    if (t < g) { vi[k] = ri[t]; vd[k] = rd[t]; vu[k] = ru[t]; }
  }
  // already present?  and the insertion position: entries ordered before (d, cand)
  bool dup = false;
  int pos = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int t = lane + 32 * k;
    bool lt = false;
    if (t < cj) {
      dup = dup || vi[k] == cand;
      lt = vd[k] < d || (vd[k] == d && vi[k] < cand);
    }
    if (32 * k < g) pos += __popc(__ballot_sync(kFull, lt));
  }
  if (__any_sync(kFull, dup)) {
    if (kRfProf && lane == 0) { atomicAdd(&g_rf_prof[4], (unsigned long long)(clock64() - t_start)); atomicAdd(&g_rf_prof[5], 1ull); }
    return 0;
  }
  const long long t_dup = clock64();
  const int cu = cu_hint >= 0 ? cu_hint : warp_u_index(a.u_list + uoff, usz, cand);
  const long long t_uidx = clock64();
  if (cu < 0) {
    err = 1;
    return 0;
  }
  if (cj < g) {
    // shift [pos, cj) one slot right from the registers, then place
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int t = lane + 32 * k;
      if (t >= pos && t < cj) { ri[t + 1] = vi[k]; rd[t + 1] = vd[k]; ru[t + 1] = vu[k]; }
    }
    if (lane == 0) {
      ri[pos] = cand; rd[pos] = d; ru[pos] = cu;
      a.counts[j] = cj + 1;
      atomicAdd(a.in_deg + cand, 1);
      if (kRfProf) { atomicAdd(&g_rf_prof[0], (unsigned long long)(clock64() - t_start)); atomicAdd(&g_rf_prof[1], 1ull); }
    }
    __syncwarp();
    return 1;
  }
  // full: merged list of g + 1, re-prune under the safeguard
  const int total = cj + 1;
  const int W = ((int)a.u_size[o] + 31) >> 5;
  const uint32_t* R = a.r_bits + a.r_off[o];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int t = lane + 32 * k;
    if (t < cj) {
      const int dst = t < pos ? t : t + 1;
      S.mi[dst] = vi[k]; S.md[dst] = vd[k]; S.mu[dst] = vu[k];
    }
  }
  if (lane == 0) { S.mi[pos] = cand; S.md[pos] = d; S.mu[pos] = cu; }
  __syncwarp();
  // in-degrees: an entry's in-degree changes in this call only when that entry is dropped,
  // after which it is never read again, so loading them all up front is exact
  // the merged entries' redundancy rows: 4-byte asynchronous copies, all in flight at once (a
  // load -> store loop paid one L2 round trip per 32 words: ~50 k cycles per re-prune, half of
  // the replay's time on a single-attribute-value index)
  for (int e = lane; e < total * W; e += 32) {
    const int t = e / W, w = e - t * W;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(S.Rs + e)),
                 "l"(R + (int64_t)S.mu[t] * W + w)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  {  // in-degrees of up to 9 entries per lane (g + 1 <= 257): every load of a level issued before any is used
    int32_t pp[9], vv[9];
    bool st[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const int t = lane + 32 * k;
      pp[k] = t < total ? S.mi[t] : cand;
      vv[k] = pp[k] == cand ? 0 : __ldcg(a.in_deg + pp[k]);  // other groups update in-degrees with L2 atomics
      st[k] = pp[k] != cand && pp[k] < s && !a.is_o[pp[k]];
    }
#pragma unroll
    for (int k = 0; k < 9; ++k)
      if (st[k]) vv[k] += a.static_ins[pp[k]];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const int t = lane + 32 * k;
      if (t < total) {
        S.midg[t] = vv[k];
        S.mkeep[t] = 1;
      }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncwarp();
  const long long t_loads = clock64();
  int kept = 1;
  if (total <= 128) {
    // Greedy re-prune in list order.  The kept-U mask lives in registers (word lane + 32 k);
    // nothing on the loop-carried path but the row test, one vote and the mask update: the
    // safeguard condition of every entry comes from ballots taken up front, the keep flags
    // collect in register masks (no shared-memory store in the loop, so the rows and U
    // positions of the next entries load ahead of the votes).
    unsigned cond[4], keep[4] = {1u, 0u, 0u, 0u};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int k = lane + 32 * c;
      const bool cd = k < total && (S.mi[k] == cand || S.midg[k] >= 2);
      cond[c] = __ballot_sync(kFull, cd);
    }
    uint32_t km[4] = {0u, 0u, 0u, 0u};
    {
      const int u0 = S.mu[0];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if ((u0 >> 5) == lane + 32 * k) km[k] |= 1u << (u0 & 31);
    }
#pragma unroll
    for (int c0 = 0; c0 < 4; ++c0) {  // (static indices: the masks stay in registers)
      const int tend = total - 32 * c0 < 32 ? total - 32 * c0 : 32;
#pragma unroll 4
      for (int tb = c0 == 0 ? 1 : 0; tb < tend; ++tb) {
        const int t = 32 * c0 + tb;
        const int ut = S.mu[t];
        const uint32_t* rr = S.Rs + t * W;
        // (all of the row's words loaded at once, no short circuit: a chain of conditional
        // loads cost four shared-memory latencies per entry)
        uint32_t hit = 0u;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int w = lane + 32 * k;
          const uint32_t rv = w < W ? rr[w] : 0u;
          hit |= rv & km[k];
        }
        const bool red = __any_sync(kFull, hit != 0u);
        if (!(red && ((cond[c0] >> tb) & 1u))) {
          keep[c0] |= 1u << tb;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if ((ut >> 5) == lane + 32 * k) km[k] |= 1u << (ut & 31);
        }
      }
    }
    kept = __popc(keep[0]) + __popc(keep[1]) + __popc(keep[2]) + __popc(keep[3]);
    __syncwarp();
    for (int t = lane; t < total; t += 32) S.mkeep[t] = (uint8_t)((keep[t >> 5] >> (t & 31)) & 1u);
  } else {
  // greedy re-prune in list order; the kept-U mask lives in registers (word lane + 32 k)
  uint32_t km[4] = {0u, 0u, 0u, 0u};
  {
    const int u0 = S.mu[0];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if ((u0 >> 5) == lane + 32 * k) km[k] |= 1u << (u0 & 31);
  }
  for (int t = 1; t < total; ++t) {
    const uint32_t* rr = S.Rs + t * W;
    bool hit = false;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int w = lane + 32 * k;
      if (w < W) hit = hit || (rr[w] & km[k]) != 0u;
    }
    const bool red = __any_sync(kFull, hit);
    const int32_t p = S.mi[t];
    if (red && (p == cand || S.midg[t] >= 2)) {
      if (lane == 0) S.mkeep[t] = 0;
    } else {
      ++kept;
      const int ut = S.mu[t];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if ((ut >> 5) == lane + 32 * k) km[k] |= 1u << (ut & 31);
    }
  }
  }
  __syncwarp();
  const long long t_greedy = clock64();
  if (kept > g && lane == 0) {
    for (int t = total - 1; t >= 0; --t) {
      if (!S.mkeep[t]) continue;
      const int32_t p = S.mi[t];
      if (p == cand) { S.mkeep[t] = 0; break; }
      if (S.midg[t] >= 2) { S.mkeep[t] = 0; break; }
    }
  }
  __syncwarp();
  // every dropped entry other than the candidate loses one in-degree
  for (int t = lane; t < total; t += 32)
    if (!S.mkeep[t] && S.mi[t] != cand) atomicSub(a.in_deg + S.mi[t], 1);
  int w0 = 0, inserted = 0;
  for (int t0 = 0; t0 < total; t0 += 32) {
    const int t = t0 + lane;
    const bool k = t < total && S.mkeep[t];
    const unsigned b = __ballot_sync(kFull, k);
    if (k) {
      const int dst = w0 + __popc(b & ((1u << lane) - 1u));
      ri[dst] = S.mi[t]; rd[dst] = S.md[t]; ru[dst] = S.mu[t];
      if (S.mi[t] == cand) inserted = 1;
    }
    w0 += __popc(b);
  }
  inserted = __any_sync(kFull, inserted) ? 1 : 0;
  if (lane == 0) {
    a.counts[j] = w0;
    if (inserted) atomicAdd(a.in_deg + cand, 1);
    if (kRfProf) {
      const long long t_end = clock64();
      atomicAdd(&g_rf_prof[2], (unsigned long long)(t_end - t_start)); atomicAdd(&g_rf_prof[3], 1ull);
      atomicAdd(&g_rf_prof[8], (unsigned long long)(t_dup - t_start));
      atomicAdd(&g_rf_prof[9], (unsigned long long)(t_uidx - t_dup));
      atomicAdd(&g_rf_prof[10], (unsigned long long)(t_loads - t_uidx));
      atomicAdd(&g_rf_prof[11], (unsigned long long)(t_greedy - t_loads));
      atomicAdd(&g_rf_prof[12], (unsigned long long)(t_end - t_greedy));
      atomicAdd(&g_rf_prof[13], (unsigned long long)W);
    }
  }
  __syncwarp();
  return inserted;
}

__global__ void rf_init_upos_kernel(RfArgs a) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= a.no * a.g) return;
  int64_t o = e / a.g;
  int t = (int)(e % a.g);
  int32_t j = a.o_nodes[o];
  if (t >= a.counts[j]) return;
  a.u_pos[e] = u_index(a, (int)o, a.ids[(int64_t)j * a.g + t]);
}

// One warp per group of O-row components (components do not interact: see rf_groups in
// capi.cu), each walking the sources its group's rows see, in ascending order, through the
// group's source bitmap.
__global__ void rf_simulate_kernel(RfArgs a) {
  extern __shared__ __align__(16) char smem_raw[];
  const int lane = lane_id();
  const int g = a.g;
  const int grp = blockIdx.x * (blockDim.x >> 5) + warp_id();
  if (grp >= a.ngroups) return;
  uint32_t* bm = a.grp_bits + (size_t)grp * a.bm_words;
  SimSmem S;
  {
    char* p = smem_raw + (size_t)warp_id() * rf_simulate_smem(g, a.sim_wmax);
    S.Rs = reinterpret_cast<uint32_t*>(p); p += sizeof(uint32_t) * (size_t)(g + 1) * a.sim_wmax;
    S.mi = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * (g + 1);
    S.mu = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * (g + 1);
    S.midg = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * (g + 1);
    S.md = reinterpret_cast<float*>(p); p += sizeof(float) * (g + 1);
    S.mkeep = reinterpret_cast<uint8_t*>(p);
  }
  uint64_t* dyn = a.dyn + (size_t)grp * a.dyn_cap;
  int32_t* dyn_cu = a.dyn_cu + (size_t)grp * a.dyn_cap;
  auto in_grp = [&](int o) { return a.grp_of_o[o] == grp; };
  int err = 0;
  const long long t_kernel = clock64();
  auto dyn_insert = [&](int q, int64_t s) {
    const uint64_t kd = dyn[q];
    const int32_t jd = (int32_t)key_id(kd);
    warp_try_insert(a, S, jd, a.o_idx[jd], (int32_t)s, key_dist(kd), s, err, dyn_cu[q]);
  };
  // Per source: count, O index, the row (gamma wide, masked by the count), the head of its
  // recorded mirrors and the targets' O indices.  Rows outside O never change during the
  // simulation and their targets' O indices are precomputed (eo), so all of it is one round
  // of independent loads, issued for the NEXT relevant source of the chunk before the current
  // one is processed.  O rows may change, so an O source is always (re)loaded when reached.
  struct Src {
    int64_t s;
    int cs, osrc;
    int64_t rh;
    int32_t vi[8];
    float vd[8];
    int oj[8];
    int cu[8];  // s's position in U_j of each static O-target edge (rows outside O)
  };
  auto load_src = [&](int64_t s, Src& D) {
    D.s = s;
    D.cs = a.counts[s];
    D.osrc = a.o_idx[s];
    D.rh = *reinterpret_cast<const volatile int64_t*>(a.rec_head + s);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int t = lane + 32 * k;
      if (t < g) {
        D.vi[k] = a.ids[s * g + t];
        D.vd[k] = a.dists[s * g + t];
        D.oj[k] = a.eo[s * g + t];
        D.cu[k] = a.ecu[s * g + t];
      } else {
        D.oj[k] = -2;
        D.cu[k] = -1;
      }
    }
  };
  const volatile uint32_t* vbm = bm;
  for (int64_t wi = 0; wi < a.bm_words; ++wi) {
    const int64_t base = wi * 32;
    unsigned bal = vbm[wi];
    Src nxt;
    nxt.s = -1;
    while (bal) {
      const int64_t s = base + __ffs(bal) - 1;
      bal &= bal - 1u;
      if (kRfProf && lane == 0) atomicAdd(&g_rf_prof[7], 1ull);
      Src D;
      if (nxt.s == s && nxt.osrc < 0) {
        D = nxt;  // valid: only O sources record mirrors, and they discard the prefetch
      } else {
        load_src(s, D);
      }
      nxt.s = -1;
      if (bal) load_src(base + __ffs(bal) - 1, nxt);
      const int cs = D.cs;
      const int osrc = D.osrc;
      const int64_t rh = D.rh;
      int32_t vi[8];
      float vd[8];
      int oj[8];
      int cuh[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        vi[k] = D.vi[k];
        vd[k] = D.vd[k];
        // an O row's entries are live: its U positions come from u_pos, its events search
        cuh[k] = osrc >= 0 ? ((lane + 32 * k) < cs ? a.u_pos[(int64_t)osrc * g + lane + 32 * k] : -1)
                           : D.cu[k];
        // an O row's entries may have changed since eo was computed: look their O index up
        oj[k] = osrc >= 0 ? ((lane + 32 * k) < cs ? a.o_idx[vi[k]] : -2) : D.oj[k];
      }
      if (osrc >= 0) {
        // mirrors into rows that cannot overflow: record each one not already present
        // (record order = row order); then the O-target events in row order
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (32 * k >= cs) break;
          const bool rec = oj[k] == -1 &&
                           row_find_key(a.ids + (int64_t)vi[k] * g, a.dists + (int64_t)vi[k] * g,
                                        a.counts[vi[k]], row_key(vd[k], (uint32_t)s)) < 0;
          const unsigned rb = __ballot_sync(kFull, rec);
          int64_t rbase = 0;
          if (lane == 0 && rb) rbase = (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(a.rec_count),
                                                          (unsigned long long)__popc(rb));
          rbase = __shfl_sync(kFull, rbase, 0);
          if (rec) {
            const int64_t r = rbase + __popc(rb & ((1u << lane) - 1u));
            if (r < a.rec_cap) {
              const int32_t j = vi[k];
              a.rec_tgt[r] = j;
              a.rec_key[r] = row_key(vd[k], (uint32_t)s);
              a.rec_cu[r] = cuh[k];  // j's position in U_s: the hint of the later event
              // lock-free push: other groups read j's list concurrently (and skip this record)
              unsigned long long* head = reinterpret_cast<unsigned long long*>(a.rec_head + j);
              unsigned long long old = *reinterpret_cast<volatile unsigned long long*>(head);
              for (;;) {
                a.rec_next[r] = (int64_t)old;
                __threadfence();
                const unsigned long long prev = atomicCAS(head, old, (unsigned long long)r);
                if (prev == old) break;
                old = prev;
              }
              if (j > s) atomicOr(bm + (j >> 5), 1u << (j & 31));
            } else {
              err = 2;
            }
          }
          const int64_t room = a.rec_cap - rbase;
          const int64_t ok = (int64_t)__popc(rb) < room ? (int64_t)__popc(rb) : (room > 0 ? room : 0);
          if (lane == 0 && ok) atomicAdd(a.in_deg + s, (int32_t)ok);
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (32 * k >= cs) break;
          unsigned ob = __ballot_sync(kFull, oj[k] >= 0);
          while (ob) {
            const int src = __ffs(ob) - 1;
            ob &= ob - 1u;
            warp_try_insert(a, S, __shfl_sync(kFull, vi[k], src), __shfl_sync(kFull, oj[k], src),
                            (int32_t)s, __shfl_sync(kFull, vd[k], src), s, err);
          }
        }
        // recorded mirrors may have made later sources of this word relevant
        __syncwarp();
        bal = vbm[wi] & (s - base == 31 ? 0u : (0xFFFFFFFFu << (s - base + 1)));
        nxt.s = -1;
      } else {
        // O-target events of a non-O row in key order: static entries j in O, plus entries
        // mirrored in by O sources processed earlier (linked list, sorted here)
        int nd = 0;
        if (lane == 0) {
          // records published by other groups' warps: read past L1 (a line cached before
          // the record was written would hand back stale words; the writer's fence orders
          // the record before its list link)
          const volatile int64_t* vnext = a.rec_next;
          const volatile uint64_t* vkey = a.rec_key;
          const volatile int32_t* vcu = a.rec_cu;
          for (int64_t r = rh; r >= 0; r = vnext[r]) {
            const uint64_t rk = vkey[r];
            if (!in_grp(a.o_idx[key_id(rk)])) continue;  // another group's mirror
            if (nd < a.dyn_cap) {
              uint64_t kk = row_key(key_dist(rk), key_id(rk));
              const int cr = vcu[r];
              int pos = nd;
              while (pos > 0 && dyn[pos - 1] > kk) {
                dyn[pos] = dyn[pos - 1];
                dyn_cu[pos] = dyn_cu[pos - 1];
                --pos;
              }
              dyn[pos] = kk;
              dyn_cu[pos] = cr;
              ++nd;
            } else {
              err = 3;
            }
          }
        }
        nd = __shfl_sync(kFull, nd, 0);
        __syncwarp();
        int q = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (32 * k >= cs) break;
          unsigned ob = __ballot_sync(kFull, oj[k] >= 0 && in_grp(oj[k]));
          while (ob) {
            const int src = __ffs(ob) - 1;
            ob &= ob - 1u;
            const int32_t jj = __shfl_sync(kFull, vi[k], src);
            const float dd = __shfl_sync(kFull, vd[k], src);
            const int oo = __shfl_sync(kFull, oj[k], src);
            const int ch = __shfl_sync(kFull, cuh[k], src);
            const uint64_t ks = row_key(dd, (uint32_t)jj);
            while (q < nd && dyn[q] < ks) dyn_insert(q++, s);
            warp_try_insert(a, S, jj, oo, (int32_t)s, dd, s, err, ch);
          }
        }
        while (q < nd) dyn_insert(q++, s);
      }
    }
  }
  err = __reduce_max_sync(kFull, err);
  if (lane == 0) {
    if (err) atomicMax(reinterpret_cast<unsigned long long*>(a.result + 1), (unsigned long long)err);
    if (kRfProf) g_rf_prof[6] = clock64() - t_kernel;
  }
}

// K8: per non-O target, merge static (non-O sources, non-mutual) + recorded insertions
__global__ void rf_apply_scatter_kernel(RfArgs a) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= a.n * a.g) return;
  int64_t s = e / a.g;
  int t = (int)(e % a.g);
  if (t >= a.counts[s] || a.is_o[s] || a.mutual[e]) return;
  int32_t j = a.ids[e];
  if (a.is_o[j]) return;
  unsigned long long p = atomicAdd(reinterpret_cast<unsigned long long*>(a.apply_cur + j), 1ull);
  a.apply_seg[a.apply_off[j] + (int64_t)p] = row_key(a.dists[e], (uint32_t)s);
}

__global__ void rf_apply_rec_kernel(RfArgs a, int64_t nrec) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrec) return;
  int32_t j = a.rec_tgt[r];
  unsigned long long p = atomicAdd(reinterpret_cast<unsigned long long*>(a.apply_cur + j), 1ull);
  a.apply_seg[a.apply_off[j] + (int64_t)p] = a.rec_key[r];
}

__global__ void rf_apply_count_rec_kernel(RfArgs a, int64_t nrec) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrec) return;
  atomicAdd(reinterpret_cast<unsigned long long*>(a.apply_cnt + a.rec_tgt[r]), 1ull);
}

// per-group source bitmaps: a non-O source is relevant to the groups of its O-target rows, an O
// source to its own row's group (rf_simulate_kernel walks these)
__global__ void rf_group_bits_kernel(RfArgs a) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= a.n * a.g) return;
  const int64_t s = e / a.g;
  const int t = (int)(e - s * a.g);
  const int os = a.o_idx[s];
  if (os >= 0) {
    if (t == 0) atomicOr(a.grp_bits + (size_t)a.grp_of_o[os] * a.bm_words + (s >> 5), 1u << (s & 31));
    return;
  }
  const int o = a.eo[e];  // -1 target outside O, -2 past the count
  if (o >= 0) atomicOr(a.grp_bits + (size_t)a.grp_of_o[o] * a.bm_words + (s >> 5), 1u << (s & 31));
}

int rf_launch_group_bits(RfArgs& a, cudaStream_t st) {
  cudaMemsetAsync(a.grp_bits, 0, sizeof(uint32_t) * (size_t)a.ngroups * a.bm_words, st);
  rf_group_bits_kernel<<<(unsigned)((a.n * a.g + 255) / 256), 256, 0, st>>>(a);
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
static inline unsigned nblk(int64_t x, int b) { return (unsigned)((x + b - 1) / b); }

int rf_launch_stage1(RfArgs& a, int64_t* oflag, int64_t* oscan, int64_t* scan_tmp, cudaStream_t st) {
  cudaMemsetAsync(a.rev_extra, 0, sizeof(int64_t) * a.n, st);
  rf_mutual_kernel<<<nblk(a.n * a.g, 256), 256, 0, st>>>(a);
  rf_over_kernel<<<nblk(a.n, 256), 256, 0, st>>>(a, oflag);
  exclusive_scan(oflag, oscan, a.n, scan_tmp, st);
  return (int)cudaGetLastError();
}

int rf_launch_stage2(RfArgs& a, const int64_t* oscan, cudaStream_t st) {
  cudaMemsetAsync(a.orev_cnt, 0, sizeof(int64_t) * a.n, st);
  cudaMemsetAsync(a.apply_cnt, 0, sizeof(int64_t) * a.n, st);
  rf_classify_kernel<<<nblk(a.n, 256), 256, 0, st>>>(a, oscan);
  rf_eo_kernel<<<nblk(a.n * a.g, 256), 256, 0, st>>>(a);
  return (int)cudaGetLastError();
}

// K6b: for every edge s -> j with j in O: s's position in U_j (static for rows outside O)
__global__ void rf_ecu_kernel(RfArgs a) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= a.n * a.g) return;
  const int o = a.eo[e];
  a.ecu[e] = o >= 0 ? u_index(a, o, (int32_t)(e / a.g)) : -1;
}

int rf_launch_stage3(RfArgs& a, int upad_max, int dc_max, int upad4_max, size_t bits_smem,
                     cudaStream_t st) {
  cudaMemsetAsync(a.u_cur, 0, sizeof(int64_t) * a.no, st);
  rf_u_scatter_kernel<<<nblk(a.n * a.g, 256), 256, 0, st>>>(a);
  int wpb = 4;
  size_t smem = (size_t)wpb * upad_max * sizeof(uint64_t);
  cudaFuncSetAttribute(rf_u_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  rf_u_sort_kernel<<<nblk(a.no, wpb), wpb * 32, smem, st>>>(a, upad_max);
  cudaFuncSetAttribute(rf_bits_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bits_smem);
  rf_bits_kernel<<<(unsigned)a.no, kRfThreads, bits_smem, st>>>(a, dc_max, upad4_max);
  rf_init_upos_kernel<<<nblk(a.no * a.g, 256), 256, 0, st>>>(a);
  rf_ecu_kernel<<<nblk(a.n * a.g, 256), 256, 0, st>>>(a);
  return (int)cudaGetLastError();
}

int rf_launch_simulate(RfArgs& a, cudaStream_t st) {
  const size_t smem = rf_simulate_smem(a.g, a.sim_wmax);
  const int kSimWarps = smem * 4 <= 200 * 1024 ? 4 : 1;
  cudaError_t e = cudaFuncSetAttribute(rf_simulate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(smem * kSimWarps));
  if (e != cudaSuccess) return (int)e;
  static const bool prof = kRfProf && getenv("SB_RF_PROF") != nullptr;
  if (prof) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_rf_prof, z, sizeof(z));
  }
  rf_simulate_kernel<<<(unsigned)((a.ngroups + kSimWarps - 1) / kSimWarps), 32 * kSimWarps,
                       smem * kSimWarps, st>>>(a);
  if (prof) {
    unsigned long long z[16];
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(z, g_rf_prof, sizeof(z));
    fprintf(stderr, "rf_sim full-row phases (cycles): dup test %llu | U index %llu | loads %llu | greedy %llu | write back %llu | sum W %llu\n",
            z[8], z[9], z[10], z[11], z[12], z[13]);
    fprintf(stderr, "rf_sim cycles: total %llu | nonfull %llu x%llu | full %llu x%llu | dup %llu x%llu | sources %llu\n",
            z[6], z[0], z[1], z[2], z[3], z[4], z[5], z[7]);
  }
  return (int)cudaGetLastError();
}

int rf_launch_apply(RfArgs& a, int64_t nrec, int64_t* scan_tmp, cudaStream_t st) {
  if (nrec > 0) rf_apply_count_rec_kernel<<<nblk(nrec, 256), 256, 0, st>>>(a, nrec);
  exclusive_scan(a.apply_cnt, a.apply_off, a.n, scan_tmp, st);
  cudaMemsetAsync(a.apply_cur, 0, sizeof(int64_t) * a.n, st);
  rf_apply_scatter_kernel<<<nblk(a.n * a.g, 256), 256, 0, st>>>(a);
  if (nrec > 0) rf_apply_rec_kernel<<<nblk(nrec, 256), 256, 0, st>>>(a, nrec);
  return (int)cudaGetLastError();
}

}  // namespace sb

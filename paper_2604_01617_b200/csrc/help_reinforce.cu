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
  // norms |p - j|^2 in ascending dimension order; thread tid owns entries tid + 256 r
  constexpr int kMaxPer = 16;  // u <= 4096
  double myn[kMaxPer];
#pragma unroll
  for (int r = 0; r < kMaxPer; ++r) myn[r] = 0.0;
  for (int d0 = 0; d0 < a.m; d0 += dc_max) {
    const int dc = a.m - d0 < dc_max ? a.m - d0 : dc_max;
    __syncthreads();
    for (int t = tid; t < dc; t += blockDim.x) xs[t] = (double)__ldg(a.F + (int64_t)j * a.m + d0 + t);
    for (int e = tid; e < u * dc; e += blockDim.x) {
      int t = e / dc, dd = e % dc;
      xr[dd * up4 + t] = __ldg(a.F + (int64_t)U[t] * a.m + d0 + dd);
    }
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
      for (int e = tid; e < u * dc; e += blockDim.x) {
        int t = e / dc, dd = e % dc;
        xr[dd * up4 + t] = __ldg(a.F + (int64_t)U[t] * a.m + d0 + dd);
      }
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
// K7: the sequential simulation (one thread)
struct Sim {
  RfArgs a;
  int err;
};

SB_DEV int u_index(const RfArgs& a, int o, int32_t node) {
  const int32_t* U = a.u_list + a.u_off[o];
  int lo = 0, hi = (int)a.u_size[o];
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (U[mid] < node) lo = mid + 1; else hi = mid;
  }
  return (lo < (int)a.u_size[o] && U[lo] == node) ? lo : -1;
}

SB_DEV int32_t indeg_read(const RfArgs& a, int32_t p, int64_t s) {
  int32_t v = a.in_deg[p];
  if (p < s && !a.is_o[p]) v += a.static_ins[p];
  return v;
}

// exact _try_insert_edge on O row j (_kernels.py:306-395); returns 1 if inserted
SB_DEV int sim_try_insert(RfArgs& a, int32_t j, int32_t cand, float d, int64_t s, int* err) {
  const int g = a.g;
  const int o = a.o_idx[j];
  int32_t* ri = a.ids + (int64_t)j * g;
  float* rd = a.dists + (int64_t)j * g;
  int32_t* ru = a.u_pos + (int64_t)o * g;
  const int cj = a.counts[j];
  for (int t = 0; t < cj; ++t)
    if (ri[t] == cand) return 0;
  const int cu = u_index(a, o, cand);
  if (cu < 0) { *err = 1; return 0; }
  if (cj < g) {
    int pos = cj;
    while (pos > 0 && (rd[pos - 1] > d || (rd[pos - 1] == d && ri[pos - 1] > cand))) {
      ri[pos] = ri[pos - 1]; rd[pos] = rd[pos - 1]; ru[pos] = ru[pos - 1];
      --pos;
    }
    ri[pos] = cand; rd[pos] = d; ru[pos] = cu;
    a.counts[j] = cj + 1;
    a.in_deg[cand] += 1;
    return 1;
  }
  // full: merged list of g + 1 in scratch, re-prune under the safeguard
  int32_t* ti = a.sim_ids;
  float* td = a.sim_d;
  int32_t* tu = a.sim_u;
  uint8_t* keep = a.sim_keep;
  int pos = cj;
  for (int t = 0; t < cj; ++t) { ti[t] = ri[t]; td[t] = rd[t]; tu[t] = ru[t]; }
  while (pos > 0 && (td[pos - 1] > d || (td[pos - 1] == d && ti[pos - 1] > cand))) {
    ti[pos] = ti[pos - 1]; td[pos] = td[pos - 1]; tu[pos] = tu[pos - 1];
    --pos;
  }
  ti[pos] = cand; td[pos] = d; tu[pos] = cu;
  const int total = cj + 1;
  const int W = ((int)a.u_size[o] + 31) >> 5;
  const uint32_t* R = a.r_bits + a.r_off[o];
  uint32_t* km = a.sim_mask;
  for (int w = 0; w < W; ++w) km[w] = 0u;
  for (int t = 0; t < total; ++t) keep[t] = 1;
  km[tu[0] >> 5] |= 1u << (tu[0] & 31);
  int kept = 1;
  for (int t = 1; t < total; ++t) {
    const int32_t p = ti[t];
    const uint32_t* rr = R + (int64_t)tu[t] * W;
    bool red = false;
    for (int w = 0; w < W && !red; ++w) red = (rr[w] & km[w]) != 0u;
    if (red && (p == cand || indeg_read(a, p, s) >= 2)) {
      keep[t] = 0;
      if (p != cand) a.in_deg[p] -= 1;
    } else {
      ++kept;
      km[tu[t] >> 5] |= 1u << (tu[t] & 31);
    }
  }
  if (kept > g) {
    for (int t = total - 1; t >= 0; --t) {
      if (!keep[t]) continue;
      const int32_t p = ti[t];
      if (p == cand) { keep[t] = 0; break; }
      if (indeg_read(a, p, s) >= 2) { keep[t] = 0; a.in_deg[p] -= 1; break; }
    }
  }
  int w = 0, inserted = 0;
  for (int t = 0; t < total; ++t) {
    if (!keep[t]) continue;
    ri[w] = ti[t]; rd[w] = td[t]; ru[w] = tu[t];
    if (ti[t] == cand) inserted = 1;
    ++w;
  }
  a.counts[j] = w;
  if (inserted) a.in_deg[cand] += 1;
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

__global__ void rf_simulate_kernel(RfArgs a) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  int err = 0;
  int64_t nrec = 0;
  const int g = a.g;
  for (int64_t s = 0; s < a.n; ++s) {
    if (!a.relevant[s]) continue;
    if (a.is_o[s]) {
      const int cs = a.counts[s];
      for (int t = 0; t < cs; ++t) {
        if (t >= a.counts[s]) break;
        const int32_t j = a.ids[s * g + t];
        const float d = a.dists[s * g + t];
        if (a.is_o[j]) {
          sim_try_insert(a, j, (int32_t)s, d, s, &err);
        } else {
          uint64_t key = row_key(d, (uint32_t)s);
          if (row_find_key(a.ids + (int64_t)j * g, a.dists + (int64_t)j * g, a.counts[j], key) < 0) {
            if (nrec >= a.rec_cap) { err = 2; continue; }
            a.rec_tgt[nrec] = j;
            a.rec_key[nrec] = key;
            a.rec_next[nrec] = a.rec_head[j];
            a.rec_head[j] = nrec;
            ++nrec;
            a.in_deg[s] += 1;
            if (j > s) a.relevant[j] = 1;
          }
        }
      }
    } else {
      // O-target events of a non-O row in key order: static entries j in O, plus entries
      // mirrored in by O sources processed earlier (linked list)
      int nd = 0;
      for (int64_t r = a.rec_head[s]; r >= 0; r = a.rec_next[r]) {
        if (nd < a.dyn_cap) {
          uint64_t k = row_key(key_dist(a.rec_key[r]), key_id(a.rec_key[r]));
          int pos = nd;
          while (pos > 0 && a.dyn[pos - 1] > k) { a.dyn[pos] = a.dyn[pos - 1]; --pos; }
          a.dyn[pos] = k;
          ++nd;
        } else {
          err = 3;
        }
      }
      const int cs = a.counts[s];
      int t = 0, q = 0;
      while (t < cs || q < nd) {
        uint64_t ks = kKeyInf;
        int32_t js = -1;
        while (t < cs) {
          js = a.ids[s * g + t];
          if (a.is_o[js]) { ks = row_key(a.dists[s * g + t], (uint32_t)js); break; }
          ++t;
        }
        uint64_t kd = q < nd ? a.dyn[q] : kKeyInf;
        if (ks == kKeyInf && kd == kKeyInf) break;
        if (ks <= kd) {
          sim_try_insert(a, js, (int32_t)s, key_dist(ks), s, &err);
          ++t;
        } else {
          sim_try_insert(a, (int32_t)key_id(kd), (int32_t)s, key_dist(kd), s, &err);
          ++q;
        }
      }
    }
  }
  a.result[0] = nrec;
  a.result[1] = err;
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
  return (int)cudaGetLastError();
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
  return (int)cudaGetLastError();
}

int rf_launch_simulate(RfArgs& a, cudaStream_t st) {
  rf_simulate_kernel<<<1, 1, 0, st>>>(a);
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

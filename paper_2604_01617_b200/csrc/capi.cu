// capi.cu — the C ABI (include/stable_b200.h): index handle, device buffers, orchestration
// of the kernels of one reference call, host<->device copies, error mapping.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/stable_b200.h"
#include "common.cuh"
#include "rng.cuh"
#include "sb_internal.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return SB_ECUDA;
}

#define CK(expr)                                              \
  do {                                                        \
    cudaError_t e_ = (expr);                                  \
    if (e_ != cudaSuccess) return cuda_fail(e_, #expr);       \
  } while (0)

// SB_SYNC_CHECK=1 (debugging): synchronize after every launch so a fault names its kernel
static bool sync_check() {
  static const bool on = [] { const char* e = getenv("SB_SYNC_CHECK"); return e && atoi(e) != 0; }();
  return on;
}
#define CKL(expr)                                                          \
  do {                                                                     \
    int r_ = (expr);                                                       \
    if (r_ == 0 && sync_check()) r_ = (int)cudaDeviceSynchronize();        \
    if (r_ != 0) return cuda_fail((cudaError_t)r_, #expr);                 \
  } while (0)

// grow-only device buffer
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t b) {
    if (b <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    size_t want = b < 256 ? 256 : b;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const { return reinterpret_cast<T*>(p); }
};

}  // namespace

// Large copies between the device and pageable host memory, through two page-locked bounce
// buffers: the DMA of one chunk overlaps the host-side copy of the other, and the host copy
// (with the first touch of fresh destination pages) is split over host threads.  A direct
// cudaMemcpy to or from pageable memory runs at a few GB/s (≈0.18 s for cfg 2's adjacency).
static cudaError_t transfer_large(cudaStream_t st, void* dst, const void* src, size_t bytes,
                                  bool d2h) {
  constexpr size_t kChunk = 32u << 20;
  if (bytes < (8u << 20))
    return cudaMemcpyAsync(dst, src, bytes, d2h ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice, st);
  static std::mutex mu;  // the bounce buffers are shared by every index of the process
  std::lock_guard<std::mutex> lock(mu);
  constexpr int kMaxDev = 64;  // events belong to a device: one pair of buffers per device
  static char* bounce_d[kMaxDev][2] = {};
  static cudaEvent_t ev_d[kMaxDev][2] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDev)
    return cudaMemcpyAsync(dst, src, bytes, d2h ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice, st);
  char** bounce = bounce_d[dev];
  cudaEvent_t* ev = ev_d[dev];
  if (!bounce[0] || !bounce[1] || !ev[0] || !ev[1]) {
    // (re)initialise every slot; a partial failure frees what was allocated so the next
    // call starts from a clean state instead of copying into a null buffer
    for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
      if (!bounce[b])
        e = cudaHostAlloc(reinterpret_cast<void**>(&bounce[b]), kChunk, cudaHostAllocPortable);
      if (e == cudaSuccess && !ev[b]) e = cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
      for (int b = 0; b < 2; ++b) {
        if (bounce[b]) cudaFreeHost(bounce[b]);
        if (ev[b]) cudaEventDestroy(ev[b]);
        bounce[b] = nullptr;
        ev[b] = nullptr;
      }
      return e;
    }
  }
  const size_t nch = (bytes + kChunk - 1) / kChunk;
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  auto host_copy = [&](char* to, const char* from, size_t len) {
    const size_t per = (len / hw + 4095) & ~(size_t)4095;
    std::vector<std::thread> th;
    for (unsigned t = 0; t < hw && (size_t)t * per < len; ++t) {
      const size_t o = (size_t)t * per, l = std::min(per, len - o);
      th.emplace_back([=] { memcpy(to + o, from + o, l); });
    }
    for (auto& x : th) x.join();
  };
  auto dma = [&](size_t c) {
    const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
    cudaError_t r = d2h ? cudaMemcpyAsync(bounce[c & 1], static_cast<const char*>(src) + off, len,
                                          cudaMemcpyDeviceToHost, st)
                        : cudaMemcpyAsync(static_cast<char*>(dst) + off, bounce[c & 1], len,
                                          cudaMemcpyHostToDevice, st);
    if (r == cudaSuccess) r = cudaEventRecord(ev[c & 1], st);
    return r;
  };
  if (d2h) {
    if ((e = dma(0)) != cudaSuccess) return e;
    for (size_t c = 0; c < nch; ++c) {
      if (c + 1 < nch && (e = dma(c + 1)) != cudaSuccess) return e;
      if ((e = cudaEventSynchronize(ev[c & 1])) != cudaSuccess) return e;
      const size_t off = c * kChunk;
      host_copy(static_cast<char*>(dst) + off, bounce[c & 1], std::min(kChunk, bytes - off));
    }
  } else {
    for (size_t c = 0; c < nch; ++c) {
      if (c >= 2 && (e = cudaEventSynchronize(ev[c & 1])) != cudaSuccess) return e;  // buffer free
      const size_t off = c * kChunk;
      host_copy(bounce[c & 1], static_cast<const char*>(src) + off, std::min(kChunk, bytes - off));
      if ((e = dma(c)) != cudaSuccess) return e;
    }
    // the caller's later host writes may not race the last DMAs out of the bounce buffers
    e = cudaStreamSynchronize(st);
  }
  return e;
}

struct sb_index {
  int64_t n = 0;
  int m = 0, l = 0, g = 0;
  int sms = 148;
  bool int_exact = false;  // all features integral (order-free exact distances possible)
  double fmax = 0.0;
  float flo = 0.f, fhi = 0.f;
  bool force_sequential = false;  // testing: always use the sequential-order distance path
  bool have_fb = false;           // bf16 feature copy + norms for the tensor-core top-k
  int fb_mk = 0;                  // its operand K (features, + 16 when |x|^2 is folded in)
  bool last_bf_tc = false;        // the last sb_bf_topk_queries ran on tensor cores
  int last_bf_path = 0;           // 0 fp64 SIMT, 1 tcgen05 integer-exact, 2 tcgen05 TF32 filter
  int64_t last_bf_fallback = 0;   // queries of the last TF32 call recomputed on the fp64 path
  int64_t last_bf_cands = 0;      // candidates the last TF32 call emitted (all queries)
  bool have_ft = false;           // TF32 operand copy + metadata (bf_tf.cu)
  int tf_strided = 1;             // walk the node tiles strided (skewed attribute codes)
  // the attribute tuple code of node_order: code = sum_u (a_u - lo_u) stride_u (grouped orders)
  int32_t code_lo[8] = {0};
  int64_t code_stride[8] = {0};
  bool code_grouped = false;
  cudaEvent_t bf_ev[2] = {nullptr, nullptr};  // around the last tensor-core top-k pass
  bool bf_ev_valid = false;
  bool have_f8 = false;           // u8 feature copy for routing (integer data in [0, 255])
  // routing layout: nodes renumbered in a locality order (route_layout); valid while
  // rl_version == graph_version (every call that changes the adjacency bumps graph_version)
  int64_t graph_version = 0, rl_version = -1;
  bool rl_have_f8 = false;
  int last_route_path = -1;
  cudaStream_t own = nullptr, st = nullptr;
  int64_t launches = 0;
  // dataset + adjacency
  DBuf F, A, ids, dists, flags, counts;
  // candidates
  int gn = 0;
  bool have_cand = false;
  DBuf new_cand, new_cnt, old_cand, old_cnt;
  DBuf fwd_new, fwd_old, rev_cnt, rev_off, rev_cur, rev, scan_tmp;
  // join
  DBuf thr, row_cnt, row_off, row_cur, push_tgt, push_key, seg, small;
  // prune / reinforce
  DBuf rbits, smax, indeg0, guard, drop_other, keep, in_deg, seqtmp;
  bool have_indeg = false;
  int64_t last_overflow_rows = 0;
  int64_t last_rf_groups = 0, last_rf_components = 0;  // overflow replay parallelism
  // exact reinforce (overflow rows)
  DBuf rf_n8, rf_nb, rf_n32, rf_n64, rf_o32, rf_o64, rf_ulist, rf_bits, rf_rec, rf_sim, rf_eo;
  // routing / brute force
  DBuf qf, qa, qm, entries, ent_scratch, out_ids, out_dists, stats, visited, vlog, counter;
  DBuf route_gr;                     // result lists in global memory (very large K)
  DBuf bf_part_d, bf_part_i, bf_self, bf_qa, bf_qm, bf_out32, fb, fb_norm, fb_tmp, qb, f8;
  DBuf rl_F, rl_A, rl_ids, rl_counts, rl_perm, rl_f8, rl_tmp;
  DBuf meta16;                       // {|x|^2, attrs} per node for u8 routing (l <= 3)
  int64_t meta_version = -1;         // graph_version / layout it was built for
  int meta_relabel = -1;
  DBuf ft, ft_meta, tq, tcand, tovf;
  DBuf bf_sort;                      // full-sort top-k scratch (bf_sort.cu: any k)
  DBuf tlists;                       // two-pass TF32 top-k: per-thread lists (q x threads x 32)
  DBuf fb_cmeta, fb_scratch;         // u8 top-k: per-16-node chunk records; sort scratch
  cudaStream_t st_up = nullptr;      // sb_route_batch: query upload beside the entry-point kernel
  cudaEvent_t ev_up = nullptr;
  ~sb_index() {
    if (st_up) cudaStreamDestroy(st_up);
    if (ev_up) cudaEventDestroy(ev_up);
    bf_sort.release();
    tlists.release();
    fb_cmeta.release();
    fb_scratch.release();
    fb.release();
    f8.release();
    DBuf* tfb[] = {&ft, &ft_meta, &tq, &tcand, &tovf};
    for (DBuf* b : tfb) b->release();
    DBuf* rl[] = {&rl_F, &rl_A, &rl_ids, &rl_counts, &rl_perm, &rl_f8, &rl_tmp, &meta16};
    for (DBuf* b : rl) b->release();
    fb_tmp.release();
    fb_norm.release();
    qb.release();
    DBuf* all[] = {&F, &A, &ids, &dists, &flags, &counts, &new_cand, &new_cnt, &old_cand,
                   &old_cnt, &fwd_new, &fwd_old, &rev_cnt, &rev_off, &rev_cur, &rev, &scan_tmp,
                   &thr, &row_cnt, &row_off, &row_cur, &push_tgt, &push_key, &seg, &small,
                   &rbits, &smax, &indeg0, &guard, &drop_other, &keep, &in_deg, &seqtmp, &qf,
                   &qa, &qm, &entries, &ent_scratch, &out_ids, &out_dists, &stats, &visited,
                   &vlog, &counter, &bf_part_d, &bf_part_i, &bf_self, &bf_qa, &bf_qm,
                   &bf_out32, &rf_n8, &rf_nb, &rf_n32, &rf_n64, &rf_o32, &rf_o64,
                   &rf_ulist, &rf_bits, &rf_rec, &rf_sim, &rf_eo, &route_gr};
    for (DBuf* b : all) b->release();
    if (bf_ev[0]) cudaEventDestroy(bf_ev[0]);
    if (bf_ev[1]) cudaEventDestroy(bf_ev[1]);
    if (own) cudaStreamDestroy(own);
  }
  cudaError_t bf_event(int i) {
    if (!bf_ev[i]) {
      cudaError_t e = cudaEventCreate(&bf_ev[i]);
      if (e != cudaSuccess) return e;
    }
    return cudaEventRecord(bf_ev[i], st);
  }
};

using sb::next_pow2;

extern "C" {

const char* sb_last_error(void) { return g_err.c_str(); }
int sb_version(void) { return (0 << 16) | 1; }

int sb_device_count(int* count) {
  if (!count) return fail(SB_EARG, "count is NULL");
  cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    *count = 0;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  return SB_OK;
}

int sb_index_create(const float* features, const int32_t* attrs, int64_t n, int32_t m, int32_t l,
                    int32_t gamma, sb_index** out) {
  if (!out) return fail(SB_EARG, "out is NULL");
  *out = nullptr;
  if (!features || !attrs) return fail(SB_EARG, "features/attrs are NULL");
  if (n < 1 || m < 1 || l < 1) return fail(SB_EARG, "n, m and l must be >= 1");
  if (gamma < 2 || gamma > 256) return fail(SB_EARG, "gamma must be in [2, 256]");
  if (n >= (int64_t)1 << 30) return fail(SB_EARG, "n must be < 2^30");
  sb_index* x = new sb_index();
  x->n = n; x->m = m; x->l = l; x->g = gamma;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&x->sms, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&x->own, cudaStreamNonBlocking);
  if (e != cudaSuccess) { delete x; return cuda_fail(e, "device/stream setup"); }
  x->st = x->own;
  size_t fb = sizeof(float) * (size_t)n * m, ab = sizeof(int32_t) * (size_t)n * l;
  size_t adj = (size_t)n * gamma;
  if ((e = x->F.ensure(fb)) != cudaSuccess || (e = x->A.ensure(ab)) != cudaSuccess ||
      (e = x->ids.ensure(adj * 4)) != cudaSuccess || (e = x->dists.ensure(adj * 4)) != cudaSuccess ||
      (e = x->flags.ensure(adj)) != cudaSuccess || (e = x->counts.ensure((size_t)n * 4)) != cudaSuccess) {
    delete x;
    return cuda_fail(e, "cudaMalloc(index)");
  }
  e = transfer_large(x->st, x->F.p, features, fb, false);
  if (e == cudaSuccess) e = cudaMemcpyAsync(x->A.p, attrs, ab, cudaMemcpyHostToDevice, x->st);
  if (e == cudaSuccess) e = cudaMemsetAsync(x->counts.p, 0, (size_t)n * 4, x->st);
  if (e == cudaSuccess) e = cudaMemsetAsync(x->flags.p, 0, adj, x->st);
  if (e == cudaSuccess) e = x->small.ensure(64);
  if (e == cudaSuccess) {
    unsigned* f3 = x->small.as<unsigned>() + 12;
    int r = sb::launch_feature_scan(x->F.as<float>(), (int64_t)n * m, f3, x->st);
    if (r) e = (cudaError_t)r;
    unsigned h[3] = {1, 0, 0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(h, f3, sizeof(h), cudaMemcpyDeviceToHost, x->st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(x->st);
    x->flo = sb::feature_key_to_float(h[1]);
    x->fhi = sb::feature_key_to_float(h[2]);
    x->int_exact = h[0] == 0;
    x->fmax = std::max(std::fabs((double)x->flo), std::fabs((double)x->fhi));
  }
  if (e != cudaSuccess) { delete x; return cuda_fail(e, "upload(index)"); }
  *out = x;
  return SB_OK;
}

int sb_index_destroy(sb_index* idx) {
  delete idx;
  return SB_OK;
}

int sb_set_stream(sb_index* idx, void* s) {
  if (!idx) return fail(SB_EARG, "idx is NULL");
  idx->st = s ? reinterpret_cast<cudaStream_t>(s) : idx->own;
  return SB_OK;
}

int sb_synchronize(sb_index* idx) {
  if (!idx) return fail(SB_EARG, "idx is NULL");
  CK(cudaStreamSynchronize(idx->st));
  return SB_OK;
}

int64_t sb_launch_count(sb_index* idx) { return idx ? idx->launches : 0; }

int sb_index_info(sb_index* idx, int32_t* int_exact, double* fmax_abs, int32_t* last_bf_tc) {
  if (!idx) return fail(SB_EARG, "idx is NULL");
  if (last_bf_tc) *last_bf_tc = idx->last_bf_tc ? 1 : 0;
  if (int_exact) *int_exact = idx->int_exact ? 1 : 0;
  if (fmax_abs) *fmax_abs = idx->fmax;
  return SB_OK;
}

int sb_bf_info(sb_index* idx, int32_t* path, int64_t* candidates, int64_t* fallback,
               double* kernel_ms) {
  if (!idx) return fail(SB_EARG, "idx is NULL");
  if (kernel_ms) {
    *kernel_ms = 0.0;
    if (idx->bf_ev_valid) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, idx->bf_ev[0], idx->bf_ev[1]));
      *kernel_ms = ms;
    }
  }
  if (path) *path = idx->last_bf_path;
  if (candidates) *candidates = idx->last_bf_cands;
  if (fallback) *fallback = idx->last_bf_fallback;
  return SB_OK;
}

int sb_host_alloc(size_t bytes, void** out) {
  if (!out) return fail(SB_EARG, "NULL argument");
  *out = nullptr;
  if (bytes == 0) return SB_OK;
  CK(cudaHostAlloc(out, bytes, cudaHostAllocDefault));
  return SB_OK;
}

int sb_host_free(void* p) {
  if (p) CK(cudaFreeHost(p));
  return SB_OK;
}

int sb_route_info(sb_index* idx, int32_t* path, int32_t* row_bytes) {
  if (!idx) return fail(SB_EARG, "idx is NULL");
  if (path) *path = idx->last_route_path;
  if (row_bytes) *row_bytes = idx->last_route_path == 4 ? idx->m : 4 * idx->m;
  return SB_OK;
}

int sb_set_distance_mode(sb_index* idx, int32_t mode) {
  if (!idx) return fail(SB_EARG, "idx is NULL");
  if (mode != 0 && mode != 1) return fail(SB_EARG, "mode must be 0 (auto) or 1 (sequential)");
  idx->force_sequential = mode == 1;
  return SB_OK;
}

int sb_adj_upload(sb_index* idx, const int32_t* ids, const float* dists, const int32_t* counts,
                  const uint8_t* flags) {
  if (idx) idx->graph_version++;
  if (!idx || !ids || !dists || !counts) return fail(SB_EARG, "NULL argument");
  size_t adj = (size_t)idx->n * idx->g;
  CK(transfer_large(idx->st, idx->ids.p, ids, adj * 4, false));
  CK(transfer_large(idx->st, idx->dists.p, dists, adj * 4, false));
  CK(cudaMemcpyAsync(idx->counts.p, counts, (size_t)idx->n * 4, cudaMemcpyHostToDevice, idx->st));
  if (flags) CK(cudaMemcpyAsync(idx->flags.p, flags, adj, cudaMemcpyHostToDevice, idx->st));
  idx->have_cand = false;
  idx->have_indeg = false;
  CK(cudaStreamSynchronize(idx->st));
  return SB_OK;
}

int sb_adj_download(sb_index* idx, int32_t* ids, float* dists, int32_t* counts, uint8_t* flags) {
  if (!idx) return fail(SB_EARG, "idx is NULL");
  size_t adj = (size_t)idx->n * idx->g;
  if (ids) CK(transfer_large(idx->st, ids, idx->ids.p, adj * 4, true));
  if (dists) CK(transfer_large(idx->st, dists, idx->dists.p, adj * 4, true));
  if (counts) CK(cudaMemcpyAsync(counts, idx->counts.p, (size_t)idx->n * 4, cudaMemcpyDeviceToHost, idx->st));
  if (flags) CK(transfer_large(idx->st, flags, idx->flags.p, adj, true));
  CK(cudaStreamSynchronize(idx->st));
  return SB_OK;
}

// ---------------------------------------------------------------------------
__global__ void sb_fill_i32(int32_t* p, int64_t n, int32_t v) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

int sb_init_random_ids(sb_index* idx, uint64_t seed, int64_t* consumed32, uint32_t* buffered,
                       int64_t* bad_rows, int64_t bad_cap, int64_t* nbad) {
  if (idx) idx->graph_version++;
  if (!idx || !consumed32 || !nbad) return fail(SB_EARG, "NULL argument");
  const int64_t n = idx->n;
  const int g = idx->g;
  if (n <= g) return fail(SB_EARG, "dataset size must exceed gamma");
  if (n - 1 > (int64_t)0xFFFFFFFF) return fail(SB_EARG, "n too large for the 32-bit draw path");
  const int64_t slots = sb::init_random_ids_scratch_slots(n, g);
  CK(idx->seg.ensure(sizeof(int64_t) * (size_t)std::max<int64_t>(slots, n + 4)));
  int64_t* scratch = idx->seg.as<int64_t>();
  CK(idx->small.ensure(64));
  int64_t* d_consumed = reinterpret_cast<int64_t*>(idx->small.as<unsigned long long>() + 2);
  unsigned long long* d_nbad = idx->small.as<unsigned long long>() + 4;
  CK(idx->rev_cnt.ensure(sizeof(int64_t) * n));
  int64_t* d_bad = idx->rev_cnt.as<int64_t>();
  CKL(sb::launch_init_random_ids(seed, n, g, idx->ids.as<int32_t>(), scratch, slots, d_consumed,
                                 d_bad, d_nbad, idx->st));
  int64_t consumed[2] = {-1, 0};
  unsigned long long nb = 0;
  CK(cudaMemcpyAsync(consumed, d_consumed, sizeof(consumed), cudaMemcpyDeviceToHost, idx->st));
  CK(cudaMemcpyAsync(&nb, d_nbad, sizeof(nb), cudaMemcpyDeviceToHost, idx->st));
  CK(cudaStreamSynchronize(idx->st));
  if (consumed[0] < 0) return fail(SB_ECUDA, "random init: rejection margin exhausted");
  *consumed32 = consumed[0];
  if (buffered) *buffered = (uint32_t)consumed[1];
  *nbad = (int64_t)nb;
  if (bad_rows && nb > 0) {
    if ((int64_t)nb > bad_cap) return fail(SB_EARG, "bad_rows capacity too small");
    CK(cudaMemcpyAsync(bad_rows, d_bad, sizeof(int64_t) * nb, cudaMemcpyDeviceToHost, idx->st));
    CK(cudaStreamSynchronize(idx->st));
    std::sort(bad_rows, bad_rows + nb);
  }
  idx->launches += 4;
  idx->have_cand = false;
  return SB_OK;
}

int sb_set_rows(sb_index* idx, const int64_t* rows, int64_t s, const int32_t* ids) {
  if (idx) idx->graph_version++;
  if (!idx || (s > 0 && (!rows || !ids))) return fail(SB_EARG, "NULL argument");
  const int g = idx->g;
  for (int64_t i = 0; i < s; ++i) {
    if (rows[i] < 0 || rows[i] >= idx->n) return fail(SB_EARG, "row out of range");
    CK(cudaMemcpyAsync(idx->ids.as<int32_t>() + rows[i] * g, ids + i * g, sizeof(int32_t) * g,
                       cudaMemcpyHostToDevice, idx->st));
  }
  CK(cudaStreamSynchronize(idx->st));
  idx->have_cand = false;
  return SB_OK;
}

int sb_init_graph(sb_index* idx, const int32_t* ids, double inv_alpha) {
  if (idx) idx->graph_version++;
  if (!idx) return fail(SB_EARG, "NULL argument");
  if (idx->n <= idx->g) return fail(SB_EARG, "dataset size must exceed gamma");
  size_t adj = (size_t)idx->n * idx->g;
  if (ids) CK(cudaMemcpyAsync(idx->ids.p, ids, adj * 4, cudaMemcpyHostToDevice, idx->st));
  CKL(sb::launch_init_dists(idx->F.as<float>(), idx->A.as<int32_t>(), idx->n, idx->m, idx->l,
                            idx->g, inv_alpha, idx->ids.as<int32_t>(), idx->dists.as<float>(),
                            idx->st));
  sb_fill_i32<<<(unsigned)((idx->n + 255) / 256), 256, 0, idx->st>>>(idx->counts.as<int32_t>(),
                                                                      idx->n, idx->g);
  CK(cudaMemsetAsync(idx->flags.p, 1, adj, idx->st));
  idx->launches += 2;
  idx->have_cand = false;
  CK(cudaStreamSynchronize(idx->st));
  return SB_OK;
}

int sb_build_candidates(sb_index* idx, int32_t gamma_new, int32_t* new_cand, int32_t* new_counts,
                        int32_t* old_cand, int32_t* old_counts) {
  if (!idx) return fail(SB_EARG, "idx is NULL");
  if (gamma_new < 1 || gamma_new > 256) return fail(SB_EARG, "gamma_new must be in [1, 256]");
  const int64_t n = idx->n;
  const int g = idx->g;
  idx->gn = gamma_new;
  CK(idx->new_cand.ensure(sizeof(int32_t) * n * gamma_new));
  CK(idx->old_cand.ensure(sizeof(int32_t) * n * g));
  CK(idx->new_cnt.ensure(sizeof(int32_t) * n));
  CK(idx->old_cnt.ensure(sizeof(int32_t) * n));
  CK(idx->fwd_new.ensure(sizeof(int32_t) * n));
  CK(idx->fwd_old.ensure(sizeof(int32_t) * n));
  CK(idx->rev_cnt.ensure(sizeof(int64_t) * n));
  CK(idx->rev_off.ensure(sizeof(int64_t) * n));
  CK(idx->rev_cur.ensure(sizeof(int64_t) * n));
  CK(idx->rev.ensure(sizeof(int32_t) * n * std::max(gamma_new, g)));
  CK(idx->scan_tmp.ensure(sizeof(int64_t) * sb::scan_tmp_slots(n)));
  sb::BuildScratch s;
  s.fwd_new = idx->fwd_new.as<int32_t>();
  s.fwd_old = idx->fwd_old.as<int32_t>();
  s.rev_cnt = idx->rev_cnt.as<int64_t>();
  s.rev_off = idx->rev_off.as<int64_t>();
  s.rev_cur = idx->rev_cur.as<int64_t>();
  s.rev = idx->rev.as<int32_t>();
  s.scan_tmp = idx->scan_tmp.as<int64_t>();
  CKL(sb::launch_build_candidates(idx->ids.as<int32_t>(), idx->flags.as<uint8_t>(), n, g,
                                  gamma_new, idx->new_cand.as<int32_t>(),
                                  idx->new_cnt.as<int32_t>(), idx->old_cand.as<int32_t>(),
                                  idx->old_cnt.as<int32_t>(), s, idx->st));
  idx->launches += 9;
  idx->have_cand = true;
  if (new_cand) CK(cudaMemcpyAsync(new_cand, idx->new_cand.p, sizeof(int32_t) * n * gamma_new, cudaMemcpyDeviceToHost, idx->st));
  if (new_counts) CK(cudaMemcpyAsync(new_counts, idx->new_cnt.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, idx->st));
  if (old_cand) CK(cudaMemcpyAsync(old_cand, idx->old_cand.p, sizeof(int32_t) * n * g, cudaMemcpyDeviceToHost, idx->st));
  if (old_counts) CK(cudaMemcpyAsync(old_counts, idx->old_cnt.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, idx->st));
  CK(cudaStreamSynchronize(idx->st));
  return SB_OK;
}

int sb_set_candidates(sb_index* idx, int32_t gamma_new, const int32_t* new_cand,
                      const int32_t* new_counts, const int32_t* old_cand,
                      const int32_t* old_counts) {
  if (!idx || !new_cand || !new_counts || !old_cand || !old_counts) return fail(SB_EARG, "NULL argument");
  if (gamma_new < 1 || gamma_new > 256) return fail(SB_EARG, "gamma_new must be in [1, 256]");
  const int64_t n = idx->n;
  const int g = idx->g;
  idx->gn = gamma_new;
  CK(idx->new_cand.ensure(sizeof(int32_t) * n * gamma_new));
  CK(idx->old_cand.ensure(sizeof(int32_t) * n * g));
  CK(idx->new_cnt.ensure(sizeof(int32_t) * n));
  CK(idx->old_cnt.ensure(sizeof(int32_t) * n));
  CK(cudaMemcpyAsync(idx->new_cand.p, new_cand, sizeof(int32_t) * n * gamma_new, cudaMemcpyHostToDevice, idx->st));
  CK(cudaMemcpyAsync(idx->new_cnt.p, new_counts, sizeof(int32_t) * n, cudaMemcpyHostToDevice, idx->st));
  CK(cudaMemcpyAsync(idx->old_cand.p, old_cand, sizeof(int32_t) * n * g, cudaMemcpyHostToDevice, idx->st));
  CK(cudaMemcpyAsync(idx->old_cnt.p, old_counts, sizeof(int32_t) * n, cudaMemcpyHostToDevice, idx->st));
  CK(cudaStreamSynchronize(idx->st));
  idx->have_cand = true;
  return SB_OK;
}

static int ensure_u8(sb_index* idx, const float* F, DBuf& buf, bool& have);

int sb_local_join(sb_index* idx, double inv_alpha, int64_t* inserted_out, int64_t* pairs_out) {
  if (idx) idx->graph_version++;
  if (!idx) return fail(SB_EARG, "idx is NULL");
  if (!idx->have_cand) return fail(SB_EARG, "sb_build_candidates must run first");
  const int64_t n = idx->n;
  const int g = idx->g, gn = idx->gn;
  // per-node worst-case pushes (2 per pair) to plan chunks
  std::vector<int32_t> nc(n), oc(n);
  CK(cudaMemcpyAsync(nc.data(), idx->new_cnt.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, idx->st));
  CK(cudaMemcpyAsync(oc.data(), idx->old_cnt.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, idx->st));
  CK(cudaStreamSynchronize(idx->st));
  std::vector<uint64_t> worst(n);
  uint64_t total_pairs = 0, total_worst = 0;
  int max_ns = 1, max_na = 1;
  for (int64_t i = 0; i < n; ++i) {
    uint64_t na = (uint64_t)nc[i], nb = (uint64_t)oc[i];
    uint64_t pairs = na * (na > 0 ? na - 1 : 0) / 2 + na * nb;
    total_pairs += pairs;
    worst[i] = 2 * pairs;
    total_worst += worst[i];
    max_ns = std::max(max_ns, (int)(na + nb));
    max_na = std::max(max_na, (int)na);
  }
  if (pairs_out) *pairs_out = (int64_t)total_pairs;
  CK(idx->thr.ensure(sizeof(uint64_t) * n));
  CK(idx->row_cnt.ensure(sizeof(int64_t) * n));
  CK(idx->row_off.ensure(sizeof(int64_t) * n));
  CK(idx->row_cur.ensure(sizeof(int64_t) * n));
  CK(idx->small.ensure(64));
  CK(idx->scan_tmp.ensure(sizeof(int64_t) * sb::scan_tmp_slots(n)));
  CKL(sb::launch_thr_init(idx->ids.as<int32_t>(), idx->dists.as<float>(), n, g,
                          idx->thr.as<uint64_t>(), idx->st));
  // integer features in [0, 255]: pair distances from u8 rows with dp4a (exact), unless
  // SB_JOIN_U8=0
  bool join_u8 = idx->int_exact && idx->flo >= 0.f && idx->fhi <= 255.f && idx->m % 4 == 0 &&
                 !idx->force_sequential;
  if (const char* e = getenv("SB_JOIN_U8")) join_u8 = join_u8 && atoi(e) != 0;
  if (join_u8) {
    int r = ensure_u8(idx, idx->F.as<float>(), idx->f8, idx->have_f8);
    if (r) return r;
  }
  // emit kernel geometry
  const int spad = (max_ns + 3) & ~3;
  const int ntiles_max = ((max_na + 3) / 4) * ((max_ns + 3) / 4);
  const size_t stage_budget = 96 * 1024;
  int dc = (int)std::min<int64_t>(idx->m, (int64_t)(stage_budget / (sizeof(float) * spad)));
  if (dc < idx->m) dc = std::max(4, dc & ~3);
  // the u8 path stages m / 4 words per slot (the stage is sized by dc): room for more CTAs
  if (join_u8) dc = idx->m / 4;
  size_t smem = sb::join_emit_smem(spad, dc, idx->l, ntiles_max);
  int per_sm = 0;
  CKL(sb::join_emit_occupancy(smem, &per_sm));
  if (per_sm < 1) return fail(SB_ECUDA, "join kernel does not fit on an SM");
  const int ctas = idx->sms * per_sm;
  // reservation padding: each warp may leave < 1024 slots of its last block unused, and a
  // block renewal pads at most 63 slots (<= 64 pushes per warp step) — plan with 7% headroom
  const uint64_t slack = (uint64_t)ctas * (256 / 32) * 1024;
  for (int64_t i = 0; i < n; ++i) worst[i] += worst[i] / 14 + 64;
  total_worst += total_worst / 14 + 64 * (uint64_t)n;
  // push buffer: 4 + 8 (emit) + 8 (segments) bytes per slot
  size_t free_b = 0, tot_b = 0;
  CK(cudaMemGetInfo(&free_b, &tot_b));
  uint64_t budget_slots = (uint64_t)(free_b * 0.6) / 20;
  uint64_t max_worst = 0;
  for (int64_t i = 0; i < n; ++i) max_worst = std::max(max_worst, worst[i]);
  uint64_t cap = std::min<uint64_t>(total_worst + slack, budget_slots);
  if (cap < slack + max_worst) return fail(SB_ECUDA, "not enough device memory for the join buffers");
  CK(idx->push_tgt.ensure(sizeof(uint32_t) * cap));
  CK(idx->push_key.ensure(sizeof(uint64_t) * cap));
  CK(idx->seg.ensure(sizeof(uint64_t) * cap));
  unsigned long long* d_count = idx->small.as<unsigned long long>();
  unsigned long long* d_inserted = d_count + 1;
  int* d_nodectr = reinterpret_cast<int*>(d_count + 2);
  int* d_overflow = d_nodectr + 1;
  unsigned long long* d_same = d_count + 3;  // small: [count, inserted, nodectr|overflow, same]
  CK(cudaMemsetAsync(d_inserted, 0, sizeof(unsigned long long), idx->st));
  CK(cudaMemsetAsync(d_same, 0, sizeof(unsigned long long), idx->st));
  int64_t begin = 0;
  while (begin < n) {
    uint64_t acc = slack;
    int64_t end = begin;
    while (end < n && acc + worst[end] <= cap) acc += worst[end++];
    if (end == begin) return fail(SB_ECUDA, "join buffer too small for one node");
    CK(cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), idx->st));
    CK(cudaMemsetAsync(d_nodectr, 0, sizeof(int) * 2, idx->st));
    CK(cudaMemsetAsync(idx->row_cnt.p, 0, sizeof(int64_t) * n, idx->st));
    sb::JoinArgs a;
    a.F = idx->F.as<float>(); a.A = idx->A.as<int32_t>(); a.n = n; a.m = idx->m; a.l = idx->l;
    a.g = g; a.gn = gn; a.inv_alpha = inv_alpha;
    a.new_cand = idx->new_cand.as<int32_t>(); a.new_cnt = idx->new_cnt.as<int32_t>();
    a.old_cand = idx->old_cand.as<int32_t>(); a.old_cnt = idx->old_cnt.as<int32_t>();
    a.thr = idx->thr.as<uint64_t>(); a.node_begin = begin; a.node_end = end;
    a.node_counter = d_nodectr; a.push_tgt = idx->push_tgt.as<uint32_t>();
    a.push_key = idx->push_key.as<uint64_t>(); a.push_cap = cap; a.push_count = d_count;
    a.row_cnt = idx->row_cnt.as<int64_t>(); a.overflow = d_overflow; a.spad = spad; a.dc = dc;
    a.same_pairs = d_same;
    a.ntiles_max = ntiles_max;
    a.F8 = join_u8 ? idx->f8.as<uint8_t>() : nullptr;
    a.nx8 = join_u8 ? reinterpret_cast<const int32_t*>(idx->f8.as<uint8_t>() + (((size_t)n * idx->m + 255) & ~(size_t)255)) : nullptr;
    int nctas = (int)std::min<int64_t>(ctas, end - begin);
    CKL(sb::launch_join_emit(a, nctas, smem, idx->st));
    unsigned long long used = 0;
    int over = 0;
    CK(cudaMemcpyAsync(&used, d_count, sizeof(used), cudaMemcpyDeviceToHost, idx->st));
    CK(cudaMemcpyAsync(&over, d_overflow, sizeof(int), cudaMemcpyDeviceToHost, idx->st));
    CK(cudaStreamSynchronize(idx->st));
    if (over) return fail(SB_ECUDA, "join push buffer overflow (planning bug)");
    uint64_t total = std::min<uint64_t>(used, cap);
    CKL(sb::exclusive_scan(idx->row_cnt.as<int64_t>(), idx->row_off.as<int64_t>(), n,
                           idx->scan_tmp.as<int64_t>(), idx->st));
    CK(cudaMemsetAsync(idx->row_cur.p, 0, sizeof(int64_t) * n, idx->st));
    CKL(sb::launch_push_scatter(idx->push_tgt.as<uint32_t>(), idx->push_key.as<uint64_t>(), total,
                                idx->row_off.as<int64_t>(), idx->row_cur.as<int64_t>(),
                                idx->seg.as<uint64_t>(), idx->st));
    CKL(sb::launch_row_merge(idx->ids.as<int32_t>(), idx->dists.as<float>(),
                             idx->flags.as<uint8_t>(), idx->thr.as<uint64_t>(), n, g,
                             idx->row_off.as<int64_t>(), idx->row_cnt.as<int64_t>(),
                             idx->seg.as<uint64_t>(), d_inserted, idx->st));
    idx->launches += 5;
    begin = end;
  }
  unsigned long long ins = 0, same = 0;
  CK(cudaMemcpyAsync(&ins, d_inserted, sizeof(ins), cudaMemcpyDeviceToHost, idx->st));
  CK(cudaMemcpyAsync(&same, d_same, sizeof(same), cudaMemcpyDeviceToHost, idx->st));
  CK(cudaStreamSynchronize(idx->st));
  if (inserted_out) *inserted_out = (int64_t)ins;
  // pairs evaluated exactly as the reference's loop counts them (j == k pairs are skipped,
  // _kernels.py:160,168)
  if (pairs_out) *pairs_out = (int64_t)(total_pairs - same);
  idx->have_cand = false;
  return SB_OK;
}

int sb_descent_iteration(sb_index* idx, int32_t gamma_new, double inv_alpha, int64_t* inserted,
                         int64_t* pairs) {
  int r = sb_build_candidates(idx, gamma_new, nullptr, nullptr, nullptr, nullptr);
  if (r) return r;
  return sb_local_join(idx, inv_alpha, inserted, pairs);
}

int sb_count_in_degrees(sb_index* idx, int64_t* in_deg) {
  if (!idx || !in_deg) return fail(SB_EARG, "NULL argument");
  const int64_t n = idx->n;
  CK(idx->in_deg.ensure(sizeof(int32_t) * n));
  CKL(sb::launch_count_in_degrees(idx->ids.as<int32_t>(), idx->counts.as<int32_t>(), n, idx->g,
                                  idx->in_deg.as<int32_t>(), nullptr, idx->st));
  idx->launches += 1;
  std::vector<int32_t> h(n);
  CK(cudaMemcpyAsync(h.data(), idx->in_deg.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, idx->st));
  CK(cudaStreamSynchronize(idx->st));
  for (int64_t i = 0; i < n; ++i) in_deg[i] = h[i];
  return SB_OK;
}

__global__ void sb_gather_rows(const int32_t* ids, const int32_t* counts, int g, const int64_t* rows,
                               int64_t s, int32_t* out_ids, int32_t* out_counts) {
  int64_t r = blockIdx.x;
  if (r >= s) return;
  int64_t row = rows[r];
  for (int t = threadIdx.x; t < g; t += blockDim.x) out_ids[r * g + t] = ids[row * g + t];
  if (threadIdx.x == 0) out_counts[r] = counts[row];
}

int sb_get_rows(sb_index* idx, const int64_t* rows, int64_t s, int32_t* ids, int32_t* counts) {
  if (!idx || !rows || !ids || !counts) return fail(SB_EARG, "NULL argument");
  if (s <= 0) return SB_OK;
  const int g = idx->g;
  size_t need = sizeof(int64_t) * s + sizeof(int32_t) * s * (g + 1);
  CK(idx->bf_self.ensure(need));
  int64_t* d_rows = idx->bf_self.as<int64_t>();
  int32_t* d_ids = reinterpret_cast<int32_t*>(d_rows + s);
  int32_t* d_cnt = d_ids + s * g;
  CK(cudaMemcpyAsync(d_rows, rows, sizeof(int64_t) * s, cudaMemcpyHostToDevice, idx->st));
  sb_gather_rows<<<(unsigned)s, 128, 0, idx->st>>>(idx->ids.as<int32_t>(), idx->counts.as<int32_t>(),
                                                    g, d_rows, s, d_ids, d_cnt);
  idx->launches += 1;
  CK(cudaMemcpyAsync(ids, d_ids, sizeof(int32_t) * s * g, cudaMemcpyDeviceToHost, idx->st));
  CK(cudaMemcpyAsync(counts, d_cnt, sizeof(int32_t) * s, cudaMemcpyDeviceToHost, idx->st));
  CK(cudaStreamSynchronize(idx->st));
  return SB_OK;
}

int sb_prune(sb_index* idx, double sigma, int32_t* rounds_out) {
  if (idx) idx->graph_version++;
  if (!idx) return fail(SB_EARG, "idx is NULL");
  const int64_t n = idx->n;
  const int g = idx->g, W = (g + 31) / 32;
  CK(idx->smax.ensure(sizeof(int32_t) * n));
  CK(idx->indeg0.ensure(sizeof(int32_t) * n));
  CK(idx->in_deg.ensure(sizeof(int32_t) * n));
  CK(idx->guard.ensure(n));
  CK(idx->drop_other.ensure(sizeof(int32_t) * n));
  CK(idx->keep.ensure(sizeof(uint32_t) * n * W));
  CK(idx->rbits.ensure(sizeof(uint32_t) * n * g * W));
  CK(idx->small.ensure(64));
  CKL(sb::launch_count_in_degrees(idx->ids.as<int32_t>(), idx->counts.as<int32_t>(), n, g,
                                  idx->indeg0.as<int32_t>(), idx->smax.as<int32_t>(), idx->st));
  CK(cudaMemsetAsync(idx->guard.p, 0, n, idx->st));
  sb::PruneArgs a;
  a.F = idx->F.as<float>(); a.A = idx->A.as<int32_t>(); a.n = n; a.m = idx->m; a.l = idx->l;
  a.g = g; a.W = W; a.ids = idx->ids.as<int32_t>(); a.dists = idx->dists.as<float>();
  a.counts = idx->counts.as<int32_t>(); a.sigma = sigma; a.rbits = idx->rbits.as<uint32_t>();
  a.smax = idx->smax.as<int32_t>(); a.indeg0 = idx->indeg0.as<int32_t>();
  a.guard = idx->guard.as<uint8_t>(); a.drop_other = idx->drop_other.as<int32_t>();
  a.keep = idx->keep.as<uint32_t>(); a.in_deg = idx->in_deg.as<int32_t>();
  a.cpad = (g + 3) & ~3;
  const size_t stage_budget = 96 * 1024;
  a.dc = (int)std::min<int64_t>(idx->m, (int64_t)(stage_budget / (sizeof(float) * a.cpad)));
  // integer features in [0, 255]: exact integer cosine terms from u8 rows (dp4a), unless
  // SB_PRUNE_U8=0
  bool prune_u8 = idx->int_exact && idx->flo >= 0.f && idx->fhi <= 255.f && idx->m % 4 == 0 &&
                  idx->m <= 4096 && !idx->force_sequential;
  if (const char* e = getenv("SB_PRUNE_U8")) prune_u8 = prune_u8 && atoi(e) != 0;
  if (prune_u8) {
    int r = ensure_u8(idx, idx->F.as<float>(), idx->f8, idx->have_f8);
    if (r) return r;
    const int32_t* nx8 = reinterpret_cast<const int32_t*>(idx->f8.as<uint8_t>() +
                                                          (((size_t)n * idx->m + 255) & ~(size_t)255));
    CKL(sb::launch_prune_bits_u8(a, idx->f8.as<uint8_t>(), nx8,
                                 sb::prune_bits_u8_smem(a.cpad, idx->m, idx->l, W), idx->st));
  } else {
    size_t smem = sb::prune_bits_smem(a.cpad, a.dc, idx->m, idx->l, W);
    CKL(sb::launch_prune_bits(a, smem, idx->st));
  }
  int* d_changed = reinterpret_cast<int*>(idx->small.p);
  int rounds = 0;
  for (;;) {
    CK(cudaMemsetAsync(idx->drop_other.p, 0, sizeof(int32_t) * n, idx->st));
    CK(cudaMemsetAsync(d_changed, 0, sizeof(int), idx->st));
    CKL(sb::launch_prune_scan(a, idx->st));
    CKL(sb::launch_prune_guard(a, d_changed, idx->st));
    idx->launches += 2;
    int changed = 0;
    CK(cudaMemcpyAsync(&changed, d_changed, sizeof(int), cudaMemcpyDeviceToHost, idx->st));
    CK(cudaStreamSynchronize(idx->st));
    ++rounds;
    if (!changed) break;
    if (rounds > 100000) return fail(SB_ECUDA, "prune guard iteration did not converge");
  }
  CK(cudaMemcpyAsync(idx->in_deg.p, idx->indeg0.p, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, idx->st));
  CKL(sb::launch_prune_compact(a, idx->st));
  idx->launches += 3;
  idx->have_indeg = true;
  CK(cudaStreamSynchronize(idx->st));
  if (rounds_out) *rounds_out = rounds;
  return SB_OK;
}

// exact reinforce when some row can overflow (help_reinforce.cu)
static int reinforce_overflow(sb_index* idx, double sigma) {
  const int64_t n = idx->n;
  const int g = idx->g;
  sb::RfArgs a{};
  a.n = n; a.m = idx->m; a.l = idx->l; a.g = g;
  a.F = idx->F.as<float>(); a.A = idx->A.as<int32_t>();
  a.ids = idx->ids.as<int32_t>(); a.dists = idx->dists.as<float>();
  a.counts = idx->counts.as<int32_t>(); a.in_deg = idx->in_deg.as<int32_t>(); a.sigma = sigma;
  CK(idx->rf_n8.ensure((size_t)n * g));            // mutual flags
  CK(idx->rf_eo.ensure(sizeof(int32_t) * (size_t)n * g * 2));  // per-edge O index, U position
  CK(idx->rf_nb.ensure((size_t)n * 2));            // is_o, relevant
  CK(idx->rf_n32.ensure(sizeof(int32_t) * n * 2)); // o_idx, static_ins
  CK(idx->rf_n64.ensure(sizeof(int64_t) * n * 8)); // rev_extra, oflag, oscan, orev, apply x3, rec_head
  a.mutual = idx->rf_n8.as<uint8_t>();
  a.eo = idx->rf_eo.as<int32_t>();
  a.ecu = a.eo + (size_t)n * g;
  a.is_o = idx->rf_nb.as<uint8_t>();
  a.relevant = a.is_o + n;
  a.o_idx = idx->rf_n32.as<int32_t>();
  a.static_ins = a.o_idx + n;
  int64_t* p64 = idx->rf_n64.as<int64_t>();
  a.rev_extra = p64; int64_t* oflag = p64 + n; int64_t* oscan = p64 + 2 * n;
  a.orev_cnt = p64 + 3 * n; a.apply_cnt = p64 + 4 * n; a.apply_off = p64 + 5 * n;
  a.apply_cur = p64 + 6 * n; a.rec_head = p64 + 7 * n;
  CKL(sb::rf_launch_stage1(a, oflag, oscan, idx->scan_tmp.as<int64_t>(), idx->st));
  int64_t last[2] = {0, 0};
  CK(cudaMemcpyAsync(&last[0], oscan + n - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, idx->st));
  CK(cudaMemcpyAsync(&last[1], oflag + n - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, idx->st));
  CK(cudaStreamSynchronize(idx->st));
  const int64_t no = last[0] + last[1];
  a.no = no;
  CK(idx->rf_o32.ensure(sizeof(int32_t) * no * (1 + (size_t)g)));
  a.o_nodes = idx->rf_o32.as<int32_t>();
  a.u_pos = a.o_nodes + no;
  CK(idx->rf_o64.ensure(sizeof(int64_t) * (no * 4 + 4)));
  a.u_size = idx->rf_o64.as<int64_t>();
  a.u_off = a.u_size + no;
  a.u_cur = a.u_off + no + 1;
  a.r_off = a.u_cur + no;
  CKL(sb::rf_launch_stage2(a, oscan, idx->st));
  std::vector<int64_t> usz(no), uoff(no + 1), roff(no + 1);
  CK(cudaMemcpyAsync(usz.data(), a.u_size, sizeof(int64_t) * no, cudaMemcpyDeviceToHost, idx->st));
  CK(cudaStreamSynchronize(idx->st));
  int64_t umax = 1, wmax = 1;
  uoff[0] = 0; roff[0] = 0;
  for (int64_t o = 0; o < no; ++o) {
    int64_t W = (usz[o] + 31) / 32;
    uoff[o + 1] = uoff[o] + usz[o];
    roff[o + 1] = roff[o] + usz[o] * W;
    umax = std::max(umax, usz[o]);
    wmax = std::max(wmax, W);
  }
  if (umax > 4096) return fail(SB_ECUDA, "reinforce: an overflow row has more than 4096 candidate members");
  CK(cudaMemcpyAsync(a.u_off, uoff.data(), sizeof(int64_t) * (no + 1), cudaMemcpyHostToDevice, idx->st));
  CK(cudaMemcpyAsync(a.r_off, roff.data(), sizeof(int64_t) * (no + 1), cudaMemcpyHostToDevice, idx->st));
  CK(idx->rf_ulist.ensure(sizeof(int32_t) * (uoff[no] + 1)));
  CK(idx->rf_bits.ensure(sizeof(uint32_t) * (roff[no] + 1)));
  a.u_list = idx->rf_ulist.as<int32_t>();
  a.r_bits = idx->rf_bits.as<uint32_t>();
  CK(cudaMemsetAsync(a.r_bits, 0, sizeof(uint32_t) * (roff[no] + 1), idx->st));
  const int upad_max = next_pow2((int)umax);
  const int upad4 = (int)((umax + 3) & ~3);
  int dc_max = (int)std::min<int64_t>(idx->m, (96 * 1024) / (4 * (int64_t)upad4));
  dc_max = std::max(1, dc_max);
  size_t bits_smem = sizeof(double) * dc_max + sizeof(double) * upad4 + sizeof(float) * (size_t)dc_max * upad4 + 64;
  CKL(sb::rf_launch_stage3(a, upad_max, dc_max, upad4, bits_smem, idx->st));
  // sequential simulation over events touching overflow rows
  a.rec_cap = std::max<int64_t>(1, no * g);
  CK(idx->rf_rec.ensure((2 * sizeof(int32_t) + sizeof(uint64_t) + sizeof(int64_t)) * a.rec_cap + 64));
  a.rec_key = idx->rf_rec.as<uint64_t>();
  a.rec_next = reinterpret_cast<int64_t*>(a.rec_key + a.rec_cap);
  a.rec_tgt = reinterpret_cast<int32_t*>(a.rec_next + a.rec_cap);
  a.rec_cu = a.rec_tgt + a.rec_cap;
  CK(cudaMemsetAsync(a.rec_head, 0xFF, sizeof(int64_t) * n, idx->st));
  a.sim_wmax = (int)wmax;
  if (g > 255) return fail(SB_EARG, "reinforce: gamma must be below 256");
  if (sb::rf_simulate_smem(g, (int)wmax) > 227 * 1024)
    return fail(SB_ECUDA, "reinforce: simulation scratch exceeds shared memory");
  // Independent groups of O rows.  Two O rows interact only (a) when one is in the other's U
  // (an event between them, or a source row that changes), or (b) through the in-degree of a
  // node p both can hold, when p's in-degree can reach the safeguard: each O row lowers it at
  // most twice (p dropped, re-inserted by its own event, dropped again), so p with
  // in_deg0[p] - 2 * exposure[p] >= 2 passes every `in_deg >= 2` test in any order.  Unsafe
  // nodes tie every O row whose U holds them (and their own row) into one component.  The
  // components, packed into at most kMaxGroups groups by work, are simulated in parallel.
  {
    std::vector<int32_t> ul((size_t)uoff[no]), onodes(no), indeg(n), oidx(n);
    CK(cudaMemcpyAsync(ul.data(), a.u_list, sizeof(int32_t) * uoff[no], cudaMemcpyDeviceToHost, idx->st));
    CK(cudaMemcpyAsync(onodes.data(), a.o_nodes, sizeof(int32_t) * no, cudaMemcpyDeviceToHost, idx->st));
    CK(cudaMemcpyAsync(indeg.data(), a.in_deg, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, idx->st));
    CK(cudaMemcpyAsync(oidx.data(), a.o_idx, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, idx->st));
    CK(cudaStreamSynchronize(idx->st));
    std::vector<int32_t> expo(n, 0), first(n, -1), par(no);
    for (int64_t o = 0; o < no; ++o)
      for (int64_t t = uoff[o]; t < uoff[o + 1]; ++t) ++expo[ul[t]];
    for (int64_t o = 0; o < no; ++o) par[o] = (int32_t)o;
    auto find = [&](int32_t x) {
      while (par[x] != x) { par[x] = par[par[x]]; x = par[x]; }
      return x;
    };
    auto unite = [&](int32_t x, int32_t y) {
      x = find(x); y = find(y);
      if (x != y) par[std::max(x, y)] = std::min(x, y);
    };
    for (int64_t o = 0; o < no; ++o)
      for (int64_t t = uoff[o]; t < uoff[o + 1]; ++t) {
        const int32_t p = ul[t];
        if (oidx[p] >= 0) unite((int32_t)o, oidx[p]);
        if ((int64_t)indeg[p] - 2 * (int64_t)expo[p] < 2) {  // unsafe
          if (first[p] < 0) {
            first[p] = (int32_t)o;
            if (oidx[p] >= 0) unite((int32_t)o, oidx[p]);
          } else {
            unite((int32_t)o, first[p]);
          }
        }
      }
    std::vector<int64_t> cwork(no, 0);
    std::vector<int32_t> croot;
    for (int64_t o = 0; o < no; ++o) {
      const int32_t r = find((int32_t)o);
      if (cwork[r] == 0) croot.push_back(r);
      cwork[r] += usz[o] + 1;
    }
    constexpr int kMaxGroups = 1024;
    int ng = (int)std::min<size_t>(croot.size(), kMaxGroups);
    if (const char* e = getenv("SB_RF_GROUPS")) ng = std::max(1, std::min(ng, atoi(e)));
    // longest-processing-time packing of components into groups
    std::sort(croot.begin(), croot.end(), [&](int32_t x, int32_t y) { return cwork[x] > cwork[y]; });
    std::vector<int32_t> cgrp(no, 0);
    std::vector<std::pair<int64_t, int32_t>> heap;
    for (int32_t q = 0; q < ng; ++q) heap.push_back({0, q});
    auto cmp = [](const std::pair<int64_t, int32_t>& x, const std::pair<int64_t, int32_t>& y) {
      return x.first > y.first;
    };
    std::make_heap(heap.begin(), heap.end(), cmp);
    for (int32_t r : croot) {
      std::pop_heap(heap.begin(), heap.end(), cmp);
      cgrp[r] = heap.back().second;
      heap.back().first += cwork[r];
      std::push_heap(heap.begin(), heap.end(), cmp);
    }
    std::vector<int32_t> gofo(no);
    for (int64_t o = 0; o < no; ++o) gofo[o] = cgrp[find((int32_t)o)];
    a.ngroups = ng;
    a.bm_words = (n + 31) / 32;
    idx->last_rf_groups = ng;
    idx->last_rf_components = (int64_t)croot.size();
    // a group's dynamic events at one source are mirrors recorded into that (non-O) row, at
    // most |rev_j| <= gamma of them
    a.dyn_cap = g + 1;
    const size_t gb = sizeof(uint32_t) * (size_t)ng * a.bm_words;
    const size_t sim_bytes = (sizeof(uint64_t) + sizeof(int32_t)) * (size_t)ng * a.dyn_cap +
                             sizeof(int32_t) * (size_t)no + gb + 128;
    CK(idx->rf_sim.ensure(sim_bytes));
    char* sp = idx->rf_sim.as<char>();
    a.result = reinterpret_cast<int64_t*>(sp); sp += 4 * sizeof(int64_t);
    a.rec_count = a.result + 2;
    a.dyn = reinterpret_cast<uint64_t*>(sp); sp += sizeof(uint64_t) * (size_t)ng * a.dyn_cap;
    a.grp_bits = reinterpret_cast<uint32_t*>(sp); sp += gb;
    a.dyn_cu = reinterpret_cast<int32_t*>(sp); sp += sizeof(int32_t) * (size_t)ng * a.dyn_cap;
    a.grp_of_o = reinterpret_cast<int32_t*>(sp);
    CK(cudaMemsetAsync(a.result, 0, 4 * sizeof(int64_t), idx->st));
    CK(cudaMemcpyAsync(a.grp_of_o, gofo.data(), sizeof(int32_t) * no, cudaMemcpyHostToDevice, idx->st));
    CKL(sb::rf_launch_group_bits(a, idx->st));
  }
  CKL(sb::rf_launch_simulate(a, idx->st));
  int64_t res[3] = {0, 0, 0};
  CK(cudaMemcpyAsync(res, a.result, sizeof(res), cudaMemcpyDeviceToHost, idx->st));
  CK(cudaStreamSynchronize(idx->st));
  res[0] = std::min(res[2], a.rec_cap);  // records allocated
  if (res[1]) return fail(SB_ECUDA, "reinforce simulation invariant violated (code " + std::to_string(res[1]) + ")");
  // parallel part: insertions into rows that cannot overflow
  CK(idx->seg.ensure(sizeof(uint64_t) * n * g));
  a.apply_seg = idx->seg.as<uint64_t>();
  CKL(sb::rf_launch_apply(a, res[0], idx->scan_tmp.as<int64_t>(), idx->st));
  CKL(sb::launch_row_union_merge(a.ids, a.dists, a.counts, n, g, a.apply_off, a.apply_cnt,
                                 a.apply_seg, idx->st));
  idx->launches += 16;
  idx->last_overflow_rows = no;
  return SB_OK;
}

// reinforce_pass (_kernels.py:398-409); in_deg continues from sb_prune, else it is counted
static int reinforce_pass(sb_index* idx, double sigma, int64_t* overflow_rows) {
  const int64_t n = idx->n;
  const int g = idx->g;
  CK(idx->rev_cnt.ensure(sizeof(int64_t) * n));
  CK(idx->rev_off.ensure(sizeof(int64_t) * n));
  CK(idx->rev_cur.ensure(sizeof(int64_t) * n));
  CK(idx->in_deg.ensure(sizeof(int32_t) * n));
  CK(idx->scan_tmp.ensure(sizeof(int64_t) * sb::scan_tmp_slots(n)));
  CK(idx->small.ensure(64));
  if (!idx->have_indeg) {
    CKL(sb::launch_count_in_degrees(idx->ids.as<int32_t>(), idx->counts.as<int32_t>(), n, g,
                                    idx->in_deg.as<int32_t>(), nullptr, idx->st));
    idx->launches += 1;
  }
  unsigned long long* d_over = idx->small.as<unsigned long long>() + 4;
  CKL(sb::launch_reinforce_check(idx->ids.as<int32_t>(), idx->dists.as<float>(),
                                 idx->counts.as<int32_t>(), n, g, idx->rev_cnt.as<int64_t>(),
                                 d_over, idx->st));
  unsigned long long over = 0;
  CK(cudaMemcpyAsync(&over, d_over, sizeof(over), cudaMemcpyDeviceToHost, idx->st));
  CK(cudaStreamSynchronize(idx->st));
  if (overflow_rows) *overflow_rows = (int64_t)over;
  if (over == 0) {
    CK(idx->seg.ensure(sizeof(uint64_t) * n * g));
    CKL(sb::launch_symmetrize(idx->ids.as<int32_t>(), idx->dists.as<float>(),
                              idx->counts.as<int32_t>(), n, g, idx->rev_cnt.as<int64_t>(),
                              idx->rev_off.as<int64_t>(), idx->rev_cur.as<int64_t>(),
                              idx->seg.as<uint64_t>(), idx->scan_tmp.as<int64_t>(), idx->st));
    idx->launches += 6;
  } else {
    int r = reinforce_overflow(idx, sigma);
    if (r) return r;
  }
  CK(cudaStreamSynchronize(idx->st));
  idx->have_indeg = false;
  return SB_OK;
}

// one reconnect_islands sweep (_kernels.py:455-487) if some node has in-degree 0;
// *ran = 1 if the sweep ran
static int reconnect_sweep(sb_index* idx, double sigma, int* ran) {
  const int64_t n = idx->n;
  const int g = idx->g;
  CK(idx->in_deg.ensure(sizeof(int32_t) * n));
  CK(idx->small.ensure(64));
  int* d_min = reinterpret_cast<int*>(idx->small.as<unsigned long long>() + 5);
  CKL(sb::launch_count_in_degrees(idx->ids.as<int32_t>(), idx->counts.as<int32_t>(), n, g,
                                  idx->in_deg.as<int32_t>(), nullptr, idx->st));
  int big = 0x7FFFFFFF;
  CK(cudaMemcpyAsync(d_min, &big, sizeof(int), cudaMemcpyHostToDevice, idx->st));
  CKL(sb::launch_min_i32(idx->in_deg.as<int32_t>(), n, d_min, idx->st));
  int mn = 0;
  CK(cudaMemcpyAsync(&mn, d_min, sizeof(int), cudaMemcpyDeviceToHost, idx->st));
  CK(cudaStreamSynchronize(idx->st));
  idx->launches += 2;
  *ran = 0;
  if (mn >= 1) return SB_OK;
  if (getenv("SB_RC_DEBUG")) {
    std::vector<int32_t> deg(n), cnt(n), ids((size_t)n * g);
    cudaMemcpy(deg.data(), idx->in_deg.p, 4 * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(cnt.data(), idx->counts.p, 4 * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(ids.data(), idx->ids.p, 4 * (size_t)n * g, cudaMemcpyDeviceToHost);
    int64_t z = 0, zfull = 0, zdeg0 = 0, full = 0;
    for (int64_t v = 0; v < n; ++v) {
      full += cnt[v] >= g;
      if (deg[v] > 0) continue;
      ++z;
      if (cnt[v] == 0) { ++zdeg0; continue; }
      zfull += cnt[ids[(size_t)v * g]] >= g;
    }
    fprintf(stderr, "[rc] zero-in-degree %lld, first target full %lld, no out-edges %lld, full rows %lld\n",
            (long long)z, (long long)zfull, (long long)zdeg0, (long long)full);
  }
  CKL(sb::launch_reconnect(idx->F.as<float>(), idx->A.as<int32_t>(), idx->m, idx->l, g,
                           idx->ids.as<int32_t>(), idx->dists.as<float>(), idx->counts.as<int32_t>(),
                           idx->in_deg.as<int32_t>(), sigma, n, idx->st));
  idx->launches += 1;
  CK(cudaStreamSynchronize(idx->st));
  *ran = 1;
  return SB_OK;
}

int sb_reinforce_pass(sb_index* idx, double sigma, int64_t* overflow_rows) {
  if (idx) idx->graph_version++;
  if (!idx) return fail(SB_EARG, "idx is NULL");
  return reinforce_pass(idx, sigma, overflow_rows);
}

int sb_reconnect_islands(sb_index* idx, double sigma, int32_t* ran) {
  if (idx) idx->graph_version++;
  if (!idx) return fail(SB_EARG, "idx is NULL");
  int r = 0;
  int rc = reconnect_sweep(idx, sigma, &r);
  if (ran) *ran = r;
  return rc;
}

int sb_reinforce(sb_index* idx, double sigma, int64_t* overflow_rows, int32_t* sweeps_out) {
  if (idx) idx->graph_version++;
  if (!idx) return fail(SB_EARG, "idx is NULL");
  int r = reinforce_pass(idx, sigma, overflow_rows);
  if (r) return r;
  // reconnect sweeps with freshly counted in-degrees (graph.py:221-230)
  int sweeps = 0;
  for (int it = 0; it < 10; ++it) {
    int ran = 0;
    r = reconnect_sweep(idx, sigma, &ran);
    if (r) return r;
    if (!ran) break;
    ++sweeps;
  }
  if (sweeps_out) *sweeps_out = sweeps;
  return SB_OK;
}

// Attribute-grouped node order for the tensor-core top-k paths: a counting sort of the nodes by
// their attribute tuple (mixed-radix code; the node id when tuples are too many to group).
// Writes the sorted order to s_orig (n) and leaves each node's code in *d_code_out (fb_tmp).
static int node_order(sb_index* idx, int32_t* s_orig, int32_t** d_code_out) {
  const int64_t n = idx->n;
  const int l = idx->l;
  CK(idx->small.ensure(64));
  CK(idx->fb_tmp.ensure(sizeof(int32_t) * (2 * 8 + n + 2) + sizeof(int64_t) * 8));
  int32_t* d_lo = idx->fb_tmp.as<int32_t>();
  int32_t* d_hi = d_lo + 8;
  int32_t* d_code = d_hi + 8;
  int64_t* d_stride = reinterpret_cast<int64_t*>(d_code + n + (n & 1));
  std::vector<int32_t> hlo(8, 0x7FFFFFFF), hhi(8, (int32_t)0x80000000);
  CK(cudaMemcpyAsync(d_lo, hlo.data(), sizeof(int32_t) * 8, cudaMemcpyHostToDevice, idx->st));
  CK(cudaMemcpyAsync(d_hi, hhi.data(), sizeof(int32_t) * 8, cudaMemcpyHostToDevice, idx->st));
  CKL(sb::launch_tc_attr_range(idx->A.as<int32_t>(), n, l, d_lo, d_hi, idx->st));
  CK(cudaMemcpyAsync(hlo.data(), d_lo, sizeof(int32_t) * 8, cudaMemcpyDeviceToHost, idx->st));
  CK(cudaMemcpyAsync(hhi.data(), d_hi, sizeof(int32_t) * 8, cudaMemcpyDeviceToHost, idx->st));
  CK(cudaStreamSynchronize(idx->st));
  std::vector<int64_t> stride(8, 0);
  int64_t combos = 1;
  for (int u = l - 1; u >= 0; --u) {
    stride[u] = combos;
    combos *= (int64_t)hhi[u] - hlo[u] + 1;
    if (combos > ((int64_t)1 << 24)) break;
  }
  const int grouped = combos <= ((int64_t)1 << 24) ? 1 : 0;
  idx->code_grouped = grouped != 0;
  for (int u = 0; u < 8; ++u) {
    idx->code_lo[u] = u < l ? hlo[u] : 0;
    idx->code_stride[u] = u < l ? stride[u] : 0;
  }
  const int64_t bins = grouped ? combos : n;
  CK(cudaMemcpyAsync(d_stride, stride.data(), sizeof(int64_t) * 8, cudaMemcpyHostToDevice, idx->st));
  CK(idx->rev_cnt.ensure(sizeof(int64_t) * std::max<int64_t>(bins, n)));
  CK(idx->rev_off.ensure(sizeof(int64_t) * std::max<int64_t>(bins, n)));
  CK(idx->rev_cur.ensure(sizeof(int64_t) * std::max<int64_t>(bins, n)));
  CK(idx->scan_tmp.ensure(sizeof(int64_t) * sb::scan_tmp_slots(std::max<int64_t>(bins, n))));
  CK(cudaMemsetAsync(idx->rev_cnt.p, 0, sizeof(int64_t) * bins, idx->st));
  CK(cudaMemsetAsync(idx->rev_cur.p, 0, sizeof(int64_t) * bins, idx->st));
  CKL(sb::launch_tc_code(idx->A.as<int32_t>(), n, l, d_lo, d_stride, grouped, d_code,
             idx->rev_cnt.as<unsigned long long>(), idx->st));
  CKL(sb::exclusive_scan(idx->rev_cnt.as<int64_t>(), idx->rev_off.as<int64_t>(), bins,
             idx->scan_tmp.as<int64_t>(), idx->st));
  CKL(sb::launch_tc_scatter(d_code, n, idx->rev_off.as<int64_t>(),
            idx->rev_cur.as<unsigned long long>(), s_orig, idx->st));
  // skewed code sizes (one tuple far above the mean, e.g. Zipf codes) make the exhaustive
  // top-k walk node tiles strided across the splits (bf_tf.cu), so no CTA owns a hot region
  idx->tf_strided = 0;
  if (grouped && bins <= ((int64_t)1 << 22)) {
    std::vector<int64_t> hist(bins);
    CK(cudaMemcpyAsync(hist.data(), idx->rev_cnt.p, sizeof(int64_t) * bins, cudaMemcpyDeviceToHost, idx->st));
    CK(cudaStreamSynchronize(idx->st));
    int64_t mx = 0, used = 0;
    for (int64_t b = 0; b < bins; ++b) {
      mx = std::max(mx, hist[b]);
      used += hist[b] > 0;
    }
    idx->tf_strided = used > 1 && mx * used > 4 * n ? 1 : 0;
  }
  if (const char* e = getenv("SB_TF_STRIDE")) idx->tf_strided = atoi(e) != 0;
  *d_code_out = d_code;
  return SB_OK;
}

// ---------------------------------------------------------------------------
static int bf_run(sb_index* idx, sb::BfArgs& a, int kout, int64_t* out64, int32_t* out32,
                  double* outd, int* uncertain_host) {
  const int64_t q = a.q;
  const int groups = (int)((q + sb::bf_group_size() - 1) / sb::bf_group_size());
  // enough CTAs to fill the GPU twice over
  int splits = std::max(1, (2 * idx->sms + groups - 1) / groups);
  splits = (int)std::min<int64_t>(splits, std::max<int64_t>(1, idx->n / 256));
  a.splits = splits;
  CK(idx->bf_part_d.ensure(sizeof(double) * q * splits * a.k));
  CK(idx->bf_part_i.ensure(sizeof(uint32_t) * q * splits * a.k));
  a.part_d = idx->bf_part_d.as<double>();
  a.part_i = idx->bf_part_i.as<uint32_t>();
  CK(idx->small.ensure(64));
  int* d_unc = reinterpret_cast<int*>(idx->small.as<unsigned long long>() + 6);
  CK(cudaMemsetAsync(d_unc, 0, sizeof(int), idx->st));
  CKL(sb::launch_bf_partial(a, idx->st));
  CKL(sb::launch_bf_merge_k(a, kout, out64, out32, outd, d_unc, idx->st));
  idx->launches += 2;
  if (uncertain_host) CK(cudaMemcpyAsync(uncertain_host, d_unc, sizeof(int), cudaMemcpyDeviceToHost, idx->st));
  return SB_OK;
}

static int bf_sorted_run(sb_index* idx, const sb::BfArgs& a, int mode, int kout, int64_t* out64,
                         int32_t* out32, double* outd, int64_t* out_counts);

// TF32 filter + exact re-rank (bf_tf.cu).  Queries whose candidates overflow the buffers are
// recomputed on the exact fp64 kernel (bf_run); the count is reported by sb_bf_info.
static int bf_tf_run(sb_index* idx, const double* qf, const int64_t* qa, const int64_t* qmask,
                     int64_t q, int k, double alpha, double qmax_abs, int64_t* out_ids,
                     double* out_dists, int* unc_out) {
  const int64_t n = idx->n;
  const int m = idx->m, l = idx->l;
  const int dpad = sb::bf_tf_dpad(m);
  const double cE = sb::tf_margin(dpad);
  const int64_t npad = (n + sb::kTcNodePad - 1) / sb::kTcNodePad * sb::kTcNodePad;
  if (!idx->have_ft) {
    CK(idx->ft.ensure((size_t)4 * npad * dpad));
    CK(idx->ft_meta.ensure((size_t)4 * npad * (4 + l)));
    CK(cudaMemsetAsync(idx->ft.p, 0, (size_t)4 * npad * dpad, idx->st));
    CK(cudaMemsetAsync(idx->ft_meta.p, 0, (size_t)4 * npad * (4 + l), idx->st));
  }
  float* nxd = idx->ft_meta.as<float>();
  int32_t* s_code = reinterpret_cast<int32_t*>(nxd + npad);
  int32_t* s_orig = s_code + npad;
  int32_t* s_run = s_orig + npad;
  int32_t* s_attr = s_run + npad;
  if (!idx->have_ft) {
    int32_t* d_code = nullptr;
    int r = node_order(idx, s_orig, &d_code);
    if (r) return r;
    CKL(sb::launch_tf_gather(idx->F.as<float>(), idx->A.as<int32_t>(), d_code, s_orig, n, m, l, cE,
                             idx->ft.as<float>(), nxd, s_code, s_attr, idx->st));
    CKL(sb::launch_tf_runend(s_code, n, s_run, idx->st));
    idx->have_ft = true;
    idx->have_cand = false;  // rev_* scratch was reused
    idx->launches += 5;
  }
  // k > 32: two full passes (bf_tf.cu "large k"): the first builds every epilogue thread's
  // list of its 32 smallest upper keys, a select kernel takes the k-th smallest of all of a
  // query's lists as its bound, the second emits the candidates under that bound.  Needs
  // (threads per query) x 32 >= k; SB_TF_TWOPASS=0 keeps the single pass with shared-memory
  // lists.
  const int KRL = 32;
  bool twopass = k > KRL && sb::bf_tf_supported(m, l, KRL);
  if (const char* e = getenv("SB_TF_TWOPASS")) twopass = twopass && atoi(e) != 0;
  const int kshape = twopass ? KRL : k;
  int qblock = 128, hsegs = 2, ew = 8;
  sb::bf_tf_layout(m, l, kshape, &qblock, &hsegs, &ew);
  const int64_t qpad = (q + qblock - 1) / qblock * qblock;
  // node-range splits: whole waves of one CTA per SM, fewest splits within 3% of the best
  const int groups = (int)(qpad / qblock);
  const int64_t tiles = npad / 256;
  int splits = 1;
  {
    double best = 1e30;
    std::vector<double> cost(65, 1e30);
    // each epilogue thread should see many more than k nodes, or its list bound stays loose
    // and nearly every node is emitted: (tiles / splits) * 128 >= 16 k
    const int64_t smax = std::max<int64_t>(1, std::min<int64_t>(64, tiles * 128 / (16 * (int64_t)kshape)));
    for (int s2 = 1; s2 <= smax; ++s2) {
      const double waves = (double)((groups * s2 + idx->sms - 1) / idx->sms);
      cost[s2] = waves / s2;
      best = std::min(best, cost[s2]);
    }
    for (int s2 = 1; s2 <= 64; ++s2)
      if (cost[s2] <= best * 1.03) { splits = s2; break; }
    if (const char* e = getenv("SB_TF_SPLITS")) splits = std::max(1, atoi(e));
    // the union of a query's thread lists must hold k keys
    if (twopass) while (splits * hsegs * KRL < k && splits < 64) ++splits;
    if (twopass && splits * hsegs * KRL < k)  // (64 splits x 2 x 32 >= 4096 > every k here)
      return fail(SB_ECUDA, "two-pass top-k: too few thread lists for k");
  }
  // one candidate segment per epilogue thread of the grid; after the seed pass a thread emits
  // a few dozen candidates (full segments spill into the query's overflow area)
  const int64_t nthreads = (int64_t)groups * splits * 32 * ew;
  int cap = twopass ? 256 : std::max(256, 32 * k);
  while (cap > 64 && (double)nthreads * cap * 8.0 > 8e9) cap /= 2;
  if (const char* e = getenv("SB_TF_CAP")) cap = std::max(1, atoi(e));
  const int scap = k > 32 ? 4096 : 2048;  // survivors of the final bound the re-rank takes
  const int ocap = std::max(4096, 64 * k);  // per-query overflow area behind full segments
  // tq: Qt (qpad x dpad f32) | nqs | nqu | gthr | ovf | ovf_count | emitted total | ocnt (q) |
  //     cnt (q x segs)
  const size_t qt_bytes = (size_t)4 * qpad * dpad;
  CK(idx->tq.ensure(qt_bytes + (size_t)4 * 5 * q + 64 + (size_t)4 * nthreads));
  float* Qt = idx->tq.as<float>();
  float* nqs = reinterpret_cast<float*>(idx->tq.as<char>() + qt_bytes);
  float* nqu = nqs + q;
  int* gthr = reinterpret_cast<int*>(nqu + q);
  int* ovf = gthr + q;
  int* ovf_count = ovf + q;
  unsigned long long* emitted_total =
      reinterpret_cast<unsigned long long*>(reinterpret_cast<uintptr_t>(ovf_count + 2) & ~(uintptr_t)7);
  uint32_t* ocnt = reinterpret_cast<uint32_t*>(emitted_total + 2);
  uint32_t* cnt = ocnt + q;
  CK(idx->tcand.ensure(sizeof(uint64_t) * ((size_t)nthreads * cap + (size_t)q * ocap)));
  uint64_t* ocand = idx->tcand.as<uint64_t>() + (size_t)nthreads * cap;
  CK(cudaMemsetAsync(gthr, 0x7F, sizeof(int) * q, idx->st));  // 0x7F7F7F7F = 3.39e38f
  CK(cudaMemsetAsync(ovf, 0, reinterpret_cast<char*>(cnt) - reinterpret_cast<char*>(ovf), idx->st));
  // absolute slack for tf32 subnormal rounding and fp32 product underflow (negligible otherwise)
  const double tiny = dpad * std::ldexp(1.0, -120) * (1.0 + idx->fmax) * (1.0 + qmax_abs);
  CKL(sb::launch_tf_prep_queries(idx->qf.as<double>(), q, qpad, m, cE, tiny, Qt, nqs, nqu, idx->st));
  // seed pass (first tile of every range, bound only), then the full pass
  // seed pass: enough evenly spread tiles that every thread's list of k fills several times
  int seed_tiles = std::min(64, std::max(4, kshape / 2));
  if (const char* e = getenv("SB_TF_SEED")) seed_tiles = std::max(0, atoi(e));
  const int nl = splits * hsegs * KRL;  // list keys per query (two-pass)
  float* lists = nullptr;
  if (twopass) {
    CK(idx->tlists.ensure(sizeof(float) * (size_t)q * nl));
    lists = idx->tlists.as<float>();
  }
  CK(idx->bf_event(0));  // the tensor-core pass = seed + full launch(es)
  auto pass = [&](int seed, int bound_only, int fixed) {
    return sb::launch_bf_tf(idx->ft.as<float>(), nxd, s_code, s_orig, s_run, s_attr, Qt, nqs, nqu,
                            idx->bf_qa.as<int64_t>(), qmask ? idx->bf_qm.as<int64_t>() : nullptr, n, q,
                            m, l, kshape, splits, alpha, gthr, cnt, idx->tcand.as<uint64_t>(), cap,
                            ocnt, ocand, ocap, seed, idx->tf_strided, bound_only, fixed,
                            bound_only ? lists : nullptr, idx->st);
  };
  if (twopass) {
    // seed lists -> a first bound on the k-th key (the k-th smallest key of the union of the
    // threads' lists: k genuine upper keys of distinct nodes lie at or below it), the full
    // list pass under that bound, the tightened bound, the emission pass
    static const bool dbg = getenv("SB_TF_DEBUG") != nullptr;
    auto dump = [&](const char* what) {
      if (!dbg) return;
      std::vector<float> h(q);
      cudaMemcpyAsync(h.data(), gthr, sizeof(float) * q, cudaMemcpyDeviceToHost, idx->st);
      cudaStreamSynchronize(idx->st);
      std::vector<float> srt(h);
      std::sort(srt.begin(), srt.end());
      fprintf(stderr, "[tf] %s splits=%d nl=%d bound p10 %.4g p50 %.4g p90 %.4g max %.4g\n", what, splits, nl,
              srt[q / 10], srt[q / 2], srt[q * 9 / 10], srt[q - 1]);
    };
    if (idx->code_grouped && !(getenv("SB_TF_CODESEED") && atoi(getenv("SB_TF_CODESEED")) == 0)) {
      CKL(sb::launch_tf_code_seed(idx->F.as<float>(), idx->A.as<int32_t>(), s_code, s_orig, n, m, l,
                                  idx->qf.as<double>(), idx->bf_qa.as<int64_t>(),
                                  qmask ? idx->bf_qm.as<int64_t>() : nullptr, q, k, alpha,
                                  idx->code_lo, idx->code_stride, gthr, idx->st));
      idx->launches += 1;
      dump("code");
    }
    if (seed_tiles > 0) {
      CKL(pass(seed_tiles, 1, 0));
      CKL(sb::launch_tf_select(lists, q, nl, k, gthr, idx->st));
      idx->launches += 1;
      dump("seed");
    }
    CKL(pass(0, 1, 0));
    CKL(sb::launch_tf_select(lists, q, nl, k, gthr, idx->st));
    dump("full");
    CKL(pass(0, 0, 1));
    idx->launches += 2;
  } else if (seed_tiles > 0) {
    CKL(pass(seed_tiles, 0, 0));
    CKL(pass(0, 0, 0));
  } else {
    CKL(pass(0, 0, 0));
  }
  CK(idx->bf_event(1));
  idx->bf_ev_valid = true;
  CKL(sb::launch_tf_refine(idx->F.as<float>(), idx->A.as<int32_t>(), m, l, idx->qf.as<double>(),
                           idx->bf_qa.as<int64_t>(), qmask ? idx->bf_qm.as<int64_t>() : nullptr, q,
                           k, alpha, cnt, idx->tcand.as<uint64_t>(), splits, hsegs, qblock, ew, cap, ocnt, ocand,
                           ocap, gthr, scap,
                           idx->out_ids.as<int64_t>(), idx->out_dists.as<double>(), ovf, ovf_count,
                           emitted_total, idx->st));
  idx->launches += 4;
  int novf = 0;
  CK(cudaMemcpyAsync(&novf, ovf_count, sizeof(int), cudaMemcpyDeviceToHost, idx->st));
  CK(cudaMemcpyAsync(out_ids, idx->out_ids.p, sizeof(int64_t) * q * k, cudaMemcpyDeviceToHost, idx->st));
  if (out_dists) CK(cudaMemcpyAsync(out_dists, idx->out_dists.p, sizeof(double) * q * k, cudaMemcpyDeviceToHost, idx->st));
  unsigned long long total = 0;
  CK(cudaMemcpyAsync(&total, emitted_total, sizeof(total), cudaMemcpyDeviceToHost, idx->st));
  CK(cudaStreamSynchronize(idx->st));
  idx->last_bf_cands = (int64_t)total;
  idx->last_bf_fallback = novf;
  idx->last_bf_tc = true;
  idx->last_bf_path = 2;
  *unc_out = 0;
  if (novf > 0) {
    // exact fp64 path for the flagged queries
    std::vector<int> hovf(q);
    CK(cudaMemcpy(hovf.data(), ovf, sizeof(int) * q, cudaMemcpyDeviceToHost));
    std::vector<int64_t> sel;
    for (int64_t i = 0; i < q; ++i)
      if (hovf[i]) sel.push_back(i);
    const int64_t s = (int64_t)sel.size();
    std::vector<double> sqf((size_t)s * m);
    std::vector<int64_t> sqa((size_t)s * l), sqm((size_t)s * l);
    for (int64_t j = 0; j < s; ++j) {
      memcpy(&sqf[j * m], qf + sel[j] * m, sizeof(double) * m);
      memcpy(&sqa[j * l], qa + sel[j] * l, sizeof(int64_t) * l);
      if (qmask) memcpy(&sqm[j * l], qmask + sel[j] * l, sizeof(int64_t) * l);
    }
    const size_t sub = sizeof(double) * s * m + 2 * sizeof(int64_t) * s * l + (sizeof(int64_t) + sizeof(double)) * s * k;
    CK(idx->tovf.ensure(sub + 64));
    double* d_qf = idx->tovf.as<double>();
    int64_t* d_qa = reinterpret_cast<int64_t*>(d_qf + s * m);
    int64_t* d_qm = d_qa + s * l;
    int64_t* d_ids = d_qm + s * l;
    double* d_d = reinterpret_cast<double*>(d_ids + s * k);
    CK(cudaMemcpyAsync(d_qf, sqf.data(), sizeof(double) * s * m, cudaMemcpyHostToDevice, idx->st));
    CK(cudaMemcpyAsync(d_qa, sqa.data(), sizeof(int64_t) * s * l, cudaMemcpyHostToDevice, idx->st));
    if (qmask) CK(cudaMemcpyAsync(d_qm, sqm.data(), sizeof(int64_t) * s * l, cudaMemcpyHostToDevice, idx->st));
    sb::BfArgs a{};
    a.F = idx->F.as<float>(); a.A = idx->A.as<int32_t>(); a.n = n; a.m = m; a.l = l;
    a.qf = d_qf; a.qa = d_qa; a.qmask = qmask ? d_qm : nullptr; a.q = s;
    a.k = (int)std::min<int64_t>(n, k + 16); a.alpha = alpha;
    int unc = 0;
    // the tiled fp64 kernel while its per-query lists fit shared memory, else the full sort
    int r = sb::bf_partial_smem(a.k) <= (size_t)227 * 1024
                ? bf_run(idx, a, k, d_ids, nullptr, d_d, &unc)
                : bf_sorted_run(idx, a, sb::kBfSortQuery, k, d_ids, nullptr, d_d, nullptr);
    if (r) return r;
    std::vector<int64_t> hi((size_t)s * k);
    std::vector<double> hd((size_t)s * k);
    CK(cudaMemcpyAsync(hi.data(), d_ids, sizeof(int64_t) * s * k, cudaMemcpyDeviceToHost, idx->st));
    CK(cudaMemcpyAsync(hd.data(), d_d, sizeof(double) * s * k, cudaMemcpyDeviceToHost, idx->st));
    CK(cudaStreamSynchronize(idx->st));
    for (int64_t j = 0; j < s; ++j) {
      memcpy(out_ids + sel[j] * k, &hi[j * k], sizeof(int64_t) * k);
      if (out_dists) memcpy(out_dists + sel[j] * k, &hd[j * k], sizeof(double) * k);
    }
    *unc_out = unc;
  }
  return SB_OK;
}

// Any k: exact keys of every node, one segmented radix sort per chunk of queries
// (bf_sort.cu).  a.q rows of a.self_ids / a.qf+a.qa(+a.qmask) are device-resident.
static int bf_sorted_run(sb_index* idx, const sb::BfArgs& a, int mode, int kout, int64_t* out64,
                         int32_t* out32, double* outd, int64_t* out_counts) {
  const int64_t chunk = sb::bf_sort_chunk(idx->n, a.q);
  const size_t bytes = sb::bf_sort_scratch_bytes(idx->n, chunk);
  CK(idx->bf_sort.ensure(bytes));
  for (int64_t q0 = 0; q0 < a.q; q0 += chunk) {
    const int64_t b = std::min<int64_t>(chunk, a.q - q0);
    CKL(sb::launch_bf_sorted(a, mode, q0, b, kout, idx->bf_sort.p, bytes, out64, out32, outd,
                             out_counts, idx->st));
    idx->launches += 4;
  }
  return SB_OK;
}

int sb_bf_topk_nodes(sb_index* idx, const int64_t* sample_ids, int64_t s, int32_t k,
                     double inv_alpha, int32_t* out_ids) {
  if (!idx || !sample_ids || !out_ids) return fail(SB_EARG, "NULL argument");
  if (k < 1) return fail(SB_EARG, "k must be >= 1");
  if (s <= 0) return SB_OK;
  if (k > 1024) {  // beyond the tiled kernel's shared-memory lists: full sort per sample
    CK(idx->bf_self.ensure(sizeof(int64_t) * s));
    CK(idx->bf_out32.ensure(sizeof(int32_t) * s * k));
    CK(cudaMemcpyAsync(idx->bf_self.p, sample_ids, sizeof(int64_t) * s, cudaMemcpyHostToDevice, idx->st));
    sb::BfArgs a{};
    a.F = idx->F.as<float>(); a.A = idx->A.as<int32_t>(); a.n = idx->n; a.m = idx->m; a.l = idx->l;
    a.self_ids = idx->bf_self.as<int64_t>(); a.q = s; a.k = k; a.inv_alpha = inv_alpha;
    int r = bf_sorted_run(idx, a, sb::kBfSortNode, k, nullptr, idx->bf_out32.as<int32_t>(), nullptr, nullptr);
    if (r) return r;
    CK(cudaMemcpyAsync(out_ids, idx->bf_out32.p, sizeof(int32_t) * s * k, cudaMemcpyDeviceToHost, idx->st));
    CK(cudaStreamSynchronize(idx->st));
    return SB_OK;
  }
  CK(idx->bf_self.ensure(sizeof(int64_t) * s));
  CK(idx->bf_out32.ensure(sizeof(int32_t) * s * k));
  CK(cudaMemcpyAsync(idx->bf_self.p, sample_ids, sizeof(int64_t) * s, cudaMemcpyHostToDevice, idx->st));
  sb::BfArgs a{};
  a.F = idx->F.as<float>(); a.A = idx->A.as<int32_t>(); a.n = idx->n; a.m = idx->m; a.l = idx->l;
  a.self_ids = idx->bf_self.as<int64_t>(); a.q = s; a.k = k; a.inv_alpha = inv_alpha;
  int r = bf_run(idx, a, k, nullptr, idx->bf_out32.as<int32_t>(), nullptr, nullptr);
  if (r) return r;
  CK(cudaMemcpyAsync(out_ids, idx->bf_out32.p, sizeof(int32_t) * s * k, cudaMemcpyDeviceToHost, idx->st));
  CK(cudaStreamSynchronize(idx->st));
  return SB_OK;
}

int sb_bf_topk_queries(sb_index* idx, const double* qf, const int64_t* qa, const int64_t* qmask,
                       int64_t q, int32_t k, double alpha, int64_t* out_ids, double* out_dists,
                       int32_t* uncertain) {
  if (!idx || !qf || !qa || !out_ids) return fail(SB_EARG, "NULL argument");
  if (k < 1 || k > idx->n) return fail(SB_EARG, "k must be in [1, n]");
  if (q <= 0) return SB_OK;
  const int extra = 16;
  int kk = (int)std::min<int64_t>(idx->n, k + extra);
  CK(idx->qf.ensure(sizeof(double) * q * idx->m));
  CK(idx->bf_qa.ensure(sizeof(int64_t) * q * idx->l));
  CK(idx->bf_qm.ensure(sizeof(int64_t) * q * idx->l));
  CK(idx->out_ids.ensure(sizeof(int64_t) * q * k));
  CK(idx->out_dists.ensure(sizeof(double) * q * k));
  CK(cudaMemcpyAsync(idx->qf.p, qf, sizeof(double) * q * idx->m, cudaMemcpyHostToDevice, idx->st));
  CK(cudaMemcpyAsync(idx->bf_qa.p, qa, sizeof(int64_t) * q * idx->l, cudaMemcpyHostToDevice, idx->st));
  if (qmask) CK(cudaMemcpyAsync(idx->bf_qm.p, qmask, sizeof(int64_t) * q * idx->l, cudaMemcpyHostToDevice, idx->st));
  sb::BfArgs a{};
  a.F = idx->F.as<float>(); a.A = idx->A.as<int32_t>(); a.n = idx->n; a.m = idx->m; a.l = idx->l;
  a.qf = idx->qf.as<double>(); a.qa = idx->bf_qa.as<int64_t>();
  a.qmask = qmask ? idx->bf_qm.as<int64_t>() : nullptr; a.q = q; a.k = kk; a.alpha = alpha;
  int unc = 0;
  if (k > 1000) {  // beyond every tiled kernel's lists: exact keys + full sort (bf_sort.cu)
    int r = bf_sorted_run(idx, a, sb::kBfSortQuery, k, idx->out_ids.as<int64_t>(), nullptr,
                          idx->out_dists.as<double>(), nullptr);
    if (r) return r;
    idx->bf_ev_valid = false;
    idx->last_bf_tc = false;
    idx->last_bf_path = 3;
    CK(cudaMemcpyAsync(out_ids, idx->out_ids.p, sizeof(int64_t) * q * k, cudaMemcpyDeviceToHost, idx->st));
    if (out_dists) CK(cudaMemcpyAsync(out_dists, idx->out_dists.p, sizeof(double) * q * k, cudaMemcpyDeviceToHost, idx->st));
    CK(cudaStreamSynchronize(idx->st));
    if (uncertain) *uncertain = 0;
    return SB_OK;
  }
  // tensor-core path: integer features and queries, |values| <= 256 (exact in bf16), every
  // partial dot product below 2^24 (exact in the fp32 accumulator)
  // (integer data: U is exact whatever the summation order, so lists of exactly k suffice)
  bool tc = idx->int_exact && idx->fmax <= 256.0 && idx->m <= 255 && !idx->force_sequential &&
            sb::bf_tc_supported(2 * idx->m, idx->l, k);
  if (const char* e = getenv("SB_BF_TC")) tc = tc && atoi(e) != 0;
  double qmin = 0.0, qmax = 0.0;
  for (int64_t i = 0; tc && i < q * idx->m; ++i) {
    double v = qf[i];
    tc = v == std::rint(v) && std::fabs(v) <= 256.0;
    qmin = std::min(qmin, v);
    qmax = std::max(qmax, v);
  }
  // Fold |x|^2 into the MMA (16 more K columns) when y = 2 x.q - |x|^2 and all its partial
  // sums stay exact integers below 2^24: non-negative data bounds every partial sum by
  // max(sum 2qx, |x|^2); mixed signs by 3 m f^2.
  bool fold = false;
  if (tc) {
    const double m = idx->m, fx = idx->fmax, fq = std::max(std::fabs(qmin), std::fabs(qmax));
    const bool nonneg = idx->flo >= 0.f && qmin >= 0.0;
    const double bound = nonneg ? std::max(2.0 * m * fx * fq, m * fx * fx)
                                : 3.0 * m * std::max(fx, fq) * std::max(fx, fq);
    fold = bound < 16777216.0;
    // measured neutral on cfg 2 (the epilogue is bound by barrier waits, not the filter):
    // opt in with SB_BF_FOLD=1
    { const char* e = getenv("SB_BF_FOLD"); fold = fold && e && atoi(e) != 0; }
    if (fold && !sb::bf_tc_supported(2 * (idx->m + 16), idx->l, k)) fold = false;
  }
  // u8 operands (tcgen05 kind::i8, exact int32 dot products) for data and queries in [0, 255]
  bool u8 = tc && idx->flo >= 0.f && idx->fhi <= 255.f && qmin >= 0.0 && qmax <= 255.0 &&
            idx->m % 32 == 0 && sb::bf_tc_supported(idx->m, idx->l, k);
  if (const char* e = getenv("SB_BF_U8")) u8 = u8 && atoi(e) != 0;
  if (u8) fold = false;
  const int mk = fold ? idx->m + 16 : idx->m;
  const int esz = u8 ? 1 : 2;  // operand bytes per element
  // other data: TF32 tensor-core filter with a certified bound + exact fp64 re-rank (bf_tf.cu)
  double qmax_abs = 0.0;
  bool tf = !tc && !idx->force_sequential && sb::bf_tf_supported(idx->m, idx->l, std::min(k, 32)) &&
            idx->fmax < 1e15;
  for (int64_t i = 0; tf && i < q * idx->m; ++i) {
    const double v = std::fabs(qf[i]);
    tf = v < 1e15;  // also rejects NaN
    qmax_abs = std::max(qmax_abs, v);
  }
  if (const char* e = getenv("SB_BF_TF")) tf = tf && atoi(e) != 0;
  if (const char* e = getenv("SB_BF_TC")) tf = tf && atoi(e) != 0;  // no tensor cores at all
  if (tc) {
    kk = k;
    a.k = kk;
    const int64_t n = idx->n;
    const int64_t npad = (n + sb::kTcNodePad - 1) / sb::kTcNodePad * sb::kTcNodePad;
    if (!idx->have_fb || idx->fb_mk != mk * esz) {
      // attribute-grouped node order: counting sort by the attribute tuple
      const int l = idx->l;
      // padded, zero-filled: every tile the kernel copies lies inside the buffers
      CK(idx->fb.ensure((size_t)esz * npad * mk));
      CK(idx->fb_norm.ensure(sizeof(int32_t) * npad * (3 + l)));  // nx | code | orig | attrs
      CK(cudaMemsetAsync(idx->fb.p, 0, (size_t)esz * npad * mk, idx->st));
      CK(cudaMemsetAsync(idx->fb_norm.p, 0, sizeof(int32_t) * npad * (3 + l), idx->st));
      int32_t* s_nx = idx->fb_norm.as<int32_t>();
      int32_t* s_code = s_nx + npad;
      int32_t* s_orig = s_code + npad;
      int32_t* s_attr = s_orig + npad;
      int32_t* d_code = nullptr;
      { int r = node_order(idx, s_orig, &d_code); if (r) return r; }
      if (u8) {
        // |x|^2 order inside each tuple + per-chunk {min |x|^2, code} records (bf_tc.cu)
        CK(idx->fb_scratch.ensure(sb::tc_norm_order_scratch(n)));
        CKL(sb::launch_tc_norm_order(idx->F.as<float>(), n, idx->m, d_code, s_orig, idx->fb_scratch.p, idx->st));
        CKL(sb::launch_tc_gather_u8(idx->F.as<float>(), idx->A.as<int32_t>(), d_code, s_orig, n,
                                    idx->m, l, idx->fb.p, s_nx, s_code, s_attr, idx->st));
        CK(idx->fb_cmeta.ensure(sizeof(int32_t) * 2 * (size_t)(npad / 16)));
        CKL(sb::launch_tc_chunk_meta(s_nx, s_code, n, npad, idx->fb_cmeta.p, idx->st));
        idx->fb_scratch.release();
      } else {
        CKL(sb::launch_tc_gather(idx->F.as<float>(), idx->A.as<int32_t>(), d_code, s_orig, n,
                                 idx->m, mk, l, idx->fb.p, s_nx, s_code, s_attr, idx->st));
      }
      idx->have_fb = true;
      idx->fb_mk = mk * esz;
      idx->have_cand = false;  // rev_* scratch was reused
      idx->launches += 6;
    }
    const int64_t qpad = (q + 127) / 128 * 128;
    CK(idx->qb.ensure((size_t)esz * qpad * mk + 2 * sizeof(int32_t) * q + 64));
    int32_t* d_nq = reinterpret_cast<int32_t*>(idx->qb.as<char>() + (size_t)esz * qpad * mk);
    int32_t* d_gthr = d_nq + q;  // per-query shared bound, 0x7F7F7F7F = 3.39e38f
    CK(cudaMemsetAsync(d_gthr, 0x7F, sizeof(int32_t) * q, idx->st));
    if (u8)
      CKL(sb::launch_bf_tc_prep_queries_u8(idx->qf.as<double>(), q, idx->m, idx->qb.p, d_nq, idx->st));
    else
      CKL(sb::launch_bf_tc_prep_queries(idx->qf.as<double>(), q, idx->m, mk, idx->qb.p, d_nq, idx->st));
    // split the node range so that whole waves of CTAs are busy: minimise waves / splits
    const int groups = (int)((q + 127) / 128);
    int splits = 1;
    double best = 1e30;
    const int slots = idx->sms * sb::bf_tc_ctas_per_sm(mk * esz, idx->l, kk);
    for (int s2 = 1; s2 <= 8 && (int64_t)s2 * 256 <= n; ++s2) {
      double waves = (double)((groups * s2 + slots - 1) / slots);
      double cost = waves / s2;
      if (cost < best - 1e-9) { best = cost; splits = s2; }
    }
    a.splits = 2 * splits;  // each CTA emits two partial lists per query (column halves)
    CK(idx->bf_part_d.ensure(sizeof(double) * q * a.splits * kk));
    CK(idx->bf_part_i.ensure(sizeof(uint32_t) * q * a.splits * kk));
    a.part_d = idx->bf_part_d.as<double>();
    a.part_i = idx->bf_part_i.as<uint32_t>();
    CK(idx->small.ensure(64));
    int* d_unc = reinterpret_cast<int*>(idx->small.as<unsigned long long>() + 6);
    CK(cudaMemsetAsync(d_unc, 0, sizeof(int), idx->st));
    {
      int32_t* s_nx = idx->fb_norm.as<int32_t>();
      CK(idx->bf_event(0));
      CKL(sb::launch_bf_tc(idx->fb.p, s_nx, s_nx + 3 * npad, s_nx + npad, s_nx + 2 * npad, idx->qb.p,
                           d_nq, a.qa, a.qmask, n, q, mk, idx->l, kk, splits, alpha, a.part_d,
                           a.part_i, d_gthr, fold ? 1 : 0, u8 ? 1 : 0, idx->fb_cmeta.p, idx->st));
      CK(idx->bf_event(1));
      idx->bf_ev_valid = true;
    }
    CKL(sb::launch_bf_merge_k(a, k, idx->out_ids.as<int64_t>(), nullptr, idx->out_dists.as<double>(),
                              d_unc, idx->st));
    CK(cudaMemcpyAsync(&unc, d_unc, sizeof(int), cudaMemcpyDeviceToHost, idx->st));
    idx->launches += 3;
    idx->last_bf_tc = true;
    idx->last_bf_path = 1;
  } else if (tf) {
    int r = bf_tf_run(idx, qf, qa, qmask, q, k, alpha, qmax_abs, out_ids, out_dists, &unc);
    if (r) return r;
    if (uncertain) *uncertain = unc;
    return SB_OK;
  } else {
    int r = sb::bf_partial_smem(a.k) <= (size_t)227 * 1024
                ? bf_run(idx, a, k, idx->out_ids.as<int64_t>(), nullptr, idx->out_dists.as<double>(), &unc)
                : bf_sorted_run(idx, a, sb::kBfSortQuery, k, idx->out_ids.as<int64_t>(), nullptr,
                                idx->out_dists.as<double>(), nullptr);
    if (r) return r;
    idx->bf_ev_valid = false;
    idx->last_bf_tc = false;
    idx->last_bf_path = 0;
  }
  CK(cudaMemcpyAsync(out_ids, idx->out_ids.p, sizeof(int64_t) * q * k, cudaMemcpyDeviceToHost, idx->st));
  if (out_dists) CK(cudaMemcpyAsync(out_dists, idx->out_dists.p, sizeof(double) * q * k, cudaMemcpyDeviceToHost, idx->st));
  CK(cudaStreamSynchronize(idx->st));
  if (uncertain) *uncertain = unc;
  return SB_OK;
}

// oracle_hybrid_groundtruth (evaluate.py:58-77) for q queries: nodes whose (masked) attribute
// Manhattan distance to the query is 0, ranked by pure feature distance (NumPy pairwise order),
// ties by id; out_ids q x k padded with -1, out_counts[i] = min(k, matches of query i).
int sb_hybrid_groundtruth(sb_index* idx, const double* qf, const int64_t* qa, const int64_t* qmask,
                          int64_t q, int32_t k, int64_t* out_ids, double* out_dists,
                          int64_t* out_counts) {
  if (!idx || !qf || !qa || !out_ids || !out_counts) return fail(SB_EARG, "NULL argument");
  if (k < 1) return fail(SB_EARG, "k must be >= 1");
  if (q <= 0) return SB_OK;
  const int64_t kk = std::min<int64_t>(k, idx->n);
  CK(idx->qf.ensure(sizeof(double) * q * idx->m));
  CK(idx->bf_qa.ensure(sizeof(int64_t) * q * idx->l));
  CK(idx->bf_qm.ensure(sizeof(int64_t) * q * idx->l));
  CK(idx->out_ids.ensure(sizeof(int64_t) * q * k));
  CK(idx->out_dists.ensure(sizeof(double) * q * k));
  CK(idx->stats.ensure(sizeof(int64_t) * q));
  CK(cudaMemcpyAsync(idx->qf.p, qf, sizeof(double) * q * idx->m, cudaMemcpyHostToDevice, idx->st));
  CK(cudaMemcpyAsync(idx->bf_qa.p, qa, sizeof(int64_t) * q * idx->l, cudaMemcpyHostToDevice, idx->st));
  if (qmask) CK(cudaMemcpyAsync(idx->bf_qm.p, qmask, sizeof(int64_t) * q * idx->l, cudaMemcpyHostToDevice, idx->st));
  if (kk < k) {  // k > n: the tail past n stays -1 / +inf
    CK(cudaMemsetAsync(idx->out_ids.p, 0xFF, sizeof(int64_t) * q * k, idx->st));
  }
  sb::BfArgs a{};
  a.F = idx->F.as<float>(); a.A = idx->A.as<int32_t>(); a.n = idx->n; a.m = idx->m; a.l = idx->l;
  a.qf = idx->qf.as<double>(); a.qa = idx->bf_qa.as<int64_t>();
  a.qmask = qmask ? idx->bf_qm.as<int64_t>() : nullptr; a.q = q; a.k = (int)kk;
  int r = bf_sorted_run(idx, a, sb::kBfSortHybrid, k, idx->out_ids.as<int64_t>(), nullptr,
                        idx->out_dists.as<double>(), idx->stats.as<int64_t>());
  if (r) return r;
  CK(cudaMemcpyAsync(out_ids, idx->out_ids.p, sizeof(int64_t) * q * k, cudaMemcpyDeviceToHost, idx->st));
  if (out_dists) CK(cudaMemcpyAsync(out_dists, idx->out_dists.p, sizeof(double) * q * k, cudaMemcpyDeviceToHost, idx->st));
  CK(cudaMemcpyAsync(out_counts, idx->stats.p, sizeof(int64_t) * q, cudaMemcpyDeviceToHost, idx->st));
  CK(cudaStreamSynchronize(idx->st));
  return SB_OK;
}

// ---------------------------------------------------------------------------
int sb_entry_points(int64_t n, int32_t k, uint64_t seed, int64_t qi0, int64_t q, int64_t* out) {
  if (!out) return fail(SB_EARG, "out is NULL");
  if (k < 1 || k > n) return fail(SB_EARG, "k must be in [1, n]");
  std::vector<int64_t> scratch(sbrng::choice_scratch_slots(n, k));
  for (int64_t i = 0; i < q; ++i)
    sbrng::entry_points(n, k, seed, (uint64_t)(qi0 + i), out + i * k, scratch.data());
  return SB_OK;
}

int sb_entry_points_device(int64_t n, int32_t k, uint64_t seed, int64_t qi0, int64_t q, int64_t* out) {
  if (!out) return fail(SB_EARG, "out is NULL");
  if (k < 1 || k > n) return fail(SB_EARG, "k must be in [1, n]");
  if (q <= 0) return SB_OK;
  const uint64_t slots = sbrng::choice_scratch_slots(n, k);
  int64_t* d_out = nullptr;
  int64_t* d_scr = nullptr;
  CK(cudaMalloc(&d_out, sizeof(int64_t) * (size_t)q * k));
  cudaError_t e = cudaMalloc(&d_scr, sizeof(int64_t) * slots * (size_t)q);
  if (e != cudaSuccess) { cudaFree(d_out); return cuda_fail(e, "cudaMalloc(scratch)"); }
  int r = sb::launch_entry_points(n, k, seed, qi0, q, d_out, d_scr, slots, 0);
  if (r == 0) r = (int)cudaMemcpy(out, d_out, sizeof(int64_t) * (size_t)q * k, cudaMemcpyDeviceToHost);
  cudaFree(d_out);
  cudaFree(d_scr);
  if (r) return cuda_fail((cudaError_t)r, "entry points on the device");
  return SB_OK;
}

// The routing layout (route.cu "routing layout"): a locality order of the nodes and the
// features, attributes and adjacency renumbered into it.  Rebuilt when the adjacency changed.
static bool relabel_enabled() {
  const char* e = getenv("SB_ROUTE_RELABEL");
  return e ? atoi(e) != 0 : true;
}

static int route_layout(sb_index* idx) {
  if (idx->rl_version == idx->graph_version) return SB_OK;
  const int64_t n = idx->n;
  const int m = idx->m, l = idx->l, g = idx->g;
  CK(idx->rl_perm.ensure(sizeof(int32_t) * 2 * (size_t)n));
  int32_t* perm = idx->rl_perm.as<int32_t>();
  int32_t* inv = perm + n;
  const size_t sb_bytes = sb::route_order_scratch_bytes(n);
  CK(idx->rl_tmp.ensure(sb_bytes));
  CKL(sb::launch_route_order(idx->F.as<float>(), n, m, perm, inv, idx->rl_tmp.p, sb_bytes, idx->st));
  CK(idx->rl_F.ensure(sizeof(float) * (size_t)n * m));
  CK(idx->rl_A.ensure(sizeof(int32_t) * (size_t)n * l));
  CK(idx->rl_ids.ensure(sizeof(int32_t) * (size_t)n * g));
  CK(idx->rl_counts.ensure(sizeof(int32_t) * (size_t)n));
  CKL(sb::launch_permute_rows_f32(idx->F.as<float>(), n, m, perm, idx->rl_F.as<float>(), idx->st));
  CKL(sb::launch_permute_rows_i32(idx->A.as<int32_t>(), n, l, perm, idx->rl_A.as<int32_t>(), idx->st));
  CKL(sb::launch_relabel_adjacency(idx->ids.as<int32_t>(), idx->counts.as<int32_t>(), n, g, perm, inv,
                                   idx->rl_ids.as<int32_t>(), idx->rl_counts.as<int32_t>(), idx->st));
  idx->rl_tmp.release();
  idx->rl_have_f8 = false;
  idx->rl_version = idx->graph_version;
  idx->launches += 7;
  return SB_OK;
}

// u8 copy (+ exact norms) of `F` into `buf` once; returns the norms pointer
static int ensure_u8(sb_index* idx, const float* F, DBuf& buf, bool& have) {
  const int64_t n = idx->n;
  const size_t fbytes = (size_t)n * idx->m;
  if (!have) {
    CK(buf.ensure(fbytes + 256 + sizeof(int32_t) * (size_t)n));
    CKL(sb::launch_pack_u8(F, n, idx->m, buf.as<uint8_t>(),
                           reinterpret_cast<int32_t*>(buf.as<uint8_t>() + ((fbytes + 255) & ~(size_t)255)),
                           idx->st));
    have = true;
    idx->launches += 1;
  }
  return SB_OK;
}

static bool u8_eligible(const sb_index* idx) {
  const char* f32env = getenv("SB_ROUTE_F32");
  const bool f32_want = f32env ? atoi(f32env) != 0 : true;
  const char* u8env = getenv("SB_ROUTE_U8");
  const bool want = u8env ? atoi(u8env) != 0 : true;
  return want && f32_want && idx->int_exact && !idx->force_sequential && idx->flo >= 0.f &&
         idx->fhi <= 255.f && idx->m % 16 == 0 && idx->m <= 512;
}

int sb_route_prepare(sb_index* idx) {
  if (!idx) return fail(SB_EARG, "idx is NULL");
  if (relabel_enabled()) {
    int r = route_layout(idx);
    if (r) return r;
    if (u8_eligible(idx)) {
      r = ensure_u8(idx, idx->rl_F.as<float>(), idx->rl_f8, idx->rl_have_f8);
      if (r) return r;
    }
  } else if (u8_eligible(idx)) {
    int r = ensure_u8(idx, idx->F.as<float>(), idx->f8, idx->have_f8);
    if (r) return r;
  }
  CK(cudaStreamSynchronize(idx->st));
  return SB_OK;
}

// entry points (router.py:42-45) of queries qi0 .. qi0 + q - 1 into idx->entries, on the
// device (one thread per query), on the handle's stream
static int gen_entries(sb_index* idx, int64_t q, int32_t k, uint64_t seed, int64_t qi0) {
  const int64_t n = idx->n;
  uint64_t slots = sbrng::choice_scratch_slots(n, k);
  CK(idx->entries.ensure(sizeof(int64_t) * q * k));
  // bound the RNG scratch: draw in slices
  int64_t slice = std::max<int64_t>(1, std::min<int64_t>(q, (int64_t)((1ull << 30) / (slots * 8))));
  CK(idx->ent_scratch.ensure(sizeof(int64_t) * slots * slice));
  for (int64_t b = 0; b < q; b += slice) {
    int64_t c = std::min(slice, q - b);
    CKL(sb::launch_entry_points(n, k, seed, qi0 + b, c, idx->entries.as<int64_t>() + b * k,
                                idx->ent_scratch.as<int64_t>(), slots, idx->st));
    idx->launches += 1;
  }
  return SB_OK;
}

static int route_dev(sb_index* idx, const double* qf, const double* qa, const double* qm, int64_t q,
                     int32_t k, int32_t p, int32_t use_coarse, const int64_t* entries,
                     uint64_t seed, int64_t qi0, double inv_alpha, int64_t* out_ids,
                     double* out_dists, int64_t* out_stats) {
  if (k < 1 || k > idx->n) return fail(SB_EARG, "k must be in [1, n]");
  if (p < 1 || p > k) return fail(SB_EARG, "pioneer_size must be in [1, k]");
  if (k > (1 << 18)) return fail(SB_EARG, "k must be <= 262144");
  if (q <= 0) return SB_OK;
  const int64_t n = idx->n;
  if (!entries) {
    int r = gen_entries(idx, q, k, seed, qi0);
    if (r) return r;
    entries = idx->entries.as<int64_t>();
  }
  sb::RouteArgs a;
  const bool relabel = relabel_enabled();
  if (relabel) {
    int r = route_layout(idx);
    if (r) return r;
    a.F = idx->rl_F.as<float>(); a.A = idx->rl_A.as<int32_t>(); a.nbr_ids = idx->rl_ids.as<int32_t>();
    a.nbr_counts = idx->rl_counts.as<int32_t>();
    a.perm = idx->rl_perm.as<int32_t>();
    a.inv = a.perm + n;
  } else {
    a.F = idx->F.as<float>(); a.A = idx->A.as<int32_t>(); a.nbr_ids = idx->ids.as<int32_t>();
    a.nbr_counts = idx->counts.as<int32_t>();
    a.perm = nullptr;
    a.inv = nullptr;
  }
  a.n = n; a.m = idx->m; a.l = idx->l; a.g = idx->g;
  a.qf = qf; a.qa = qa; a.qm = qm; a.entries = entries; a.q = q; a.K = k; a.P = p;
  a.use_coarse = use_coarse ? 1 : 0; a.inv_alpha = inv_alpha; a.out_ids = out_ids;
  a.out_dists = out_dists; a.stats = out_stats;
  a.Kpad = next_pow2(k);
  a.Cpad = next_pow2(idx->g);
  // fp32-exact path for integer data (per query the kernel checks the query and the range,
  // and falls back to the sequential fp64 path): one row per lane by default (SB_ROUTE_LPR > 1
  // selects the lane-group variant; SB_ROUTE_F32=0 forces fp64)
  const char* f32env = getenv("SB_ROUTE_F32");
  const bool f32_want = f32env ? atoi(f32env) != 0 : true;
  a.f32_ok = (f32_want && idx->int_exact && idx->m % 4 == 0 && !idx->force_sequential) ? 1 : 0;
  a.flo = idx->flo;
  a.fhi = idx->fhi;
  a.lpr = 1;
  if (const char* e = getenv("SB_ROUTE_LPR")) a.lpr = std::max(1, std::min(32, next_pow2(atoi(e))));
  a.pf_rows = 1;
  if (const char* e = getenv("SB_ROUTE_PF")) a.pf_rows = atoi(e);
  // real-valued rows: SB_ROUTE_FILT=1 puts a certified fp32 filter (coalesced, lanes split
  // each row) in front of the exact sequential fp64 evaluation of the rows that can still enter
  // the result list (route.cu kModeF64Filt).  Off by default: measured slower (cfg 4: 38.7 vs
  // 29.3 ms, cfg 5 cardinality 10: 29.6 vs 20.6 ms; a batch almost always has a survivor, so
  // the exact chain stays on the critical path and the filter adds a pass)
  {
    const int nq = idx->m / 4;
    int lpr = 8;
    while (lpr < 32 && lpr * 4 < nq) lpr *= 2;
    a.flt_lpr = 0;
    if (const char* e = getenv("SB_ROUTE_FILT"))
      a.flt_lpr = (atoi(e) != 0 && idx->m % 4 == 0 && !idx->force_sequential) ? lpr : 0;
  }
  // real-valued rows, register-pipelined instance (one 8-warp CTA per SM): when rows are longer
  // than 1 KB (a lane walks its row in many dependent chunks) or the batch cannot fill more than
  // one such CTA per SM anyway.  SB_ROUTE_DEEP=0/1 forces it off/on.
  a.deep = (idx->m * 4 > 1024 || q <= (int64_t)idx->sms * 8) ? 1 : 0;
  if (const char* e = getenv("SB_ROUTE_DEEP")) a.deep = atoi(e) != 0;
  // its conversion-free fp32 -> fp64 step needs finite features (min/max of the upload scan)
  if (!(idx->flo >= -3.4028234e38f && idx->fhi <= 3.4028234e38f)) a.deep = 0;
  a.ring_slots = 0;
  // integer features in [0, 255]: route over a u8 copy with dp4a dot products (exact), unless
  // SB_ROUTE_U8=0; built once per layout
  a.F8 = nullptr;
  a.nx8 = nullptr;
  if (a.f32_ok && u8_eligible(idx)) {
    DBuf& buf = relabel ? idx->rl_f8 : idx->f8;
    int r = relabel ? ensure_u8(idx, a.F, idx->rl_f8, idx->rl_have_f8)
                    : ensure_u8(idx, a.F, idx->f8, idx->have_f8);
    if (r) return r;
    a.F8 = buf.as<uint8_t>();
    a.nx8 = reinterpret_cast<const int32_t*>(buf.as<uint8_t>() + (((size_t)n * idx->m + 255) & ~(size_t)255));
  }
  a.meta16 = nullptr;
  if (a.F8 && idx->l <= 3) {
    const int rl = relabel ? 1 : 0;
    const int64_t ver = relabel ? idx->rl_version : 0;
    if (idx->meta_version != ver || idx->meta_relabel != rl || !idx->meta16.p) {
      CK(idx->meta16.ensure(16 * (size_t)n));
      CKL(sb::launch_pack_meta16(a.nx8, a.A, n, idx->l, idx->meta16.p, idx->st));
      idx->meta_version = ver;
      idx->meta_relabel = rl;
      idx->launches += 1;
    }
    a.meta16 = reinterpret_cast<const uint4*>(idx->meta16.p);
  }
  a.gr_d = nullptr;
  a.gr_i = nullptr;
  idx->last_route_path = sb::route_path(a);
  size_t per_warp = sb::route_smem_per_warp(a);
  // large K (thousands to tens of thousands): once shared-memory result
  // lists would hold the SM below 16 resident queries, each slot's R lives in global memory
  // (L1/L2-resident in practice) and the insertion buffer and batch stay in shared memory:
  // 2.1x the QPS at K=4000, 7.1x at K=16000 on cfg 5 (cardinality 10^4), equal at K=1000.
  // SB_ROUTE_RGLOBAL=1 forces it, 0 disables it (unless R cannot fit shared memory at all).
  bool rglobal = per_warp * 16 > (size_t)227 * 1024;
  if (const char* e = getenv("SB_ROUTE_RGLOBAL")) rglobal = atoi(e) != 0 || per_warp > (size_t)200 * 1024;
  rglobal = rglobal && sb::route_large_k(a);  // the small-K instance keeps R in shared memory
  if (rglobal) {
    a.gr_d = reinterpret_cast<double*>(16);  // placeholder until the slots are known
    per_warp = sb::route_smem_per_warp(a);
  }
  int wpc_max = 8;
  if (const char* e = getenv("SB_ROUTE_WPC")) wpc_max = std::max(1, std::min(8, atoi(e)));
  int wpc = (int)std::max<size_t>(1, std::min<size_t>(wpc_max, (size_t)(110 * 1024) / per_warp));
  if (sb::route_path(a) == 6) {
    // the staged instance runs one CTA per SM: just enough warps for the batch (at most 8), and
    // what is left of the SM's shared memory becomes the warps' row-line rings
    const size_t budget = (size_t)220 * 1024;
    wpc = (int)std::max<int64_t>(1, std::min<int64_t>(wpc_max, (q + idx->sms - 1) / idx->sms));
    while (wpc > 1 && budget / wpc < per_warp + 64 * 144 + 256) --wpc;
    const size_t spare = budget / wpc > per_warp + 256 ? budget / wpc - per_warp - 256 : 0;
    a.ring_slots = (int)std::min<size_t>(512, spare / 144);
    if (a.ring_slots < 64) {  // no room for a useful ring: the three-CTA instance
      a.deep = 0;
      a.ring_slots = 0;
      idx->last_route_path = sb::route_path(a);
      wpc = (int)std::max<size_t>(1, std::min<size_t>(wpc_max, (size_t)(110 * 1024) / per_warp));
    } else {
      per_warp = sb::route_smem_per_warp(a);
    }
  }
  if (per_warp * wpc > 227 * 1024) return fail(SB_EARG, "k too large for the routing kernel");
  int per_sm = 0;
  CKL(sb::route_occupancy(a, wpc, per_warp * wpc, &per_sm));
  if (per_sm < 1) return fail(SB_EARG, "routing kernel does not fit on an SM for this k");
  if (const char* e = getenv("SB_ROUTE_QPSM"))  // resident queries per SM cap (experiments)
    per_sm = std::max(1, std::min(per_sm, atoi(e) / wpc));
  int ctas = (int)std::min<int64_t>((int64_t)idx->sms * per_sm, (q + wpc - 1) / wpc);
  int64_t slots = (int64_t)ctas * wpc;
  a.vwords = (n + 31) / 32;
  a.logcap = 8192;
  size_t vis_bytes = sizeof(uint32_t) * slots * a.vwords;
  bool fresh = idx->visited.bytes < vis_bytes;
  CK(idx->visited.ensure(vis_bytes));
  if (fresh) CK(cudaMemsetAsync(idx->visited.p, 0, idx->visited.bytes, idx->st));
  CK(idx->vlog.ensure(sizeof(uint32_t) * slots * a.logcap));
  CK(idx->counter.ensure(sizeof(int) * 4));
  CK(cudaMemsetAsync(idx->counter.p, 0, sizeof(int), idx->st));
  if (rglobal) {
    CK(idx->route_gr.ensure((size_t)12 * slots * a.Kpad));
    a.gr_d = idx->route_gr.as<double>();
    a.gr_i = reinterpret_cast<uint32_t*>(a.gr_d + slots * a.Kpad);
  }
  a.visited = idx->visited.as<uint32_t>();
  a.vlog = idx->vlog.as<uint32_t>();
  a.counter = idx->counter.as<int>();
  CKL(sb::launch_route(a, wpc, ctas, idx->st));
  idx->launches += 1;
  return SB_OK;
}

int sb_route_batch_dev(sb_index* idx, const double* qf, const double* qa, const double* qmask,
                       int64_t q, int32_t k, int32_t pioneer, int32_t use_coarse,
                       const int64_t* entries, uint64_t seed, int64_t qi0, double inv_alpha,
                       int64_t* out_ids, double* out_dists, int64_t* out_stats) {
  if (!idx || !qf || !qa || !out_ids || !out_dists) return fail(SB_EARG, "NULL argument");
  return route_dev(idx, qf, qa, qmask, q, k, pioneer, use_coarse, entries, seed, qi0, inv_alpha,
                   out_ids, out_dists, out_stats);
}

// device address of page-locked host memory (cudaHostAlloc / registered), or null
static void* mapped_host(const void* p) {
  if (!p) return nullptr;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

int sb_route_batch(sb_index* idx, const double* qf, const double* qa, const double* qmask,
                   int64_t q, int32_t k, int32_t pioneer, int32_t use_coarse,
                   const int64_t* entries, uint64_t seed, int64_t qi0, double inv_alpha,
                   int64_t* out_ids, double* out_dists, int64_t* out_stats) {
  if (!idx || !qf || !qa || !out_ids || !out_dists) return fail(SB_EARG, "NULL argument");
  if (q <= 0) return SB_OK;
  const int m = idx->m, l = idx->l;
  // Page-locked result buffers are written by the kernel itself, over the link, while it
  // runs (cfg 2, same box: 8.0 ms per 10k-query call vs 8.6 ms with a copy at the end and
  // 10.0 ms into pageable memory); SB_ROUTE_DIRECT=0 forces the copy.
  const char* de = getenv("SB_ROUTE_DIRECT");
  const bool want_direct = de ? atoi(de) != 0 : true;
  int64_t* d_ids_h = want_direct ? static_cast<int64_t*>(mapped_host(out_ids)) : nullptr;
  double* d_dists_h = want_direct ? static_cast<double*>(mapped_host(out_dists)) : nullptr;
  int64_t* d_st_h = want_direct && out_stats ? static_cast<int64_t*>(mapped_host(out_stats)) : nullptr;
  const bool direct = d_ids_h && d_dists_h && (!out_stats || d_st_h);
  // one device block for all per-call inputs/outputs
  size_t o_qf = 0, o_qa = o_qf + sizeof(double) * q * m, o_qm = o_qa + sizeof(double) * q * l;
  size_t o_en = o_qm + sizeof(double) * q * l, o_ids = o_en + (entries ? sizeof(int64_t) * q * k : 0);
  size_t o_d = o_ids + sizeof(int64_t) * q * k, o_st = o_d + sizeof(double) * q * k;
  size_t total = direct ? o_ids : o_st + sizeof(int64_t) * q * 5;
  CK(idx->qf.ensure(total));
  char* base = idx->qf.as<char>();
  // entry points drawn on the device need no query data: draw them first on the handle's
  // stream while the queries upload on a side stream (the upload overlaps the RNG kernel)
  const int64_t* dev_entries = nullptr;
  cudaStream_t up = idx->st;
  if (!entries && k >= 1 && k <= idx->n && k <= (1 << 18) && pioneer >= 1 && pioneer <= k) {
    int r = gen_entries(idx, q, k, seed, qi0);
    if (r) return r;
    dev_entries = idx->entries.as<int64_t>();
    if (!idx->st_up) {
      CK(cudaStreamCreateWithFlags(&idx->st_up, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&idx->ev_up, cudaEventDisableTiming));
    }
    up = idx->st_up;
  }
  CK(cudaMemcpyAsync(base + o_qf, qf, sizeof(double) * q * m, cudaMemcpyHostToDevice, up));
  CK(cudaMemcpyAsync(base + o_qa, qa, sizeof(double) * q * l, cudaMemcpyHostToDevice, up));
  if (qmask) CK(cudaMemcpyAsync(base + o_qm, qmask, sizeof(double) * q * l, cudaMemcpyHostToDevice, up));
  if (entries) CK(cudaMemcpyAsync(base + o_en, entries, sizeof(int64_t) * q * k, cudaMemcpyHostToDevice, up));
  if (up != idx->st) {
    CK(cudaEventRecord(idx->ev_up, up));
    CK(cudaStreamWaitEvent(idx->st, idx->ev_up, 0));
  }
  int64_t* r_ids = direct ? d_ids_h : reinterpret_cast<int64_t*>(base + o_ids);
  double* r_d = direct ? d_dists_h : reinterpret_cast<double*>(base + o_d);
  int64_t* r_st = direct ? d_st_h : (out_stats ? reinterpret_cast<int64_t*>(base + o_st) : nullptr);
  int r = route_dev(idx, reinterpret_cast<double*>(base + o_qf), reinterpret_cast<double*>(base + o_qa),
                    qmask ? reinterpret_cast<double*>(base + o_qm) : nullptr, q, k, pioneer,
                    use_coarse, entries ? reinterpret_cast<int64_t*>(base + o_en) : dev_entries, seed,
                    qi0, inv_alpha, r_ids, r_d, r_st);
  if (r) return r;
  if (!direct) {
    CK(cudaMemcpyAsync(out_ids, base + o_ids, sizeof(int64_t) * q * k, cudaMemcpyDeviceToHost, idx->st));
    CK(cudaMemcpyAsync(out_dists, base + o_d, sizeof(double) * q * k, cudaMemcpyDeviceToHost, idx->st));
    if (out_stats) CK(cudaMemcpyAsync(out_stats, base + o_st, sizeof(int64_t) * q * 5, cudaMemcpyDeviceToHost, idx->st));
  }
  CK(cudaStreamSynchronize(idx->st));
  return SB_OK;
}

}  // extern "C"

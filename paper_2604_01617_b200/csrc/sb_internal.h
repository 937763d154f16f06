// sb_internal.h — kernel launch interfaces shared between the .cu files and the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace sb {

// ---- routing (route.cu) ----------------------------------------------------
struct RouteArgs {
  const float* F;
  const int32_t* A;
  const int32_t* nbr_ids;
  const int32_t* nbr_counts;
  int64_t n;
  int m, l, g;
  const double* qf;        // q x m
  const double* qa;        // q x l
  const double* qm;        // q x l or null (all ones)
  const int64_t* entries;  // q x K
  int64_t q;
  int K, P, use_coarse;
  double inv_alpha;
  int64_t* out_ids;   // q x K
  double* out_dists;  // q x K
  int64_t* stats;     // q x 5 or null
  uint32_t* visited;  // slots x vwords
  int64_t vwords;
  uint32_t* vlog;     // slots x logcap
  int logcap;
  int* counter;
  int Kpad, Cpad;
  // fp32-exact path (integer data): enabled for the index, feature range, lanes per row
  int f32_ok;
  float flo, fhi;
  int lpr;
  // real-valued data (m % 4 == 0): lanes per row of the certified fp32 filter in front of the
  // exact fp64 rows (8, 16 or 32); 0 = every row exact (no filter)
  int flt_lpr;
  int pf_rows;  // prefetch each batch's rows into L2 before evaluating
  // real-valued rows: the register-pipelined instance (one CTA per SM, 128 registers of row
  // loads in flight per lane) instead of the three-CTA one
  int deep;
  int ring_slots;  // its per-warp staging ring, in 144-byte row-line slots
  // u8 copy of integer features in [0, 255] (null: not available) and exact |x|^2
  const uint8_t* F8;
  const int32_t* nx8;
  // relabeled layout (route_layout): every id the kernel sees is a new id; entries arrive as
  // original ids (mapped through inv), results leave as original ids (through perm), and
  // exact distance ties compare original ids.  Null: identity.
  const int32_t* perm;  // new -> original
  const int32_t* inv;   // original -> new
  // u8 path, l <= 3: {|x|^2, attrs} per node in one 16-byte record (null: separate arrays)
  const uint4* meta16;
  // very large K: the result list R of each slot in global memory (slots x Kpad dists and
  // ids) instead of shared memory; null: R in shared memory
  double* gr_d;
  uint32_t* gr_i;
};
int launch_pack_meta16(const int32_t* nx, const int32_t* A, int64_t n, int l, void* out, cudaStream_t st);
// locality order of the nodes for routing: Z-order of random projections (route.cu)
int launch_route_order(const float* F, int64_t n, int m, int32_t* perm, int32_t* inv,
                       void* scratch, size_t scratch_bytes, cudaStream_t st);
size_t route_order_scratch_bytes(int64_t n);
int launch_permute_rows_f32(const float* src, int64_t n, int m, const int32_t* perm, float* dst,
                            cudaStream_t st);
int launch_permute_rows_i32(const int32_t* src, int64_t n, int w, const int32_t* perm,
                            int32_t* dst, cudaStream_t st);
int launch_relabel_adjacency(const int32_t* ids, const int32_t* counts, int64_t n, int g,
                             const int32_t* perm, const int32_t* inv, int32_t* ids_r,
                             int32_t* counts_r, cudaStream_t st);

size_t route_smem_per_warp(const RouteArgs& a);
// the insertion-buffer (large-K) kernel instance serves this launch
bool route_large_k(const RouteArgs& a);
int launch_feature_scan(const float* F, int64_t count, unsigned* out3, cudaStream_t st);
int launch_pack_u8(const float* F, int64_t n, int m, uint8_t* F8, int32_t* nx, cudaStream_t st);
float feature_key_to_float(unsigned k);
int route_occupancy(const RouteArgs& a, int warps_per_cta, size_t smem, int* ctas_per_sm);
int launch_route(const RouteArgs& a, int warps_per_cta, int ctas, cudaStream_t st);
int route_path(const RouteArgs& a);  // distance path route_kernel takes for these args
int launch_entry_points(int64_t n, int K, uint64_t seed, int64_t qi0, int64_t q, int64_t* out,
                        int64_t* scratch, uint64_t scratch_slots, cudaStream_t st);

// ---- exhaustive AUTO top-k (bf_topk.cu) --------------------------------------
struct BfArgs {
  const float* F;
  const int32_t* A;
  int64_t n;
  int m, l;
  const int64_t* self_ids;  // node mode when non-null
  const double* qf;         // query mode: f64 q x m
  const int64_t* qa;        // query mode: i64 q x l
  const int64_t* qmask;     // query mode: i64 q x l or null
  int64_t q;
  int k;                    // list length kept per query (>= requested k)
  double inv_alpha;         // node mode: s_a * inv_alpha (_kernels.py:23)
  double alpha;             // query mode: s_a / alpha (evaluate.py:53)
  int splits;
  double* part_d;           // q x splits x k
  uint32_t* part_i;
};
int bf_group_size();
size_t bf_partial_smem(int k);
int launch_bf_partial(const BfArgs& a, cudaStream_t st);
int launch_bf_merge_k(const BfArgs& a, int kout, int64_t* out_ids64, int32_t* out_ids32,
                      double* out_dists, int* uncertain, cudaStream_t st);

// exhaustive top-k of any k by a full segmented radix sort of exact keys (bf_sort.cu)
enum { kBfSortNode = 0, kBfSortQuery = 1, kBfSortHybrid = 2 };
int64_t bf_sort_chunk(int64_t n, int64_t q);               // queries per sort launch
size_t bf_sort_scratch_bytes(int64_t n, int64_t b);
int launch_bf_sorted(const BfArgs& a, int mode, int64_t q0, int64_t b, int kout, void* scratch,
                     size_t scratch_bytes, int64_t* out_ids64, int32_t* out_ids32,
                     double* out_dists, int64_t* out_counts, cudaStream_t st);

// tensor-core query-mode top-k for integer data (bf_tc.cu)
// rowb = operand bytes per row: 2 x features (bf16) or features (u8)
int bf_tc_supported(int rowb, int l, int kk);
int bf_tc_ctas_per_sm(int rowb, int l, int kk);
int launch_tc_gather_u8(const float* F, const int32_t* A, const int32_t* code_in,
                        const int32_t* orig, int64_t n, int m, int l, void* Fb, int32_t* nx,
                        int32_t* code, int32_t* As, cudaStream_t st);
int launch_bf_tc_prep_queries_u8(const double* qf, int64_t q, int m, void* Qb, int32_t* nq,
                                 cudaStream_t st);
constexpr int kTcNodePad = 256;  // node arrays of the tensor-core path are padded to this
int launch_tc_attr_range(const int32_t* A, int64_t n, int l, int32_t* lo, int32_t* hi,
                         cudaStream_t st);
int launch_tc_code(const int32_t* A, int64_t n, int l, const int32_t* lo, const int64_t* stride,
                   int grouped, int32_t* code, unsigned long long* hist, cudaStream_t st);
int launch_tc_scatter(const int32_t* code, int64_t n, const int64_t* off, unsigned long long* cur,
                      int32_t* orig, cudaStream_t st);
int launch_tc_gather(const float* F, const int32_t* A, const int32_t* code_in, const int32_t* orig,
                     int64_t n, int m, int mk, int l, void* Fb, int32_t* nx, int32_t* code,
                     int32_t* As, cudaStream_t st);
int launch_bf_tc_prep_queries(const double* qf, int64_t q, int m, int mk, void* Qb, int32_t* nq,
                              cudaStream_t st);
// m below is the operand K: the feature count, plus 16 when fold (|x|^2 folded into the MMA)
// |x|^2 order inside attribute tuples (u8 tensor-core top-k) and its per-16-node chunk records
size_t tc_norm_order_scratch(int64_t n);
int launch_tc_norm_order(const float* F, int64_t n, int m, const int32_t* code_in, int32_t* orig,
                         void* scratch, cudaStream_t st);
int launch_tc_chunk_meta(const int32_t* nx, const int32_t* code, int64_t n, int64_t npad, void* cm,
                         cudaStream_t st);
int launch_bf_tc(const void* Fb, const int32_t* nx, const int32_t* A, const int32_t* code,
                 const int32_t* orig, const void* Qb, const int32_t* nq, const int64_t* qa,
                 const int64_t* qmask, int64_t n, int64_t q, int m, int l, int kk, int splits,
                 double alpha, double* part_d, uint32_t* part_i, int* gthr, int fold, int u8, const void* cmeta,
                 cudaStream_t st);

// tensor-core query-mode top-k for real-valued data (bf_tf.cu): TF32 filter, exact re-rank
double tf_margin(int dpad);
int bf_tf_supported(int m, int l, int kk);
int bf_tf_dpad(int m);
void bf_tf_layout(int m, int l, int kk, int* qblock, int* ppq, int* ew);
int launch_tf_gather(const float* F, const int32_t* A, const int32_t* code_in, const int32_t* orig,
                     int64_t n, int m, int l, double cE, float* Ft, float* nxd, int32_t* code,
                     int32_t* As, cudaStream_t st);
int launch_tf_runend(const int32_t* code, int64_t n, int32_t* runend, cudaStream_t st);
int launch_tf_prep_queries(const double* qf, int64_t q, int64_t qpad, int m, double cE, double tiny,
                           float* Qt, float* nqs, float* nqu, cudaStream_t st);
int launch_bf_tf(const float* Ft, const float* nxd, const int32_t* code,
                 const int32_t* orig, const int32_t* runend, const int32_t* As, const float* Qt, const float* nqs,
                 const float* nqu, const int64_t* qa, const int64_t* qmask, int64_t n, int64_t q,
                 int m, int l, int kk, int splits, double alpha, int* gthr, uint32_t* cnt,
                 uint64_t* cand, int cap, uint32_t* ocnt, uint64_t* ocand, int ocap, int seed,
                 int strided, int bound_only, int fixed, float* lists, cudaStream_t st);
// large k: gthr[g] = the k-th smallest of the q x nl per-thread list keys (bf_tf.cu)
int launch_tf_select(const float* lists, int64_t q, int nl, int k, int* gthr, cudaStream_t st);
// exact seed bound of each query's k-th key from the nodes of its own attribute-code run
int launch_tf_code_seed(const float* F, const int32_t* A, const int32_t* s_code, const int32_t* s_orig,
                        int64_t n, int m, int l, const double* qf, const int64_t* qa,
                        const int64_t* qmask, int64_t q, int k, double alpha, const int32_t* lo8,
                        const int64_t* stride8, int* gthr, cudaStream_t st);
int launch_tf_refine(const float* F, const int32_t* A, int m, int l, const double* qf,
                     const int64_t* qa, const int64_t* qmask, int64_t q, int k, double alpha,
                     const uint32_t* cnt, const uint64_t* cand, int splits, int hsegs, int qblock,
                     int ew, int cap,
                     const uint32_t* ocnt, const uint64_t* ocand, int ocap, const int* gthr, int scap, int64_t* out_ids, double* out_d, int* ovf, int* ovf_count,
                     unsigned long long* emitted_total, cudaStream_t st);

// ---- HELP build ---------------------------------------------------------------
// random initial rows (help_init.cu): device ids, consumed PCG64 outputs, rows with repeats
int launch_init_random_ids(uint64_t seed, int64_t n, int g, int32_t* ids, int64_t* scratch,
                           int64_t scratch_slots, int64_t* consumed, int64_t* bad,
                           unsigned long long* nbad, cudaStream_t st);
int64_t init_random_ids_scratch_slots(int64_t n, int g);

struct BuildScratch {
  int32_t* fwd_new;   // n
  int32_t* fwd_old;   // n
  int64_t* rev_cnt;   // n
  int64_t* rev_off;   // n
  int64_t* rev_cur;   // n
  int32_t* rev;       // n * max(gn, g)
  int64_t* scan_tmp;  // scan_tmp_slots(n)
};

int64_t scan_tmp_slots(int64_t n);
int exclusive_scan(const int64_t* in, int64_t* out, int64_t n, int64_t* tmp, cudaStream_t st);
int launch_init_dists(const float* F, const int32_t* A, int64_t n, int m, int l, int g,
                      double inv_alpha, int32_t* ids, float* dists, cudaStream_t st);
int launch_count_in_degrees(const int32_t* ids, const int32_t* counts, int64_t n, int g,
                            int32_t* in_deg, int32_t* smax, cudaStream_t st);
int launch_build_candidates(const int32_t* ids, uint8_t* flags, int64_t n, int g, int gn,
                            int32_t* new_cand, int32_t* new_cnt, int32_t* old_cand,
                            int32_t* old_cnt, BuildScratch& s, cudaStream_t st);

struct JoinArgs {
  const float* F;
  const int32_t* A;
  int64_t n;
  int m, l, g, gn;
  double inv_alpha;
  const int32_t* new_cand;
  const int32_t* new_cnt;
  const int32_t* old_cand;
  const int32_t* old_cnt;
  const uint64_t* thr;     // current row tails
  int64_t node_begin, node_end;
  int* node_counter;
  uint32_t* push_tgt;
  uint64_t* push_key;
  uint64_t push_cap;
  unsigned long long* push_count;
  int64_t* row_cnt;
  int* overflow;
  unsigned long long* same_pairs;  // pairs skipped because new[x] == old[y] (j == k)
  int spad, dc, ntiles_max;
  const uint8_t* F8;      // u8 rows (integer data in [0, 255]) or null: fp64 path
  const int32_t* nx8;     // exact |x|^2 of the u8 rows
};
size_t join_emit_smem(int spad, int dc, int l, int ntiles_max);
int join_emit_occupancy(size_t smem, int* ctas_per_sm);
int launch_thr_init(const int32_t* ids, const float* dists, int64_t n, int g, uint64_t* thr,
                    cudaStream_t st);
int launch_join_emit(const JoinArgs& a, int ctas, size_t smem, cudaStream_t st);
int launch_push_scatter(const uint32_t* tgt, const uint64_t* key, uint64_t total,
                        const int64_t* row_off, int64_t* row_cur, uint64_t* seg, cudaStream_t st);
int launch_row_merge(int32_t* ids, float* dists, uint8_t* flags, uint64_t* thr, int64_t n, int g,
                     const int64_t* row_off, const int64_t* row_cnt, const uint64_t* seg,
                     unsigned long long* inserted, cudaStream_t st);

struct PruneArgs {
  const float* F;
  const int32_t* A;
  int64_t n;
  int m, l, g, W;
  int32_t* ids;
  float* dists;
  int32_t* counts;
  double sigma;
  uint32_t* rbits;     // n x g x W
  const int32_t* smax;
  const int32_t* indeg0;
  uint8_t* guard;
  int32_t* drop_other;
  uint32_t* keep;      // n x W
  int32_t* in_deg;
  int cpad, dc;
};
size_t prune_bits_smem(int cpad, int dc, int m, int l, int W);
int launch_prune_bits(const PruneArgs& a, size_t smem, cudaStream_t st);
size_t prune_bits_u8_smem(int cpad, int m, int l, int W);
int launch_prune_bits_u8(const PruneArgs& a, const uint8_t* F8, const int32_t* nx8, size_t smem,
                         cudaStream_t st);
int launch_prune_scan(const PruneArgs& a, cudaStream_t st);
int launch_prune_guard(const PruneArgs& a, int* changed, cudaStream_t st);
int launch_prune_compact(const PruneArgs& a, cudaStream_t st);
int launch_reinforce_check(const int32_t* ids, const float* dists, const int32_t* counts,
                           int64_t n, int g, int64_t* rev_extra, unsigned long long* over,
                           cudaStream_t st);
int launch_symmetrize(int32_t* ids, float* dists, int32_t* counts, int64_t n, int g,
                      const int64_t* rev_extra, int64_t* off, int64_t* cur, uint64_t* seg,
                      int64_t* scan_tmp, cudaStream_t st);
// one reconnect_islands sweep (_kernels.py:455-487), exact, by one CTA (help_prune.cu)
int launch_reconnect(const float* F, const int32_t* A, int m, int l, int g, int32_t* ids,
                     float* dists, int32_t* counts, int32_t* in_deg, double sigma, int64_t n,
                     cudaStream_t st);
int launch_min_i32(const int32_t* x, int64_t n, int* out, cudaStream_t st);
int launch_row_union_merge(int32_t* ids, float* dists, int32_t* counts, int64_t n, int g,
                           const int64_t* off, const int64_t* extra, const uint64_t* seg,
                           cudaStream_t st);

// exact reinforce with the sequential part confined to overflow rows (help_reinforce.cu)
struct RfArgs {
  int64_t n;
  int m, l, g;
  const float* F;
  const int32_t* A;
  int32_t* ids;
  float* dists;
  int32_t* counts;
  int32_t* in_deg;
  double sigma;
  uint8_t* mutual;      // n x g
  int32_t* eo;          // n x g: O index of each edge's target (-1 not in O, -2 past count)
  int32_t* ecu;         // n x g: the source's position in U_target for edges into O, else -1
  int64_t* rev_extra;   // n
  uint8_t* is_o;        // n
  int32_t* o_idx;       // n
  int64_t no;
  int32_t* o_nodes;     // no
  int64_t* u_size;      // no
  int64_t* u_off;       // no + 1
  int64_t* u_cur;       // no
  int32_t* u_list;      // sum u
  int64_t* r_off;       // no + 1
  uint32_t* r_bits;
  int32_t* u_pos;       // no x g
  int32_t* static_ins;  // n
  uint8_t* relevant;    // n
  int64_t* orev_cnt;    // n
  int64_t* apply_cnt;   // n
  int64_t* apply_off;   // n
  int64_t* apply_cur;   // n
  uint64_t* apply_seg;
  int32_t* rec_tgt;
  uint64_t* rec_key;
  int64_t* rec_next;
  int32_t* rec_cu;      // per record: the mirrored node's position in U_source
  int64_t* rec_head;    // n
  int64_t rec_cap;
  uint64_t* dyn;
  int32_t* dyn_cu;      // U position of each dynamic event's candidate
  int dyn_cap;
  int sim_wmax;         // max redundancy-row words over O rows (simulation scratch size)
  int64_t* result;      // [nrec, err]
  int64_t* rec_count;   // records allocated (all groups)
  // groups of O-row components simulated in parallel (one warp each)
  int ngroups;
  int32_t* grp_of_o;    // no
  uint32_t* grp_bits;   // ngroups x bm_words source bitmaps
  int64_t bm_words;
};
__host__ __device__ size_t rf_simulate_smem(int g, int wmax);
int rf_launch_stage1(RfArgs& a, int64_t* oflag, int64_t* oscan, int64_t* scan_tmp, cudaStream_t st);
int rf_launch_stage2(RfArgs& a, const int64_t* oscan, cudaStream_t st);
int rf_launch_stage3(RfArgs& a, int upad_max, int dc_max, int upad4_max, size_t bits_smem,
                     cudaStream_t st);
int rf_launch_simulate(RfArgs& a, cudaStream_t st);
int rf_launch_group_bits(RfArgs& a, cudaStream_t st);
int rf_launch_apply(RfArgs& a, int64_t nrec, int64_t* scan_tmp, cudaStream_t st);

}  // namespace sb

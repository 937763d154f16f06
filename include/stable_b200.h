/*
 * stable_b200.h — C ABI of the B200 (sm_100a) hot path of STABLE's AUTO metric:
 * exhaustive AUTO top-k, HELP graph construction and Dynamic Heterogeneity Routing.
 *
 * The reference (hybridann 0.1.0, pure Python + Numba) reaches its hot path only through
 * module-attribute calls `_kernels.<fn>(...)` on C-contiguous NumPy buffers
 * (graph.py:13, router.py:15).  Each entry point below replaces one of those functions, or a
 * Python loop around them, with the same argument meaning; the binding a maintainer adds on
 * the reference side is a ctypes stub.
 *
 * Conventions
 *   - plain pointers + sizes, no C++ or torch types; host buffers unless the name ends in
 *     _dev (device pointers, asynchronous on the handle's stream).
 *   - every call returns SB_OK or an error code and never throws; sb_last_error() gives a
 *     thread-local message.  Codes map onto the reference's exception taxonomy
 *     (errors.py:8-31, exit codes cli.py:353-361):
 *       SB_EARG -> ValueError, SB_EFORMAT -> FormatError, SB_ECONSTRAINT -> ConstraintError,
 *       SB_ECUDA -> a device failure (no reference counterpart; raised as RuntimeError).
 *   - layouts as the reference passes them (_kernels.py:1-6, graph.py:64-72):
 *       features f32[n*m], attrs i32[n*l], nbr_ids i32[n*gamma], nbr_dists f32[n*gamma],
 *       nbr_flags u8[n*gamma], nbr_counts i32[n].
 *   - one CUDA stream per handle: calls on one handle serialise; distinct handles may run
 *     concurrently.
 */
#ifndef STABLE_B200_H
#define STABLE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { SB_OK = 0, SB_EARG = 1, SB_EFORMAT = 2, SB_ECONSTRAINT = 3, SB_ECUDA = 4 };

typedef struct sb_index sb_index;

const char* sb_last_error(void);
int sb_version(void);                 /* (major << 16) | minor */
int sb_device_count(int* count);

/* ---- handle ----------------------------------------------------------------------
 * Uploads the dataset (RelationGraph.features / .attrs, graph.py:64-65) and reserves an
 * adjacency of capacity gamma (graph.py:69-72).  Replaces nothing by itself: the reference
 * keeps these arrays on the Python object and re-passes them to every kernel. */
int sb_index_create(const float* features, const int32_t* attrs, int64_t n, int32_t m,
                    int32_t l, int32_t gamma, sb_index** out);
int sb_index_destroy(sb_index* idx);
int sb_set_stream(sb_index* idx, void* cuda_stream);   /* NULL: the handle's own stream */
int sb_synchronize(sb_index* idx);
/* nbr_flags may be NULL (frozen graphs carry none, graph.py:231) */
int sb_adj_upload(sb_index* idx, const int32_t* nbr_ids, const float* nbr_dists,
                  const int32_t* nbr_counts, const uint8_t* nbr_flags);
int sb_adj_download(sb_index* idx, int32_t* nbr_ids, float* nbr_dists, int32_t* nbr_counts,
                    uint8_t* nbr_flags);

/* ---- HELP construction ----------------------------------------------------------- */

/* compute_row_distances (_kernels.py:71-78) + the per-row lexsort((ids, dists))
 * (graph.py:132-136) of init_random_graph: ids are the host-drawn random neighbours
 * (graph.py:120-129); afterwards the device adjacency is sorted, counts = gamma, flags = 1. */
int sb_init_graph(sb_index* idx, const int32_t* ids, double inv_alpha);
/* The random initial rows of graph.py:120-129 drawn on the device: fills the handle's ids with
 *   rng = default_rng(seed); ids = rng.integers(0, n - 1, (n, gamma)); ids += ids >= arange(n)
 * bit-exactly.  Reports the 32-bit draws consumed (*consumed32; the 64-bit PCG64 outputs are
 * ceil(consumed32 / 2), and when consumed32 is odd NumPy keeps the unused high half,
 * *buffered, in the generator) and the ascending rows that hold a repeated id (*nbad of them,
 * written to bad_rows when non-NULL and bad_cap suffices).  The host redraws those rows
 * (graph.py:124-128) from the generator so restored and writes them with sb_set_rows.  Pass
 * ids = NULL to sb_init_graph to keep the device rows. */
int sb_init_random_ids(sb_index* idx, uint64_t seed, int64_t* consumed32, uint32_t* buffered,
                       int64_t* bad_rows, int64_t bad_cap, int64_t* nbad);
/* overwrite the ids of rows[0..s) (s x gamma, row-major) on the device */
int sb_set_rows(sb_index* idx, const int64_t* rows, int64_t s, const int32_t* ids);

/* build_candidates (_kernels.py:81-135) on the device adjacency; the new/old lists stay on
 * the device for sb_local_join.  Output pointers may be NULL (download skipped). */
int sb_build_candidates(sb_index* idx, int32_t gamma_new, int32_t* new_cand,
                        int32_t* new_counts, int32_t* old_cand, int32_t* old_counts);

/* hand the device a candidate split computed elsewhere (the arrays build_candidates
 * returns, _kernels.py:81-135), for a kernel-level local_join call */
int sb_set_candidates(sb_index* idx, int32_t gamma_new, const int32_t* new_cand,
                      const int32_t* new_counts, const int32_t* old_cand,
                      const int32_t* old_counts);

/* local_join (_kernels.py:138-173).  *inserted > 0 iff some row changed (the reference's
 * return value is only compared with 0, graph.py:256); *pairs = distance evaluations. */
int sb_local_join(sb_index* idx, double inv_alpha, int64_t* inserted, int64_t* pairs);

/* descent_iteration (graph.py:151-176) = sb_build_candidates + sb_local_join */
int sb_descent_iteration(sb_index* idx, int32_t gamma_new, double inv_alpha, int64_t* inserted,
                         int64_t* pairs);

/* count_in_degrees (_kernels.py:256-263) */
int sb_count_in_degrees(sb_index* idx, int64_t* in_deg);

/* rows ids[s*gamma], counts[s] of the given nodes (the inputs graph_quality reads,
 * _kernels.py:207-224; psi itself is summed on the host in the reference's order). */
int sb_get_rows(sb_index* idx, const int64_t* rows, int64_t s, int32_t* ids, int32_t* counts);

/* prune_pass (_kernels.py:266-303) with in_deg = count_in_degrees (graph.py:212-216).
 * *rounds = Jacobi guard rounds used. */
int sb_prune(sb_index* idx, double sigma, int32_t* rounds);

/* reinforce_pass (_kernels.py:398-409) and the <= 10 reconnect_islands sweeps
 * (graph.py:217-230), continuing from sb_prune's in-degrees.  *overflow_rows = rows that would
 * exceed capacity (0: symmetrisation fast path), *sweeps = reconnect sweeps run. */
int sb_reinforce(sb_index* idx, double sigma, int64_t* overflow_rows, int32_t* sweeps);

/* the two halves of sb_reinforce at kernel granularity: reinforce_pass
 * (_kernels.py:398-409) alone, and one reconnect_islands sweep (_kernels.py:455-487) with
 * freshly counted in-degrees (*ran = 0 when every node already has an in-edge). */
int sb_reinforce_pass(sb_index* idx, double sigma, int64_t* overflow_rows);
int sb_reconnect_islands(sb_index* idx, double sigma, int32_t* ran);

/* ---- exhaustive AUTO top-k ------------------------------------------------------ */

/* brute_force_topk (_kernels.py:176-204): exact top-k over all v != u, ids padded -1.
 * Any k >= 1 (k > 1024 takes the full-sort kernel, bf_sort.cu). */
int sb_bf_topk_nodes(sb_index* idx, const int64_t* sample_ids, int64_t s, int32_t k,
                     double inv_alpha, int32_t* out_ids);

/* oracle_auto_topk (evaluate.py:32-55) for q queries at once: qf f64[q*m], qa i64[q*l],
 * qmask i64[q*l] or NULL; fused = sqrt(s_v) * (1 + s_a / alpha), ties by id.
 * *uncertain counts queries whose exact re-rank could not be certified (0 expected).
 * Any 1 <= k <= n (k > 1000 takes the full-sort kernel, bf_sort.cu). */
int sb_bf_topk_queries(sb_index* idx, const double* qf, const int64_t* qa, const int64_t* qmask,
                       int64_t q, int32_t k, double alpha, int64_t* out_ids, double* out_dists,
                       int32_t* uncertain);

/* oracle_hybrid_groundtruth (evaluate.py:58-77) for q queries: the nodes whose (masked)
 * attribute Manhattan distance to the query is 0, ranked by pure feature distance
 * (sqrt of NumPy's pairwise sum, evaluate.py:73-74), ties by id.  out_ids i64[q*k] padded
 * with -1, out_dists f64[q*k] (+inf padding) or NULL, out_counts i64[q] = min(k, matches). */
int sb_hybrid_groundtruth(sb_index* idx, const double* qf, const int64_t* qa, const int64_t* qmask,
                          int64_t q, int32_t k, int64_t* out_ids, double* out_dists,
                          int64_t* out_counts);

/* ---- Dynamic Heterogeneity Routing --------------------------------------------- */

/* entry_points (router.py:42-45) for query indices qi0 .. qi0+q-1, host computation:
 * default_rng(SeedSequence((seed, qi))).choice(n, k, replace=False). out i64[q*k]. */
int sb_entry_points(int64_t n, int32_t k, uint64_t seed, int64_t qi0, int64_t q, int64_t* out);

/* the same on the device (the kernels sb_route_batch uses when entries is NULL), copied back to
 * out i64[q*k]; for tests and comparisons */
int sb_entry_points_device(int64_t n, int32_t k, uint64_t seed, int64_t qi0, int64_t q, int64_t* out);

/* search_batch (router.py:98-124) as one device call: route (_kernels.py:504-610) for q
 * queries with query_index = qi0 + row.  qf f64[q*m], qa f64[q*l], qmask f64[q*l] or NULL
 * (router.py:62-73 widens to f64); entries i64[q*k] or NULL (drawn on the device with the
 * reference's stream).  out_stats i64[q*5] or NULL: dist_evals, phase1_evals,
 * phase1_expansions, hops (SearchStats, router.py:34-39) + neighbours scanned.
 * 1 <= k <= min(n, 262144); 1 <= pioneer <= k (SB_EARG otherwise).  k above ~16,000 keeps
 * its result lists in global memory, which only the large-K kernel instance supports: that
 * instance needs gamma > 8 and SB_ROUTE_LAZY != 0; otherwise such k fails with SB_EARG
 * "k too large for the routing kernel". */
int sb_route_batch(sb_index* idx, const double* qf, const double* qa, const double* qmask,
                   int64_t q, int32_t k, int32_t pioneer, int32_t use_coarse,
                   const int64_t* entries, uint64_t seed, int64_t qi0, double inv_alpha,
                   int64_t* out_ids, double* out_dists, int64_t* out_stats);

/* same, all pointers on the device, asynchronous on the handle's stream */
int sb_route_batch_dev(sb_index* idx, const double* qf, const double* qa, const double* qmask,
                       int64_t q, int32_t k, int32_t pioneer, int32_t use_coarse,
                       const int64_t* entries, uint64_t seed, int64_t qi0, double inv_alpha,
                       int64_t* out_ids, double* out_dists, int64_t* out_stats);

/* page-locked host memory (cudaHostAlloc) for inputs and results: copies to and from it run
 * at full link speed, asynchronously */
int sb_host_alloc(size_t bytes, void** out);
int sb_host_free(void* p);

/* number of kernel launches this handle issued since creation (instrumentation) */
int64_t sb_launch_count(sb_index* idx);

/* *int_exact = 1 when every feature is an integer (|x| <= *fmax_abs); such data admits exact
 * reduced-precision / reordered distance sums.  *last_bf_tc = 1 when the last
 * sb_bf_topk_queries ran on the tensor cores (tcgen05). */
int sb_index_info(sb_index* idx, int32_t* int_exact, double* fmax_abs, int32_t* last_bf_tc);
/* distance evaluation order for routing and exhaustive top-k: 0 = automatic (order-free
 * exact paths for integer data: u8/dp4a or fp32 routing rows, tensor-core top-k; the
 * certified fp32 routing filter for real-valued data), 1 = always
 * the sequential fp64 order of _query_dist (_kernels.py:26-35).  Both are bit-exact. */
int sb_set_distance_mode(sb_index* idx, int32_t mode);
/* the last sb_route_batch / sb_route_batch_dev on this handle: *path = 0 fp64 rows (d % 4 == 0),
 * 1 fp32 rows (integer data), 2 fp32 lane groups, 3 fp64 generic, 4 u8 rows with dp4a (integer
 * data in [0, 255]), 5 certified fp32 filter + exact fp64 rows for the survivors (real-valued
 * data, d % 4 == 0); *row_bytes = bytes read per feature row evaluated */
int sb_route_info(sb_index* idx, int32_t* path, int32_t* row_bytes);
/* the last sb_bf_topk_queries on this handle: *path = 0 exact fp64 kernel, 1 tcgen05 with exact
 * integer products (integer data), 2 tcgen05 TF32 filter with a certified error bound + exact
 * fp64 re-rank (other data); *candidates = pairs the TF32 filter passed to the re-rank (all
 * queries); *fallback = queries whose candidates overflowed and were recomputed on path 0;
 * *kernel_ms = duration of the tensor-core pass over all nodes (CUDA events on the handle's
 * stream; 0 on path 0).  Any pointer may be NULL.  Replaces nothing in the reference
 * (instrumentation of evaluate.py:32-55's replacement). */
int sb_bf_info(sb_index* idx, int32_t* path, int64_t* candidates, int64_t* fallback,
               double* kernel_ms);
/* Prepare the routing layout now instead of at the first routing call: the nodes renumbered
 * along a locality order (features, attributes and adjacency permuted; results, entries and
 * distance ties still use the original ids, so routing output is unchanged) and, for
 * integer data in [0, 255], the u8 feature copy.  SB_ROUTE_RELABEL=0 disables the layout. */
int sb_route_prepare(sb_index* idx);

#ifdef __cplusplus
}
#endif
#endif /* STABLE_B200_H */

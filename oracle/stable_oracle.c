/*
 * stable_oracle.c — TEST INFRASTRUCTURE ONLY (parity checker + CPU baseline).
 *
 * A plain-C restatement of the CPU reference's hot path (hybridann 0.1.0,
 * /root/reference/pkg/src/hybridann/_kernels.py, Numba @njit → x86).  Every
 * function cites the reference lines it restates.  Only tests/, smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library; the
 * product path (paper_2604_01617_b200) never links or calls it.
 *
 * Semantics are the reference's exactly: fp64 accumulation over fp32 inputs in
 * ascending-dimension order, stored build distances rounded to fp32, ties by
 * ascending id, in-place mutation of adjacency rows, sequential row order.
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py) — see tests/test_oracle_golden.py.
 *
 * Layouts (C-contiguous, as the reference passes them, _kernels.py:1-6):
 *   features f32[n*m]   attrs i32[n*l]
 *   nbr_ids i32[n*g]    nbr_dists f32[n*g]   nbr_flags u8[n*g]   nbr_counts i32[n]
 *
 * Two ways to run the build:
 *  - the or_* functions below the metric: the reference's loops one for one, sequential
 *    (what tests/test_oracle_golden.py pins against the reference's own outputs);
 *  - the or_*_x functions: the same results computed in parallel on the host cores (OpenMP),
 *    so the oracle can build 100k-2M node graphs in seconds to minutes.  Each one states why
 *    its order of work cannot change the result, and the tests pin
 *    every _x function bit-exact against its sequential twin.  The _x functions also accept
 *    an optional u8 copy of the features (F8, NULL = none) for data whose features are all
 *    integers in [0, 255]: then every partial sum of _pair_dist / _diff_cosine is an integer
 *    below 2^53, so an int32 sum converted to double IS the sequential fp64 sum, bit for bit.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#ifdef __AVX2__
#include <immintrin.h>
#endif

/* ---- metric (_kernels.py:14-35) -------------------------------------- */

/* the data a distance needs: fp32 features, optional exact u8 copy, attributes */
typedef struct {
    const float *F;
    const uint8_t *F8; /* NULL unless every feature is an integer in [0, 255] */
    const int32_t *A;
    int64_t m, l;
} feat_t;

/* _pair_dist (_kernels.py:14-23): sequential fp64 sums, then sqrt(s_v)*(1+s_a*inv_alpha). */
static inline double pair_dist(const float *F, const int32_t *A, int64_t m, int64_t l,
                               int64_t i, int64_t j, double inv_alpha) {
    const float *xi = F + i * m, *xj = F + j * m;
    double s_v = 0.0;
    for (int64_t t = 0; t < m; ++t) {
        double d = (double)xi[t] - (double)xj[t];
        s_v += d * d;
    }
    const int32_t *ai = A + i * l, *aj = A + j * l;
    double s_a = 0.0;
    for (int64_t t = 0; t < l; ++t) s_a += fabs((double)ai[t] - (double)aj[t]);
    return sqrt(s_v) * (1.0 + s_a * inv_alpha);
}

/* _query_dist (_kernels.py:26-35): query widened to fp64, per-dimension mask multiplier. */
static inline double query_dist(const float *F, const int32_t *A, int64_t m, int64_t l, int64_t v,
                                const double *qf, const double *qa, const double *qm,
                                double inv_alpha) {
    const float *x = F + v * m;
    double s_v = 0.0;
    for (int64_t t = 0; t < m; ++t) {
        double d = (double)x[t] - qf[t];
        s_v += d * d;
    }
    const int32_t *a = A + v * l;
    double s_a = 0.0;
    for (int64_t t = 0; t < l; ++t) s_a += qm[t] * fabs((double)a[t] - qa[t]);
    return sqrt(s_v) * (1.0 + s_a * inv_alpha);
}

/* ---- build-row push (_kernels.py:38-68) ------------------------------- */

/* _heap_push: replace the farthest entry of a full row if (f32 d, id) strictly beats it;
 * rejects self and duplicates; inserted entry gets flag 1. */
static inline int heap_push(int32_t *ids, float *dists, uint8_t *flags, int64_t g, int64_t row,
                            int32_t cand, double dd) {
    if (cand == row) return 0;
    float d = (float)dd;                       /* compare in stored precision (line 48) */
    int32_t *ri = ids + row * g;
    float *rd = dists + row * g;
    uint8_t *rf = flags + row * g;
    float wd = rd[g - 1];
    if (d > wd || (d == wd && cand >= ri[g - 1])) return 0;
    for (int64_t t = 0; t < g; ++t)
        if (ri[t] == cand) return 0;
    int64_t pos = g - 1;
    while (pos > 0 && (rd[pos - 1] > d || (rd[pos - 1] == d && ri[pos - 1] > cand))) {
        ri[pos] = ri[pos - 1];
        rd[pos] = rd[pos - 1];
        rf[pos] = rf[pos - 1];
        --pos;
    }
    ri[pos] = cand;
    rd[pos] = d;
    rf[pos] = 1;
    return 1;
}

/* compute_row_distances (_kernels.py:71-78). */
void or_compute_row_distances(const float *F, const int32_t *A, int64_t n, int64_t m, int64_t l,
                              const int32_t *ids, int64_t g, double inv_alpha, float *out) {
    for (int64_t i = 0; i < n; ++i)
        for (int64_t t = 0; t < g; ++t)
            out[i * g + t] = (float)pair_dist(F, A, m, l, i, ids[i * g + t], inv_alpha);
}

/* build_candidates (_kernels.py:81-135).  Outputs must be pre-sized:
 * new_cand i32[n*gn], old_cand i32[n*g] (filled with -1 here), counts i32[n]. */
void or_build_candidates(const int32_t *ids, uint8_t *flags, int64_t n, int64_t g, int64_t gn,
                         int32_t *new_cand, int32_t *new_counts, int32_t *old_cand,
                         int32_t *old_counts) {
    for (int64_t i = 0; i < n * gn; ++i) new_cand[i] = -1;
    for (int64_t i = 0; i < n * g; ++i) old_cand[i] = -1;
    for (int64_t i = 0; i < n; ++i) { new_counts[i] = 0; old_counts[i] = 0; }
    /* forward split, list order (lines 95-109) */
    for (int64_t i = 0; i < n; ++i) {
        int32_t c = 0;
        for (int64_t t = 0; t < g; ++t) {
            int32_t j = ids[i * g + t];
            if (flags[i * g + t] == 1) {
                new_cand[i * gn + c] = j;
                flags[i * g + t] = 0;
                ++c;
                if (c >= gn) break;
            } else if (old_counts[i] < g) {
                old_cand[i * g + old_counts[i]] = j;
                old_counts[i] += 1;
            }
        }
        new_counts[i] = c;
    }
    /* reverse union in ascending source order (lines 110-134) */
    int32_t *fwd_new = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int32_t *fwd_old = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    memcpy(fwd_new, new_counts, sizeof(int32_t) * (size_t)n);
    memcpy(fwd_old, old_counts, sizeof(int32_t) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        for (int32_t x = 0; x < fwd_new[i]; ++x) {
            int32_t j = new_cand[i * gn + x];
            if (new_counts[j] < gn) {
                int dup = 0;
                for (int32_t t = 0; t < new_counts[j]; ++t)
                    if (new_cand[(int64_t)j * gn + t] == i) { dup = 1; break; }
                if (!dup) new_cand[(int64_t)j * gn + new_counts[j]++] = (int32_t)i;
            }
        }
        for (int32_t x = 0; x < fwd_old[i]; ++x) {
            int32_t j = old_cand[i * g + x];
            if (old_counts[j] < g) {
                int dup = 0;
                for (int32_t t = 0; t < old_counts[j]; ++t)
                    if (old_cand[(int64_t)j * g + t] == i) { dup = 1; break; }
                if (!dup) old_cand[(int64_t)j * g + old_counts[j]++] = (int32_t)i;
            }
        }
    }
    free(fwd_new);
    free(fwd_old);
}

/* local_join (_kernels.py:138-173): sequential pair loop with two pushes per pair.
 * Also counts evaluated pairs into *pairs_out (instrumentation, may be NULL). */
int64_t or_local_join(const float *F, const int32_t *A, int64_t n, int64_t m, int64_t l,
                      double inv_alpha, const int32_t *new_cand, const int32_t *new_counts,
                      int64_t gn, const int32_t *old_cand, const int32_t *old_counts,
                      int32_t *ids, float *dists, uint8_t *flags, int64_t g, int64_t *pairs_out) {
    int64_t changes = 0, pairs = 0;
    for (int64_t i = 0; i < n; ++i) {
        int32_t na = new_counts[i], nb = old_counts[i];
        const int32_t *nw = new_cand + i * gn, *od = old_cand + i * g;
        for (int32_t x = 0; x < na; ++x) {
            int32_t j = nw[x];
            for (int32_t y = x + 1; y < na; ++y) {
                int32_t k = nw[y];
                if (j == k) continue;
                double d = pair_dist(F, A, m, l, j, k, inv_alpha);
                ++pairs;
                changes += heap_push(ids, dists, flags, g, j, k, d);
                changes += heap_push(ids, dists, flags, g, k, j, d);
            }
            for (int32_t y = 0; y < nb; ++y) {
                int32_t k = od[y];
                if (j == k) continue;
                double d = pair_dist(F, A, m, l, j, k, inv_alpha);
                ++pairs;
                changes += heap_push(ids, dists, flags, g, j, k, d);
                changes += heap_push(ids, dists, flags, g, k, j, d);
            }
        }
    }
    if (pairs_out) *pairs_out = pairs;
    return changes;
}

/* brute_force_topk (_kernels.py:176-204): per sample u, exact top-k over v != u,
 * running insertion sort in fp64 by (d, id); ids padded with -1.  Parallel over
 * samples exactly like the reference's prange (each sample is independent). */
void or_brute_force_topk(const float *F, const int32_t *A, int64_t n, int64_t m, int64_t l,
                         double inv_alpha, const int64_t *sample_ids, int64_t s, int64_t k,
                         int32_t *out_ids) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t si = 0; si < s; ++si) {
        int64_t u = sample_ids[si];
        double *bd = (double *)malloc(sizeof(double) * (size_t)k);
        int64_t *bi = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
        for (int64_t t = 0; t < k; ++t) { bd[t] = INFINITY; bi[t] = n; }
        for (int64_t v = 0; v < n; ++v) {
            if (v == u) continue;
            double d = pair_dist(F, A, m, l, u, v, inv_alpha);
            double wd = bd[k - 1];
            if (d > wd || (d == wd && v >= bi[k - 1])) continue;
            int64_t pos = k - 1;
            while (pos > 0 && (bd[pos - 1] > d || (bd[pos - 1] == d && bi[pos - 1] > v))) {
                bd[pos] = bd[pos - 1];
                bi[pos] = bi[pos - 1];
                --pos;
            }
            bd[pos] = d;
            bi[pos] = v;
        }
        for (int64_t t = 0; t < k; ++t) out_ids[si * k + t] = bi[t] < n ? (int32_t)bi[t] : -1;
        free(bd);
        free(bi);
    }
}

/* graph_quality (_kernels.py:207-224): sequential fp64 mean of hits/k. */
double or_graph_quality(const int32_t *ids, const int32_t *counts, int64_t g,
                        const int64_t *sample_ids, int64_t s, const int32_t *gt, int64_t k) {
    double total = 0.0;
    for (int64_t si = 0; si < s; ++si) {
        int64_t u = sample_ids[si];
        int64_t c = counts[u] < k ? counts[u] : k;
        int64_t hits = 0;
        for (int64_t t = 0; t < c; ++t) {
            int32_t x = ids[u * g + t];
            for (int64_t y = 0; y < k; ++y)
                if (gt[si * k + y] == x) { ++hits; break; }
        }
        total += (double)hits / (double)k;
    }
    return total / (double)s;
}

/* _attrs_equal (_kernels.py:227-232). */
static inline int attrs_equal(const int32_t *A, int64_t l, int64_t a, int64_t b) {
    for (int64_t t = 0; t < l; ++t)
        if (A[a * l + t] != A[b * l + t]) return 0;
    return 1;
}

/* _diff_cosine (_kernels.py:235-253): cos angle of (p-s, k-s), 1.0 for zero-length offsets. */
static inline double diff_cosine(const float *F, int64_t m, int64_t s, int64_t p, int64_t k) {
    const float *xs = F + s * m, *xp = F + p * m, *xk = F + k * m;
    double dot = 0.0, np2 = 0.0, nk2 = 0.0;
    for (int64_t t = 0; t < m; ++t) {
        double dp = (double)xp[t] - (double)xs[t];
        double dk = (double)xk[t] - (double)xs[t];
        dot += dp * dk;
        np2 += dp * dp;
        nk2 += dk * dk;
    }
    if (np2 == 0.0 || nk2 == 0.0) return 1.0;
    return dot / sqrt(np2 * nk2);
}

/* _pair_dist over feat_t: the u8 path sums exact integers (equal to the sequential fp64 sum,
 * see the header), the fp32 path is pair_dist above. */
/* exact integer sums over u8 rows: sum (a-b)^2, and the three sums of _diff_cosine */
static inline int32_t u8_l2(const uint8_t *a, const uint8_t *b, int64_t m) {
    int64_t t = 0;
    int32_t s = 0;
#ifdef __AVX2__
    __m256i acc = _mm256_setzero_si256();
    for (; t + 16 <= m; t += 16) {
        __m256i x = _mm256_cvtepu8_epi16(_mm_loadu_si128((const __m128i *)(a + t)));
        __m256i y = _mm256_cvtepu8_epi16(_mm_loadu_si128((const __m128i *)(b + t)));
        __m256i d = _mm256_sub_epi16(x, y);
        acc = _mm256_add_epi32(acc, _mm256_madd_epi16(d, d));
    }
    __m128i h = _mm_add_epi32(_mm256_castsi256_si128(acc), _mm256_extracti128_si256(acc, 1));
    h = _mm_add_epi32(h, _mm_shuffle_epi32(h, 0x4E));
    h = _mm_add_epi32(h, _mm_shuffle_epi32(h, 0xB1));
    s = _mm_cvtsi128_si32(h);
#endif
    for (; t < m; ++t) {
        int32_t d = (int32_t)a[t] - (int32_t)b[t];
        s += d * d;
    }
    return s;
}

static inline void u8_cos3(const uint8_t *xs, const uint8_t *xp, const uint8_t *xk, int64_t m,
                           int32_t *dot, int32_t *np2, int32_t *nk2) {
    int64_t t = 0;
    int32_t sd = 0, sp = 0, sk = 0;
#ifdef __AVX2__
    __m256i ad = _mm256_setzero_si256(), ap = ad, ak = ad;
    for (; t + 16 <= m; t += 16) {
        __m256i s0 = _mm256_cvtepu8_epi16(_mm_loadu_si128((const __m128i *)(xs + t)));
        __m256i dp = _mm256_sub_epi16(_mm256_cvtepu8_epi16(_mm_loadu_si128((const __m128i *)(xp + t))), s0);
        __m256i dk = _mm256_sub_epi16(_mm256_cvtepu8_epi16(_mm_loadu_si128((const __m128i *)(xk + t))), s0);
        ad = _mm256_add_epi32(ad, _mm256_madd_epi16(dp, dk));
        ap = _mm256_add_epi32(ap, _mm256_madd_epi16(dp, dp));
        ak = _mm256_add_epi32(ak, _mm256_madd_epi16(dk, dk));
    }
    int32_t buf[8];
    _mm256_storeu_si256((__m256i *)buf, ad);
    for (int i = 0; i < 8; ++i) sd += buf[i];
    _mm256_storeu_si256((__m256i *)buf, ap);
    for (int i = 0; i < 8; ++i) sp += buf[i];
    _mm256_storeu_si256((__m256i *)buf, ak);
    for (int i = 0; i < 8; ++i) sk += buf[i];
#endif
    for (; t < m; ++t) {
        int32_t dp = (int32_t)xp[t] - (int32_t)xs[t];
        int32_t dk = (int32_t)xk[t] - (int32_t)xs[t];
        sd += dp * dk;
        sp += dp * dp;
        sk += dk * dk;
    }
    *dot = sd;
    *np2 = sp;
    *nk2 = sk;
}

static inline double fpair_dist(const feat_t *f, int64_t i, int64_t j, double inv_alpha) {
    if (!f->F8) return pair_dist(f->F, f->A, f->m, f->l, i, j, inv_alpha);
    int32_t s = u8_l2(f->F8 + i * f->m, f->F8 + j * f->m, f->m);
    const int32_t *ai = f->A + i * f->l, *aj = f->A + j * f->l;
    double s_a = 0.0;
    for (int64_t t = 0; t < f->l; ++t) s_a += fabs((double)ai[t] - (double)aj[t]);
    return sqrt((double)s) * (1.0 + s_a * inv_alpha);
}

/* _pair_dist of row j against four rows k[0..3] at once (fp32 features): each AVX2 lane
 * carries one pair's own sequential fp64 chain, t ascending, multiply and add separately
 * rounded (no FMA), so every lane equals pair_dist bit for bit. */
static inline void fpair_dist4(const feat_t *f, int64_t j, const int32_t *k, double inv_alpha,
                               double out[4]) {
    if (f->F8) {
        for (int u = 0; u < 4; ++u) out[u] = fpair_dist(f, j, k[u], inv_alpha);
        return;
    }
    const int64_t m = f->m;
    const float *xj = f->F + j * m;
    const float *x0 = f->F + (int64_t)k[0] * m, *x1 = f->F + (int64_t)k[1] * m;
    const float *x2 = f->F + (int64_t)k[2] * m, *x3 = f->F + (int64_t)k[3] * m;
    double acc[4];
    int64_t t = 0;
#ifdef __AVX2__
    __m256d s = _mm256_setzero_pd();
    for (; t + 4 <= m; t += 4) {
        __m256d r0 = _mm256_cvtps_pd(_mm_loadu_ps(x0 + t));
        __m256d r1 = _mm256_cvtps_pd(_mm_loadu_ps(x1 + t));
        __m256d r2 = _mm256_cvtps_pd(_mm_loadu_ps(x2 + t));
        __m256d r3 = _mm256_cvtps_pd(_mm_loadu_ps(x3 + t));
        /* transpose: c_u = (x0[t+u], x1[t+u], x2[t+u], x3[t+u]) */
        __m256d a01l = _mm256_unpacklo_pd(r0, r1), a01h = _mm256_unpackhi_pd(r0, r1);
        __m256d a23l = _mm256_unpacklo_pd(r2, r3), a23h = _mm256_unpackhi_pd(r2, r3);
        __m256d c0 = _mm256_permute2f128_pd(a01l, a23l, 0x20);
        __m256d c1 = _mm256_permute2f128_pd(a01h, a23h, 0x20);
        __m256d c2 = _mm256_permute2f128_pd(a01l, a23l, 0x31);
        __m256d c3 = _mm256_permute2f128_pd(a01h, a23h, 0x31);
        __m256d d;
        d = _mm256_sub_pd(_mm256_set1_pd((double)xj[t]), c0);
        s = _mm256_add_pd(s, _mm256_mul_pd(d, d));
        d = _mm256_sub_pd(_mm256_set1_pd((double)xj[t + 1]), c1);
        s = _mm256_add_pd(s, _mm256_mul_pd(d, d));
        d = _mm256_sub_pd(_mm256_set1_pd((double)xj[t + 2]), c2);
        s = _mm256_add_pd(s, _mm256_mul_pd(d, d));
        d = _mm256_sub_pd(_mm256_set1_pd((double)xj[t + 3]), c3);
        s = _mm256_add_pd(s, _mm256_mul_pd(d, d));
    }
    _mm256_storeu_pd(acc, s);
#else
    acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
#endif
    const float *xs[4] = {x0, x1, x2, x3};
    for (int u = 0; u < 4; ++u) {
        double a = acc[u];
        for (int64_t tt = t; tt < m; ++tt) {
            double d = (double)xj[tt] - (double)xs[u][tt];
            a += d * d;
        }
        const int32_t *ai = f->A + j * f->l, *ak = f->A + (int64_t)k[u] * f->l;
        double s_a = 0.0;
        for (int64_t q = 0; q < f->l; ++q) s_a += fabs((double)ai[q] - (double)ak[q]);
        out[u] = sqrt(a) * (1.0 + s_a * inv_alpha);
    }
}

/* _diff_cosine over feat_t (u8 path: exact integer dot products, then the same fp64 finish) */
static inline double fdiff_cosine(const feat_t *f, int64_t s, int64_t p, int64_t k) {
    if (!f->F8) return diff_cosine(f->F, f->m, s, p, k);
    int32_t dot, np2, nk2;
    u8_cos3(f->F8 + s * f->m, f->F8 + p * f->m, f->F8 + k * f->m, f->m, &dot, &np2, &nk2);
    if (np2 == 0 || nk2 == 0) return 1.0;
    return (double)dot / sqrt((double)np2 * (double)nk2);
}

/* count_in_degrees (_kernels.py:256-263). */
void or_count_in_degrees(const int32_t *ids, const int32_t *counts, int64_t n, int64_t g,
                         int64_t *in_deg) {
    for (int64_t i = 0; i < n; ++i) in_deg[i] = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int32_t t = 0; t < counts[i]; ++t) in_deg[ids[i * g + t]] += 1;
}

/* prune_pass (_kernels.py:266-303): rows in ascending order, in-degree safeguard. */
void or_prune_pass(const float *F, const int32_t *A, int64_t n, int64_t m, int64_t l,
                   int32_t *ids, float *dists, int32_t *counts, int64_t g, int64_t *in_deg,
                   double sigma) {
    uint8_t *keep = (uint8_t *)malloc((size_t)g);
    for (int64_t s = 0; s < n; ++s) {
        int32_t cnt = counts[s];
        if (cnt <= 1) continue;
        int32_t *ri = ids + s * g;
        float *rd = dists + s * g;
        memset(keep, 0, (size_t)cnt);
        keep[0] = 1;
        for (int32_t t = 1; t < cnt; ++t) {
            int32_t p = ri[t];
            int redundant = 0;
            for (int32_t u = 0; u < t; ++u) {
                if (!keep[u]) continue;
                int32_t kk = ri[u];
                if (attrs_equal(A, l, p, kk) && diff_cosine(F, m, s, p, kk) > sigma) {
                    redundant = 1;
                    break;
                }
            }
            if (redundant && in_deg[p] >= 2) in_deg[p] -= 1;
            else keep[t] = 1;
        }
        int32_t w = 0;
        for (int32_t t = 0; t < cnt; ++t)
            if (keep[t]) { ri[w] = ri[t]; rd[w] = rd[t]; ++w; }
        counts[s] = w;
    }
    free(keep);
}

/* _try_insert_edge (_kernels.py:306-395): insert j->cand; full rows merge + re-prune
 * under the safeguard, then drop the farthest safe entry.  Returns 1 if inserted. */
static int try_insert_edge(const feat_t *f, int32_t *ids,
                           float *dists, int32_t *counts, int64_t g, int64_t *in_deg, int64_t j,
                           int64_t cand, double dd, double sigma, int64_t *tmp_ids,
                           double *tmp_dists, uint8_t *keep) {
    float d = (float)dd;
    int32_t *ri = ids + j * g;
    float *rd = dists + j * g;
    int32_t cj = counts[j];
    for (int32_t t = 0; t < cj; ++t)
        if (ri[t] == cand) return 0;
    if (cj < g) {
        int32_t pos = cj;
        while (pos > 0 && (rd[pos - 1] > d || (rd[pos - 1] == d && ri[pos - 1] > cand))) {
            ri[pos] = ri[pos - 1];
            rd[pos] = rd[pos - 1];
            --pos;
        }
        ri[pos] = (int32_t)cand;
        rd[pos] = d;
        counts[j] = cj + 1;
        in_deg[cand] += 1;
        return 1;
    }
    /* full: scratch list of g+1 in fp64 keys (lines 337-351) */
    int32_t pos = cj;
    for (int32_t t = 0; t < cj; ++t) { tmp_ids[t] = ri[t]; tmp_dists[t] = (double)rd[t]; }
    while (pos > 0 && (tmp_dists[pos - 1] > (double)d ||
                       (tmp_dists[pos - 1] == (double)d && tmp_ids[pos - 1] > cand))) {
        tmp_ids[pos] = tmp_ids[pos - 1];
        tmp_dists[pos] = tmp_dists[pos - 1];
        --pos;
    }
    tmp_ids[pos] = cand;
    tmp_dists[pos] = (double)d;
    int32_t total = cj + 1;
    for (int32_t t = 0; t < total; ++t) keep[t] = 1;
    int32_t kept = 1;
    for (int32_t t = 1; t < total; ++t) {
        int64_t p = tmp_ids[t];
        int redundant = 0;
        for (int32_t u = 0; u < t; ++u) {
            if (!keep[u]) continue;
            int64_t kk = tmp_ids[u];
            if (attrs_equal(f->A, f->l, p, kk) && fdiff_cosine(f, j, p, kk) > sigma) {
                redundant = 1;
                break;
            }
        }
        if (redundant && (p == cand || in_deg[p] >= 2)) {
            keep[t] = 0;
            if (p != cand) in_deg[p] -= 1;
        } else {
            ++kept;
        }
    }
    if (kept > g) {
        for (int32_t t = total - 1; t >= 0; --t) {
            if (!keep[t]) continue;
            int64_t p = tmp_ids[t];
            if (p == cand) { keep[t] = 0; break; }
            if (in_deg[p] >= 2) { keep[t] = 0; in_deg[p] -= 1; break; }
        }
    }
    int32_t w = 0;
    int inserted = 0;
    for (int32_t t = 0; t < total; ++t) {
        if (!keep[t]) continue;
        ri[w] = (int32_t)tmp_ids[t];
        rd[w] = (float)tmp_dists[t];
        if (tmp_ids[t] == cand) inserted = 1;
        ++w;
    }
    counts[j] = w;
    if (inserted) in_deg[cand] += 1;
    return inserted;
}

/* reinforce_pass (_kernels.py:398-409).  Returns the number of full-row merges
 * (instrumentation: 0 means reinforce acted as plain symmetrisation). */
static int64_t reinforce_pass(const feat_t *f, int64_t n, int32_t *ids, float *dists,
                              int32_t *counts, int64_t g, int64_t *in_deg, double sigma) {
    int64_t *tmp_ids = (int64_t *)malloc(sizeof(int64_t) * (size_t)(g + 1));
    double *tmp_dists = (double *)malloc(sizeof(double) * (size_t)(g + 1));
    uint8_t *keep = (uint8_t *)malloc((size_t)(g + 1));
    int64_t full_merges = 0;
    for (int64_t s = 0; s < n; ++s) {
        int32_t cs = counts[s];
        for (int32_t t = 0; t < cs; ++t) {
            if (t >= counts[s]) break; /* row may shrink while being mirrored (line 405) */
            int32_t j = ids[s * g + t];
            double d = (double)dists[s * g + t];
            if (counts[j] >= g) {
                int present = 0;
                for (int32_t u = 0; u < counts[j]; ++u)
                    if (ids[(int64_t)j * g + u] == s) { present = 1; break; }
                if (!present) ++full_merges;
            }
            try_insert_edge(f, ids, dists, counts, g, in_deg, j, s, d, sigma, tmp_ids,
                            tmp_dists, keep);
        }
    }
    free(tmp_ids);
    free(tmp_dists);
    free(keep);
    return full_merges;
}

int64_t or_reinforce_pass(const float *F, const int32_t *A, int64_t n, int64_t m, int64_t l,
                          int32_t *ids, float *dists, int32_t *counts, int64_t g, int64_t *in_deg,
                          double sigma) {
    feat_t f = {F, NULL, A, m, l};
    return reinforce_pass(&f, n, ids, dists, counts, g, in_deg, sigma);
}

/* reinforce_pass with the optional exact u8 features (sequential: the overflow re-prune makes
 * the order of mirrored edges matter, _kernels.py:336-395). */
int64_t or_reinforce_pass_x(const float *F, const uint8_t *F8, const int32_t *A, int64_t n,
                            int64_t m, int64_t l, int32_t *ids, float *dists, int32_t *counts,
                            int64_t g, int64_t *in_deg, double sigma) {
    feat_t f = {F, F8, A, m, l};
    return reinforce_pass(&f, n, ids, dists, counts, g, in_deg, sigma);
}

/* _force_insert_edge (_kernels.py:412-452). */
static int force_insert_edge(int32_t *ids, float *dists, int32_t *counts, int64_t g,
                             int64_t *in_deg, int64_t j, int64_t cand, double dd,
                             int allow_unsafe) {
    float d = (float)dd;
    int32_t *ri = ids + j * g;
    float *rd = dists + j * g;
    int32_t cj = counts[j];
    for (int32_t t = 0; t < cj; ++t)
        if (ri[t] == cand) return 0;
    if (cj >= g) {
        int32_t evict = -1;
        for (int32_t t = cj - 1; t >= 0; --t)
            if (in_deg[ri[t]] >= 2) { evict = t; break; }
        if (evict < 0) {
            if (!allow_unsafe) return 0;
            evict = cj - 1;
        }
        in_deg[ri[evict]] -= 1;
        for (int32_t t = evict; t < cj - 1; ++t) { ri[t] = ri[t + 1]; rd[t] = rd[t + 1]; }
        --cj;
    }
    int32_t pos = cj;
    while (pos > 0 && (rd[pos - 1] > d || (rd[pos - 1] == d && ri[pos - 1] > cand))) {
        ri[pos] = ri[pos - 1];
        rd[pos] = rd[pos - 1];
        --pos;
    }
    ri[pos] = (int32_t)cand;
    rd[pos] = d;
    counts[j] = cj + 1;
    in_deg[cand] += 1;
    return 1;
}

/* reconnect_islands (_kernels.py:455-487). */
static void reconnect_islands(const feat_t *f, int64_t n, int32_t *ids, float *dists,
                              int32_t *counts, int64_t g, int64_t *in_deg, double sigma) {
    int64_t *tmp_ids = (int64_t *)malloc(sizeof(int64_t) * (size_t)(g + 1));
    double *tmp_dists = (double *)malloc(sizeof(double) * (size_t)(g + 1));
    uint8_t *keep = (uint8_t *)malloc((size_t)(g + 1));
    for (int64_t v = 0; v < n; ++v) {
        if (in_deg[v] > 0) continue;
        int done = 0;
        for (int32_t t = 0; t < counts[v]; ++t) {
            int64_t u = ids[v * g + t];
            double d = (double)dists[v * g + t];
            if (try_insert_edge(f, ids, dists, counts, g, in_deg, u, v, d, sigma,
                                tmp_ids, tmp_dists, keep)) { done = 1; break; }
        }
        if (done) continue;
        for (int32_t t = 0; t < counts[v]; ++t) {
            int64_t u = ids[v * g + t];
            double d = (double)dists[v * g + t];
            if (force_insert_edge(ids, dists, counts, g, in_deg, u, v, d, 0)) { done = 1; break; }
        }
        if (!done && counts[v] > 0)
            force_insert_edge(ids, dists, counts, g, in_deg, ids[v * g], v,
                              (double)dists[v * g], 1);
    }
    free(tmp_ids);
    free(tmp_dists);
    free(keep);
}

void or_reconnect_islands(const float *F, const int32_t *A, int64_t n, int64_t m, int64_t l,
                          int32_t *ids, float *dists, int32_t *counts, int64_t g,
                          int64_t *in_deg, double sigma) {
    feat_t f = {F, NULL, A, m, l};
    reconnect_islands(&f, n, ids, dists, counts, g, in_deg, sigma);
}

void or_reconnect_islands_x(const float *F, const uint8_t *F8, const int32_t *A, int64_t n,
                            int64_t m, int64_t l, int32_t *ids, float *dists, int32_t *counts,
                            int64_t g, int64_t *in_deg, double sigma) {
    feat_t f = {F, F8, A, m, l};
    reconnect_islands(&f, n, ids, dists, counts, g, in_deg, sigma);
}

/* _list_insert (_kernels.py:490-501). */
static inline void list_insert(int64_t *ids, double *dists, uint8_t *checked, int64_t size,
                               int64_t cand, double d) {
    int64_t pos = size - 1;
    while (pos > 0 && (dists[pos - 1] > d || (dists[pos - 1] == d && ids[pos - 1] > cand))) {
        ids[pos] = ids[pos - 1];
        dists[pos] = dists[pos - 1];
        checked[pos] = checked[pos - 1];
        --pos;
    }
    ids[pos] = cand;
    dists[pos] = d;
    checked[pos] = 0;
}

/* route (_kernels.py:504-610): two-phase routing for one query.
 * visited: caller scratch u8[n] zeroed on entry (left dirty on exit).
 * stats: i64[4] = evals, phase1_evals, phase1_expansions, hops. */
static void route_one(const float *F, const int32_t *A, int64_t n, int64_t m, int64_t l,
                      const int32_t *nbr_ids, const int32_t *nbr_counts, int64_t g,
                      const double *qf, const double *qa, const double *qm, double inv_alpha,
                      const int64_t *entries, int64_t k, int64_t p, int use_coarse,
                      int64_t *r_ids, double *r_dists, int64_t *stats, uint8_t *visited,
                      uint8_t *r_checked, int64_t *p_ids, double *p_dists, uint8_t *p_checked) {
    (void)n;
    int64_t evals = 0, p1_evals = 0, p1_exp = 0, hops = 0;
    for (int64_t t = 0; t < k; ++t) {
        int64_t v = entries[t];
        visited[v] = 1;
        r_ids[t] = v;
        r_dists[t] = query_dist(F, A, m, l, v, qf, qa, qm, inv_alpha);
        ++evals;
        r_checked[t] = 0;
    }
    for (int64_t t = 1; t < k; ++t) { /* insertion sort by (d, id), lines 542-551 */
        int64_t cid = r_ids[t];
        double cd = r_dists[t];
        int64_t pos = t;
        while (pos > 0 && (r_dists[pos - 1] > cd || (r_dists[pos - 1] == cd && r_ids[pos - 1] > cid))) {
            r_ids[pos] = r_ids[pos - 1];
            r_dists[pos] = r_dists[pos - 1];
            --pos;
        }
        r_ids[pos] = cid;
        r_dists[pos] = cd;
    }
    if (use_coarse) { /* phase 1, lines 556-585 */
        for (int64_t t = 0; t < p; ++t) { p_ids[t] = r_ids[t]; p_dists[t] = r_dists[t]; p_checked[t] = 0; }
        for (;;) {
            int64_t sel = -1;
            for (int64_t t = 0; t < p; ++t)
                if (!p_checked[t]) { sel = t; break; }
            if (sel < 0) break;
            p_checked[sel] = 1;
            int64_t node = p_ids[sel];
            ++p1_exp;
            int32_t deg = nbr_counts[node];
            int32_t half = (deg + 1) / 2;
            for (int32_t t = 0; t < half; ++t) {
                int64_t nb = nbr_ids[node * g + t];
                if (visited[nb]) continue;
                visited[nb] = 1;
                double d = query_dist(F, A, m, l, nb, qf, qa, qm, inv_alpha);
                ++evals;
                ++p1_evals;
                if (d < r_dists[k - 1] || (d == r_dists[k - 1] && nb < r_ids[k - 1]))
                    list_insert(r_ids, r_dists, r_checked, k, nb, d);
                if (d < p_dists[p - 1] || (d == p_dists[p - 1] && nb < p_ids[p - 1]))
                    list_insert(p_ids, p_dists, p_checked, p, nb, d);
            }
        }
    }
    for (int64_t t = 0; t < k; ++t) r_checked[t] = 0; /* phase 2, lines 587-609 */
    for (;;) {
        int64_t sel = -1;
        for (int64_t t = 0; t < k; ++t)
            if (!r_checked[t]) { sel = t; break; }
        if (sel < 0) break;
        r_checked[sel] = 1;
        int64_t node = r_ids[sel];
        ++hops;
        int32_t deg = nbr_counts[node];
        for (int32_t t = 0; t < deg; ++t) {
            int64_t nb = nbr_ids[node * g + t];
            if (visited[nb]) continue;
            visited[nb] = 1;
            double d = query_dist(F, A, m, l, nb, qf, qa, qm, inv_alpha);
            ++evals;
            if (d < r_dists[k - 1] || (d == r_dists[k - 1] && nb < r_ids[k - 1]))
                list_insert(r_ids, r_dists, r_checked, k, nb, d);
        }
    }
    stats[0] = evals;
    stats[1] = p1_evals;
    stats[2] = p1_exp;
    stats[3] = hops;
}

/* route over a batch of q queries (the reference's search_batch loop, router.py:98-124,
 * with the query widened to fp64 as router.py:62-73 does).  qmask may be NULL (all ones).
 * Queries are independent, so threads split the batch (nthreads <= 0: all cores). */
void or_route_batch(const float *F, const int32_t *A, int64_t n, int64_t m, int64_t l,
                    const int32_t *nbr_ids, const int32_t *nbr_counts, int64_t g,
                    const double *qf, const double *qa, const double *qm, int64_t q,
                    double inv_alpha, const int64_t *entries, int64_t k, int64_t p,
                    int use_coarse, int64_t *out_ids, double *out_dists, int64_t *stats,
                    int nthreads) {
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#else
    nthreads = 1;
#endif
#pragma omp parallel num_threads(nthreads)
    {
        uint8_t *visited = (uint8_t *)calloc((size_t)n, 1);
        uint8_t *r_checked = (uint8_t *)malloc((size_t)k);
        int64_t *p_ids = (int64_t *)malloc(sizeof(int64_t) * (size_t)p);
        double *p_dists = (double *)malloc(sizeof(double) * (size_t)p);
        uint8_t *p_checked = (uint8_t *)malloc((size_t)p);
        double *ones = (double *)malloc(sizeof(double) * (size_t)(l > 0 ? l : 1));
        for (int64_t t = 0; t < l; ++t) ones[t] = 1.0;
#pragma omp for schedule(dynamic, 4)
        for (int64_t qi = 0; qi < q; ++qi) {
            memset(visited, 0, (size_t)n);
            route_one(F, A, n, m, l, nbr_ids, nbr_counts, g, qf + qi * m, qa + qi * l,
                      qm ? qm + qi * l : ones, inv_alpha, entries + qi * k, k, p, use_coarse,
                      out_ids + qi * k, out_dists + qi * k, stats + qi * 4, visited, r_checked,
                      p_ids, p_dists, p_checked);
        }
        free(visited); free(r_checked); free(p_ids); free(p_dists); free(p_checked); free(ones);
    }
}

/* ---- oracle_auto_topk (evaluate.py:32-55) -----------------------------------
 * The reference computes s_v with NumPy's add.reduce over axis 1 of a C-contiguous
 * fp64 array, which is NumPy's pairwise summation of the whole row (8-way unrolled
 * blocks of <= 128, split in halves above that); restated here so fused values match
 * bit for bit (checked against NumPy in tests/test_oracle_golden.py).
 * s_a: int64 Manhattan (optionally masked, int64 mask), then s_v*(1+s_a/alpha). */
static double np_pairwise(const double *a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; ++i) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return np_pairwise(a, n2) + np_pairwise(a + n2, n - n2);
    }
}

double or_np_row_sum(const double *a, int64_t n) {
    return np_pairwise(a, n);
}

/* fused distances of every node against one query (evaluate.py:47-53). */
void or_fused_all(const float *F, const int32_t *A, int64_t n, int64_t m, int64_t l,
                  const double *qf, const int64_t *qa, const int64_t *qmask, double alpha,
                  double *out) {
#pragma omp parallel
    {
        double *sq = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
#pragma omp for schedule(static)
        for (int64_t v = 0; v < n; ++v) {
            const float *x = F + v * m;
            for (int64_t t = 0; t < m; ++t) {
                double d = (double)x[t] - qf[t];
                sq[t] = d * d;
            }
            double s_v = sqrt(or_np_row_sum(sq, m));
            int64_t sa = 0;
            for (int64_t t = 0; t < l; ++t) {
                int64_t ad = (int64_t)A[v * l + t] - qa[t];
                if (ad < 0) ad = -ad;
                sa += qmask ? ad * qmask[t] : ad;
            }
            out[v] = s_v * (1.0 + (double)sa / alpha);
        }
        free(sq);
    }
}

/* =====================================================================================
 * Parallel restatements of the build (OpenMP, all host cores).  Each _x function returns
 * exactly what its sequential twin above returns; tests/test_oracle_golden.py pins that.
 * nthreads <= 0 means all cores.  F8 may be NULL (see the header).
 * ===================================================================================== */

static int omp_threads(int nthreads) {
#ifdef _OPENMP
    return nthreads > 0 ? nthreads : omp_get_max_threads();
#else
    (void)nthreads;
    return 1;
#endif
}

/* compute_row_distances (_kernels.py:71-78): every (i, t) entry is independent. */
void or_compute_row_distances_x(const float *F, const uint8_t *F8, const int32_t *A, int64_t n,
                                int64_t m, int64_t l, const int32_t *ids, int64_t g,
                                double inv_alpha, float *out, int nthreads) {
    feat_t f = {F, F8, A, m, l};
#pragma omp parallel for schedule(static) num_threads(omp_threads(nthreads))
    for (int64_t i = 0; i < n; ++i)
        for (int64_t t = 0; t < g; ++t)
            out[i * g + t] = (float)fpair_dist(&f, i, ids[i * g + t], inv_alpha);
}

/* reverse union of build_candidates for one list kind: row j gains sources i (ascending) while
 * it has room and i is not already in it.  Row j changes only through its own appends (row i is
 * read only in its forward prefix, which appends never touch), so targets are independent. */
static void reverse_union(const int32_t *fwd, int64_t n, int64_t cap, int32_t *cand,
                          int32_t *counts, int nthreads) {
    int64_t *off = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i)
        for (int32_t x = 0; x < fwd[i]; ++x) off[cand[i * cap + x] + 1] += 1;
    for (int64_t j = 0; j < n; ++j) off[j + 1] += off[j];
    int32_t *src = (int32_t *)malloc(sizeof(int32_t) * (size_t)(off[n] > 0 ? off[n] : 1));
    int64_t *pos = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    memcpy(pos, off, sizeof(int64_t) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) /* ascending source order within every target */
        for (int32_t x = 0; x < fwd[i]; ++x) src[pos[cand[i * cap + x]]++] = (int32_t)i;
#pragma omp parallel for schedule(dynamic, 1024) num_threads(omp_threads(nthreads))
    for (int64_t j = 0; j < n; ++j) {
        int32_t *row = cand + j * cap;
        for (int64_t e = off[j]; e < off[j + 1] && counts[j] < cap; ++e) {
            int32_t i = src[e];
            int dup = 0;
            for (int32_t t = 0; t < counts[j]; ++t)
                if (row[t] == i) { dup = 1; break; }
            if (!dup) row[counts[j]++] = i;
        }
    }
    free(src);
    free(pos);
    free(off);
}

/* build_candidates (_kernels.py:81-135): the forward split is per row, then the two reverse
 * unions (lines 110-134 interleave them per source, but they write disjoint arrays). */
void or_build_candidates_x(const int32_t *ids, uint8_t *flags, int64_t n, int64_t g, int64_t gn,
                           int32_t *new_cand, int32_t *new_counts, int32_t *old_cand,
                           int32_t *old_counts, int nthreads) {
#pragma omp parallel for schedule(static) num_threads(omp_threads(nthreads))
    for (int64_t i = 0; i < n; ++i) {
        int32_t *nc = new_cand + i * gn, *oc = old_cand + i * g;
        for (int64_t t = 0; t < gn; ++t) nc[t] = -1;
        for (int64_t t = 0; t < g; ++t) oc[t] = -1;
        int32_t c = 0, o = 0;
        for (int64_t t = 0; t < g; ++t) {
            int32_t j = ids[i * g + t];
            if (flags[i * g + t] == 1) {
                nc[c++] = j;
                flags[i * g + t] = 0;
                if (c >= gn) break;
            } else if (o < g) {
                oc[o++] = j;
            }
        }
        new_counts[i] = c;
        old_counts[i] = o;
    }
    int32_t *fwd = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    memcpy(fwd, new_counts, sizeof(int32_t) * (size_t)n);
    reverse_union(fwd, n, gn, new_cand, new_counts, nthreads);
    memcpy(fwd, old_counts, sizeof(int32_t) * (size_t)n);
    reverse_union(fwd, n, g, old_cand, old_counts, nthreads);
    free(fwd);
}

/* _heap_push under row j's spinlock.  The row's tail key only ever decreases, so a candidate
 * whose distance exceeds a (possibly stale) unlocked read of the tail distance would be
 * rejected by the locked test too; everything else takes the lock and runs heap_push. */
static inline int heap_push_locked(int32_t *ids, float *dists, uint8_t *flags, int64_t g,
                                   int64_t row, int32_t cand, double dd, uint8_t *lk) {
    if (cand == row) return 0;
    const float d = (float)dd;
    uint32_t tb = __atomic_load_n((const uint32_t *)(dists + row * g + g - 1), __ATOMIC_RELAXED);
    float tail;
    memcpy(&tail, &tb, sizeof tail);
    if (d > tail) return 0;
    while (__atomic_test_and_set(lk + row, __ATOMIC_ACQUIRE))
        ;
    int32_t *ri = ids + row * g;
    float *rd = dists + row * g;
    uint8_t *rf = flags + row * g;
    int r = 0;
    float wd = rd[g - 1];
    if (!(d > wd || (d == wd && cand >= ri[g - 1]))) {
        int dup = 0;
        for (int64_t t = 0; t < g; ++t)
            if (ri[t] == cand) { dup = 1; break; }
        if (!dup) {
            int64_t pos = g - 1;
            while (pos > 0 && (rd[pos - 1] > d || (rd[pos - 1] == d && ri[pos - 1] > cand))) --pos;
            /* shift [pos, g-2] up by one; the tail slot is the one read without the lock */
            uint32_t nb;
            memcpy(&nb, pos == g - 1 ? &d : &rd[g - 2], sizeof nb);
            for (int64_t t = g - 1; t > pos; --t) {
                ri[t] = ri[t - 1];
                rf[t] = rf[t - 1];
                if (t < g - 1) rd[t] = rd[t - 1];
            }
            __atomic_store_n((uint32_t *)(rd + g - 1), nb, __ATOMIC_RELAXED);
            ri[pos] = cand;
            if (pos < g - 1) rd[pos] = d;
            rf[pos] = 1;
            r = 1;
        }
    }
    __atomic_clear(lk + row, __ATOMIC_RELEASE);
    return r;
}

/* local_join (_kernels.py:138-173) in parallel over i.  Every pushed candidate has a fixed key
 * (f32 of its pair distance, id), rows reject duplicates, and a row's tail only improves, so
 * after all pushes each row is the top-g of (its old entries U everything pushed to it) in any
 * order; old entries that survive keep their flags, new ones get 1.  The
 * returned count of successful pushes depends on the order, but it is 0 exactly when no row
 * changed, which is all graph.py:256 tests. */
int64_t or_local_join_x(const float *F, const uint8_t *F8, const int32_t *A, int64_t n, int64_t m,
                        int64_t l, double inv_alpha, const int32_t *new_cand,
                        const int32_t *new_counts, int64_t gn, const int32_t *old_cand,
                        const int32_t *old_counts, int32_t *ids, float *dists, uint8_t *flags,
                        int64_t g, int64_t *pairs_out, int nthreads) {
    feat_t f = {F, F8, A, m, l};
    uint8_t *lk = (uint8_t *)calloc((size_t)n, 1);
    int64_t changes = 0, pairs = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : changes, pairs) \
    num_threads(omp_threads(nthreads))
    for (int64_t i = 0; i < n; ++i) {
        int32_t na = new_counts[i], nb = old_counts[i];
        const int32_t *nw = new_cand + i * gn, *od = old_cand + i * g;
        for (int32_t x = 0; x < na; ++x) {
            int32_t j = nw[x];
            /* the partners of j in the reference's order: new[y > x], then old[0..nb) (j == k
             * skipped); distances four at a time, pushes in that same order per j (the order
             * is immaterial anyway, see above) */
            int32_t blk[4];
            int nblk = 0;
            for (int32_t y = x + 1; y < na + nb; ++y) {
                int32_t k = y < na ? nw[y] : od[y - na];
                if (j == k) continue;
                blk[nblk++] = k;
                if (nblk == 4) {
                    double dd[4];
                    fpair_dist4(&f, j, blk, inv_alpha, dd);
                    for (int u = 0; u < 4; ++u) {
                        ++pairs;
                        changes += heap_push_locked(ids, dists, flags, g, j, blk[u], dd[u], lk);
                        changes += heap_push_locked(ids, dists, flags, g, blk[u], j, dd[u], lk);
                    }
                    nblk = 0;
                }
            }
            if (nblk) {
                for (int u = 0; u < nblk; ++u) {
                    double d = fpair_dist(&f, j, blk[u], inv_alpha);
                    ++pairs;
                    changes += heap_push_locked(ids, dists, flags, g, j, blk[u], d, lk);
                    changes += heap_push_locked(ids, dists, flags, g, blk[u], j, d, lk);
                }
            }
        }
    }
    free(lk);
    if (pairs_out) *pairs_out = pairs;
    return changes;
}

/* brute_force_topk (_kernels.py:176-204) with the optional u8 features. */
void or_brute_force_topk_x(const float *F, const uint8_t *F8, const int32_t *A, int64_t n,
                           int64_t m, int64_t l, double inv_alpha, const int64_t *sample_ids,
                           int64_t s, int64_t k, int32_t *out_ids, int nthreads) {
    feat_t f = {F, F8, A, m, l};
#pragma omp parallel for schedule(dynamic, 1) num_threads(omp_threads(nthreads))
    for (int64_t si = 0; si < s; ++si) {
        int64_t u = sample_ids[si];
        double *bd = (double *)malloc(sizeof(double) * (size_t)k);
        int64_t *bi = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
        for (int64_t t = 0; t < k; ++t) { bd[t] = INFINITY; bi[t] = n; }
        for (int64_t v = 0; v < n; ++v) {
            if (v == u) continue;
            double d = fpair_dist(&f, u, v, inv_alpha);
            double wd = bd[k - 1];
            if (d > wd || (d == wd && v >= bi[k - 1])) continue;
            int64_t pos = k - 1;
            while (pos > 0 && (bd[pos - 1] > d || (bd[pos - 1] == d && bi[pos - 1] > v))) {
                bd[pos] = bd[pos - 1];
                bi[pos] = bi[pos - 1];
                --pos;
            }
            bd[pos] = d;
            bi[pos] = v;
        }
        for (int64_t t = 0; t < k; ++t) out_ids[si * k + t] = bi[t] < n ? (int32_t)bi[t] : -1;
        free(bd);
        free(bi);
    }
}

/* One row of prune_pass given the guard decisions: entry p is dropped iff it is redundant and
 * the in-degree safeguard allows it.  For a row s that is NOT p's highest-id in-neighbour,
 * in_deg[p] >= 2 when s is processed (s itself and the higher in-neighbour still hold p), so
 * the safeguard never blocks; for s = maxin[p] it blocks exactly when every other in-neighbour
 * has already dropped p, which is fire[p].  keep[] receives the row's decisions. */
static void prune_row(const feat_t *f, const int32_t *ids, const int32_t *counts, int64_t g,
                      const int32_t *maxin, const uint8_t *fire, double sigma, int64_t s,
                      uint8_t *keep) {
    int32_t cnt = counts[s];
    const int32_t *ri = ids + s * g;
    if (cnt <= 1) {
        for (int32_t t = 0; t < cnt; ++t) keep[t] = 1;
        return;
    }
    memset(keep, 0, (size_t)cnt);
    keep[0] = 1;
    for (int32_t t = 1; t < cnt; ++t) {
        int32_t p = ri[t];
        int redundant = 0;
        for (int32_t u = 0; u < t; ++u) {
            if (!keep[u]) continue;
            int32_t kk = ri[u];
            if (attrs_equal(f->A, f->l, p, kk) && fdiff_cosine(f, s, p, kk) > sigma) {
                redundant = 1;
                break;
            }
        }
        int blocked = maxin[p] == s && fire[p];
        keep[t] = !(redundant && !blocked);
    }
}

/* prune_pass (_kernels.py:266-303) in parallel.  in_deg[p] when row s is
 * processed = 1 + (rows s' < s that still hold p); it can fall below 2 only at p's highest-id
 * in-neighbour maxin[p], and there exactly when all other in-neighbours dropped p.  Let
 * fire[p] be that event.  Rows are evaluated in parallel given fire[], then fire[] is
 * recomputed from the drops; rows whose maxin entries changed are re-evaluated until nothing
 * changes.  fire[p] depends only on rows below maxin[p], whose decisions depend only on fire[]
 * of entries with an even lower maxin, so the iteration reaches the sequential result.
 * in_deg: in = count_in_degrees (graph.py:212), out = as the sequential pass leaves it. */
int32_t or_prune_pass_x(const float *F, const uint8_t *F8, const int32_t *A, int64_t n, int64_t m,
                        int64_t l, int32_t *ids, float *dists, int32_t *counts, int64_t g,
                        int64_t *in_deg, double sigma, int nthreads) {
    feat_t f = {F, F8, A, m, l};
    const int nt = omp_threads(nthreads);
    int32_t *maxin = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    uint8_t *fire = (uint8_t *)calloc((size_t)n, 1);
    uint8_t *keep = (uint8_t *)malloc((size_t)(n * g));
    uint8_t *dirty = (uint8_t *)malloc((size_t)n);
    int64_t *drops = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    for (int64_t p = 0; p < n; ++p) maxin[p] = -1;
    for (int64_t s = 0; s < n; ++s) /* ascending s: the last writer is the highest id */
        for (int32_t t = 0; t < counts[s]; ++t) maxin[ids[s * g + t]] = (int32_t)s;
    memset(dirty, 1, (size_t)n);
    int32_t rounds = 0;
    for (;;) {
        ++rounds;
#pragma omp parallel for schedule(dynamic, 256) num_threads(nt)
        for (int64_t s = 0; s < n; ++s)
            if (dirty[s]) prune_row(&f, ids, counts, g, maxin, fire, sigma, s, keep + s * g);
        /* drops of p by rows other than maxin[p] */
        memset(drops, 0, sizeof(int64_t) * (size_t)n);
        for (int64_t s = 0; s < n; ++s)
            for (int32_t t = 0; t < counts[s]; ++t) {
                int32_t p = ids[s * g + t];
                if (!keep[s * g + t] && maxin[p] != s) drops[p] += 1;
            }
        memset(dirty, 0, (size_t)n);
        int changed = 0;
        for (int64_t p = 0; p < n; ++p) {
            uint8_t nf = maxin[p] >= 0 && drops[p] == in_deg[p] - 1;
            if (nf != fire[p]) {
                fire[p] = nf;
                dirty[maxin[p]] = 1;
                changed = 1;
            }
        }
        if (!changed) break;
    }
    /* compact rows, final in-degrees */
    for (int64_t s = 0; s < n; ++s) {
        int32_t cnt = counts[s];
        if (cnt <= 1) continue;
        int32_t *ri = ids + s * g;
        float *rd = dists + s * g;
        int32_t w = 0;
        for (int32_t t = 0; t < cnt; ++t) {
            if (keep[s * g + t]) {
                ri[w] = ri[t];
                rd[w] = rd[t];
                ++w;
            } else {
                in_deg[ri[t]] -= 1;
            }
        }
        counts[s] = w;
    }
    free(maxin);
    free(fire);
    free(keep);
    free(dirty);
    free(drops);
    return rounds;
}

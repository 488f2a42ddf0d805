/*
 * cortex_oracle.c -- TEST INFRASTRUCTURE ONLY (see cortex_oracle.h).
 *
 * Plain-C restatement of the reference's synapse / attend / injection-path
 * arithmetic.  Each function follows the cited reference lines operation by
 * operation: the same promotions (float -> double before subtracting or
 * multiplying), the same sequential accumulation order, and the same
 * std::min / std::max comparison forms, so that with -ffp-contract=off the
 * results are bit-identical to the reference built with its own flags.
 */
#include "cortex_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- rng.hpp:11-48 ------------------------------------------------------ */

void orc_rng_init(orc_rng* r, uint64_t seed) {
    r->state = seed;
    r->spare = 0.0;
    r->has_spare = 0;
}

uint64_t orc_rng_next_u64(orc_rng* r) { /* rng.hpp:16-21 */
    uint64_t z = (r->state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

double orc_rng_next_unit(orc_rng* r) { /* rng.hpp:24-26 */
    return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53;
}

uint64_t orc_rng_next_below(orc_rng* r, uint64_t n) { /* rng.hpp:28 */
    return orc_rng_next_u64(r) % n;
}

double orc_rng_next_gaussian(orc_rng* r, double mean, double stddev) { /* rng.hpp:30-43 */
    if (r->has_spare) {
        r->has_spare = 0;
        return mean + r->spare * stddev;
    }
    const double u1 = 1.0 - orc_rng_next_unit(r);
    const double u2 = orc_rng_next_unit(r);
    const double rad = sqrt(-2.0 * log(u1));
    const double a = 2.0 * 3.14159265358979323846 * u2;
    r->spare = rad * sin(a);
    r->has_spare = 1;
    return mean + rad * cos(a) * stddev;
}

void orc_rng_fill_gaussian_f32(orc_rng* r, float* dst, int64_t n, double mean, double stddev) {
    for (int64_t i = 0; i < n; ++i) dst[i] = (float)orc_rng_next_gaussian(r, mean, stddev);
}

/* ---- helpers: std::min / std::max forms --------------------------------- */

/* std::min(a, b) returns (b < a) ? b : a;  std::max(a, b) returns (a < b) ? b : a. */
static inline double std_min(double a, double b) { return (b < a) ? b : a; }
static inline double std_max(double a, double b) { return (a < b) ? b : a; }

/* synapse.cpp:18-25: sq_dist(span<float>, span<float>) */
static double sq_dist_ff(const float* a, const float* b, int n) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) {
        const double d = (double)a[i] - (double)b[i];
        acc += d * d;
    }
    return acc;
}

/* synapse.cpp:27-34: sq_dist(span<float>, vector<double>) */
static double sq_dist_fd(const float* a, const double* b, int n) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) {
        const double d = (double)a[i] - b[i];
        acc += d * d;
    }
    return acc;
}

/* ---- kernels.cpp:66-81 ------------------------------------------------ */

int orc_softmax(const double* scores, int64_t n, double* out) {
    if (n <= 0) return ORC_PRECONDITION_ERROR; /* "softmax: empty input" */
    double maxv = -INFINITY;
    for (int64_t i = 0; i < n; ++i) {
        if (!isfinite(scores[i])) return ORC_PRECONDITION_ERROR; /* non-finite */
        maxv = std_max(maxv, scores[i]);
    }
    double sum = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        out[i] = exp(scores[i] - maxv);
        sum += out[i];
    }
    for (int64_t i = 0; i < n; ++i) out[i] /= sum;
    return ORC_OK;
}

/* ---- kernels.cpp:94-101 (argmax): best = 0; i wins iff v[i] > v[best] ---- */
int orc_argmax(const float* v, int64_t n) {
    int best = 0;
    for (int i = 1; i < (int)n; ++i)
        if (v[i] > v[best]) best = i;
    return best;
}

/* ---- synapse.cpp:63-93 ------------------------------------------------ */

int orc_attention_scores_points(const float* keys, int64_t count, int dim,
                                const float* query, int64_t query_len, int n_heads,
                                double* out) {
    if (count == 0) return ORC_PRECONDITION_ERROR;            /* :66 */
    if (query_len != (int64_t)dim) return ORC_PRECONDITION_ERROR; /* :67-68 */
    if (n_heads < 1 || dim % n_heads != 0) return ORC_PRECONDITION_ERROR; /* :69-70 */
    const int d_k = dim / n_heads;
    const double inv_sqrt_dk = 1.0 / sqrt((double)d_k);
    double* scores = (double*)malloc(sizeof(double) * (size_t)count);
    double* probs = (double*)malloc(sizeof(double) * (size_t)count);
    for (int64_t i = 0; i < count; ++i) out[i] = 0.0;
    int st = ORC_OK;
    for (int h = 0; h < n_heads && st == ORC_OK; ++h) {
        const size_t off = (size_t)h * (size_t)d_k;
        for (int64_t i = 0; i < count; ++i) {
            const float* kp = keys + (size_t)i * (size_t)dim;
            double dot = 0.0;
            for (int c = 0; c < d_k; ++c) dot += (double)query[off + (size_t)c] * (double)kp[off + (size_t)c];
            scores[i] = dot * inv_sqrt_dk;
        }
        st = orc_softmax(scores, count, probs);
        if (st == ORC_OK)
            for (int64_t i = 0; i < count; ++i) out[i] += probs[i];
    }
    free(scores);
    free(probs);
    return st;
}

/* ---- synapse.cpp:36-44, 103-120 --------------------------------------- */

void orc_centroid(const float* cloud, int64_t count, int dim, double* c) {
    for (int j = 0; j < dim; ++j) c[j] = 0.0;
    for (int64_t i = 0; i < count; ++i) {
        const float* p = cloud + (size_t)i * (size_t)dim;
        for (int j = 0; j < dim; ++j) c[j] += p[j];
    }
    for (int j = 0; j < dim; ++j) c[j] /= (double)count;
}

int orc_coverage_scores_points(const float* cloud, int64_t count, int dim,
                               const int64_t* selected, int64_t n_selected, double* out) {
    for (int64_t i = 0; i < count; ++i) out[i] = 0.0;
    if (count == 0) return ORC_OK;
    if (n_selected == 0) {
        double* c = (double*)malloc(sizeof(double) * (size_t)(dim > 0 ? dim : 1));
        orc_centroid(cloud, count, dim, c);
        for (int64_t i = 0; i < count; ++i)
            out[i] = sqrt(sq_dist_fd(cloud + (size_t)i * (size_t)dim, c, dim));
        free(c);
        return ORC_OK;
    }
    for (int64_t i = 0; i < count; ++i) {
        double best = INFINITY;
        for (int64_t s = 0; s < n_selected; ++s)
            best = std_min(best, sq_dist_ff(cloud + (size_t)i * (size_t)dim,
                                            cloud + (size_t)selected[s] * (size_t)dim, dim));
        out[i] = sqrt(best);
    }
    return ORC_OK;
}

/* ---- synapse.cpp:216-284 ------------------------------------------------ */

typedef struct { int64_t row; double score; } orc_pick;

static int pick_cmp(const void* a, const void* b) {
    const int64_t ra = ((const orc_pick*)a)->row, rb = ((const orc_pick*)b)->row;
    return (ra > rb) - (ra < rb);
}

int orc_select_landmarks_points(const float* cloud, int64_t count, int dim,
                                const double* attention, int64_t attention_len,
                                int k, double lambda,
                                int64_t* out_indices, double* out_scores, int64_t* out_n) {
    if (k < 1) return ORC_CONFIG_ERROR;                        /* :219 */
    if (lambda < 0.0 || lambda > 1.0) return ORC_CONFIG_ERROR; /* :220-221 */
    if (attention_len != count) return ORC_PRECONDITION_ERROR; /* :222-223 */
    const int64_t n = count;
    const int64_t take = (int64_t)k < n ? (int64_t)k : n;      /* :226 */
    if (out_n) *out_n = take;
    if (n == 0) return ORC_OK;
    unsigned char* remaining = (unsigned char*)malloc((size_t)n);
    memset(remaining, 1, (size_t)n);
    double* mindist = (double*)malloc(sizeof(double) * (size_t)n);
    orc_coverage_scores_points(cloud, count, dim, NULL, 0, mindist); /* :228 */
    orc_pick* picked = (orc_pick*)malloc(sizeof(orc_pick) * (size_t)(take > 0 ? take : 1));

    for (int64_t round = 0; round < take; ++round) {
        /* minmax_remaining (:232-241) for attention then coverage (:245-246) */
        double amin = INFINITY, amax = -INFINITY, cmin = INFINITY, cmax = -INFINITY;
        for (int64_t i = 0; i < n; ++i) {
            if (!remaining[i]) continue;
            amin = std_min(amin, attention[i]);
            amax = std_max(amax, attention[i]);
        }
        for (int64_t i = 0; i < n; ++i) {
            if (!remaining[i]) continue;
            cmin = std_min(cmin, mindist[i]);
            cmax = std_max(cmax, mindist[i]);
        }
        int64_t best = -1;
        double best_score = -1.0;
        for (int64_t i = 0; i < n; ++i) { /* :249-260 */
            if (!remaining[i]) continue;
            const double na = amax > amin ? (attention[i] - amin) / (amax - amin) : 0.0;
            const double nc = cmax > cmin ? (mindist[i] - cmin) / (cmax - cmin) : 0.0;
            const double hybrid = lambda * nc + (1.0 - lambda) * na;
            if (hybrid > best_score) { best = i; best_score = hybrid; }
        }
        if (best < 0) { /* only reachable with NaN inputs (reference UB) */
            free(remaining); free(mindist); free(picked);
            return ORC_PRECONDITION_ERROR;
        }
        remaining[best] = 0;
        picked[round].row = best;
        picked[round].score = best_score;
        const float* bp = cloud + (size_t)best * (size_t)dim; /* :265-273 */
        for (int64_t i = 0; i < n; ++i) {
            const double d = sqrt(sq_dist_ff(cloud + (size_t)i * (size_t)dim, bp, dim));
            mindist[i] = (round == 0) ? d : std_min(mindist[i], d);
        }
    }
    qsort(picked, (size_t)take, sizeof(orc_pick), pick_cmp); /* :276-277 (rows unique) */
    for (int64_t s = 0; s < take; ++s) {
        out_indices[s] = picked[s].row;
        out_scores[s] = picked[s].score;
    }
    free(remaining); free(mindist); free(picked);
    return ORC_OK;
}

/* ---- gate.cpp:27-43 ------------------------------------------------------ */

int orc_gate_score(const float* h_main, const float* t_side, int64_t n, double* out) {
    double dot = 0.0, na = 0.0, nb = 0.0;
    for (int64_t i = 0; i < n; ++i) {  /* one pass, three sequential sums */
        const double a = h_main[i], b = t_side[i];
        dot += a * b;
        na += a * a;
        nb += b * b;
    }
    if (na == 0.0 || nb == 0.0) return ORC_DEGENERATE_INPUT_ERROR;
    double s = dot / (sqrt(na) * sqrt(nb));
    s = s < -1.0 ? -1.0 : (1.0 < s ? 1.0 : s); /* std::clamp(s, -1, 1) */
    *out = s;
    return ORC_OK;
}

/* ---- synapse.cpp:139-165 ------------------------------------------------ */

int orc_hausdorff_distance(const float* cloud, int64_t count, int dim,
                           const float* landmarks, int64_t m, int ldim, double* out) {
    if (count == 0 || m == 0) return ORC_PRECONDITION_ERROR;
    if (dim != ldim) return ORC_PRECONDITION_ERROR;
    double worst = 0.0;
    for (int64_t i = 0; i < count; ++i) {
        double best = INFINITY;
        for (int64_t j = 0; j < m; ++j)
            best = std_min(best, sq_dist_ff(cloud + (size_t)i * (size_t)dim,
                                            landmarks + (size_t)j * (size_t)dim, dim));
        worst = std_max(worst, best);
    }
    *out = sqrt(worst);
    return ORC_OK;
}

int orc_hausdorff_to_subset(const float* cloud, int64_t count, int dim,
                            const int64_t* rows, int64_t n_rows, double* out) {
    if (n_rows == 0) return ORC_PRECONDITION_ERROR;
    double worst = 0.0;
    for (int64_t i = 0; i < count; ++i) {
        double best = INFINITY;
        for (int64_t s = 0; s < n_rows; ++s)
            best = std_min(best, sq_dist_ff(cloud + (size_t)i * (size_t)dim,
                                            cloud + (size_t)rows[s] * (size_t)dim, dim));
        worst = std_max(worst, best);
    }
    *out = sqrt(worst);
    return ORC_OK;
}

/* ---- synapse.cpp:169-214 ------------------------------------------------ */

static double mean_pairwise(const float* cloud, int64_t count, int dim) {
    double sum = 0.0;
    int64_t pairs = 0;
    for (int64_t i = 0; i < count; ++i)
        for (int64_t j = i + 1; j < count; ++j) {
            sum += sqrt(sq_dist_ff(cloud + (size_t)i * (size_t)dim, cloud + (size_t)j * (size_t)dim, dim));
            ++pairs;
        }
    return pairs > 0 ? sum / (double)pairs : 0.0;
}

static double mean_pairwise_subset(const float* cloud, int dim, const int64_t* rows, int64_t n) {
    double sum = 0.0;
    int64_t pairs = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = i + 1; j < n; ++j) {
            sum += sqrt(sq_dist_ff(cloud + (size_t)rows[i] * (size_t)dim,
                                   cloud + (size_t)rows[j] * (size_t)dim, dim));
            ++pairs;
        }
    return pairs > 0 ? sum / (double)pairs : 0.0;
}

int orc_mean_pairwise_reduction(const float* cloud, int64_t count, int dim,
                                const float* landmarks, int64_t m, int ldim, double* out) {
    if (m < 2) return ORC_PRECONDITION_ERROR;
    if (count < 2) return ORC_PRECONDITION_ERROR;
    const double cloud_mean = mean_pairwise(cloud, count, dim);
    if (cloud_mean == 0.0) { *out = 0.0; return ORC_OK; }
    *out = 1.0 - mean_pairwise(landmarks, m, ldim) / cloud_mean;
    return ORC_OK;
}

int orc_mean_pairwise_reduction_subset(const float* cloud, int64_t count, int dim,
                                       const int64_t* rows, int64_t n_rows, double* out) {
    if (n_rows < 2) return ORC_PRECONDITION_ERROR;
    if (count < 2) return ORC_PRECONDITION_ERROR;
    const double cloud_mean = mean_pairwise(cloud, count, dim);
    if (cloud_mean == 0.0) { *out = 0.0; return ORC_OK; }
    *out = 1.0 - mean_pairwise_subset(cloud, dim, rows, n_rows) / cloud_mean;
    return ORC_OK;
}

/* ---- kernels.cpp:103-142 ------------------------------------------------ */

void orc_attend(const float* q, const float* keys, const float* values,
                int64_t n_entries, int n_heads, int d_k, float* out) {
    const int d_model = n_heads * d_k;
    const double inv_sqrt_dk = 1.0 / sqrt((double)d_k);
    double* w = (double*)malloc(sizeof(double) * (size_t)(n_entries > 0 ? n_entries : 1));
    for (int h = 0; h < n_heads; ++h) {
        const float* qh = q + (size_t)h * (size_t)d_k;
        double maxs = -INFINITY;
        for (int64_t j = 0; j < n_entries; ++j) {
            const float* kh = keys + (size_t)j * (size_t)d_model + (size_t)h * (size_t)d_k;
            double dot = 0.0;
            for (int c = 0; c < d_k; ++c) dot += (double)qh[c] * (double)kh[c];
            w[j] = dot * inv_sqrt_dk;
            maxs = std_max(maxs, w[j]);
        }
        double sum = 0.0;
        for (int64_t j = 0; j < n_entries; ++j) {
            w[j] = exp(w[j] - maxs);
            sum += w[j];
        }
        for (int c = 0; c < d_k; ++c) {
            double acc = 0.0;
            for (int64_t j = 0; j < n_entries; ++j)
                acc += w[j] * (double)values[(size_t)j * (size_t)d_model + (size_t)h * (size_t)d_k + (size_t)c];
            out[(size_t)h * (size_t)d_k + (size_t)c] = (float)(acc / sum);
        }
    }
    free(w);
}

/* Batched decode oracle (GQA composition): for agents
 * [a0, a1), every layer l and q-head h of KV head g = h / (n_q / n_kv), the
 * reference's kernels::attend (kernels.cpp:103-142) with n_heads = 1 over the
 * agent's cache as run_agent builds it (scheduler.cpp:245-262): the k_syn
 * synapse rows of (l, g) first, then the agent's private rows [0, tail_len[a]).
 * Layouts: syn [n_layers][n_kv][k_syn][d_k]; tail [N][n_layers][n_kv][t_cap][d_k];
 * q / out [N][n_layers][n_q][d_k]. */
void orc_decode_attend_agents(int64_t a0, int64_t a1, int n_layers, int n_kv, int n_q, int d_k, int64_t k_syn,
                              int64_t t_cap, const float* syn_k, const float* syn_v, const float* tail_k,
                              const float* tail_v, const int32_t* tail_len, const float* q, float* out) {
    const int64_t cap = k_syn + t_cap;
    float* kk = (float*)malloc(sizeof(float) * (size_t)(cap > 0 ? cap : 1) * (size_t)d_k);
    float* vv = (float*)malloc(sizeof(float) * (size_t)(cap > 0 ? cap : 1) * (size_t)d_k);
    const int qpg = n_q / n_kv;
    for (int64_t a = a0; a < a1; ++a) {
        const int64_t nt = tail_len[a];
        for (int l = 0; l < n_layers; ++l)
            for (int g = 0; g < n_kv; ++g) {
                const size_t so = ((size_t)l * (size_t)n_kv + (size_t)g) * (size_t)k_syn * (size_t)d_k;
                const size_t to = (((size_t)a * (size_t)n_layers + (size_t)l) * (size_t)n_kv + (size_t)g) *
                                  (size_t)t_cap * (size_t)d_k;
                memcpy(kk, syn_k + so, sizeof(float) * (size_t)k_syn * (size_t)d_k);
                memcpy(vv, syn_v + so, sizeof(float) * (size_t)k_syn * (size_t)d_k);
                memcpy(kk + (size_t)k_syn * (size_t)d_k, tail_k + to, sizeof(float) * (size_t)nt * (size_t)d_k);
                memcpy(vv + (size_t)k_syn * (size_t)d_k, tail_v + to, sizeof(float) * (size_t)nt * (size_t)d_k);
                for (int hh = 0; hh < qpg; ++hh) {
                    const size_t qo = (((size_t)a * (size_t)n_layers + (size_t)l) * (size_t)n_q +
                                       (size_t)g * (size_t)qpg + (size_t)hh) * (size_t)d_k;
                    orc_attend(q + qo, kk, vv, k_syn + nt, 1, d_k, out + qo);
                }
            }
    }
    free(kk);
    free(vv);
}

/* ---- harness/bench.cpp:65-125 ------------------------------------------- */

void orc_make_clustered_cloud(orc_rng* r, int64_t count, int dim, int n_clusters,
                              double separation, double sigma, int rare_cluster_size,
                              float* cloud, float* query, int32_t* cluster_of) {
    double qnorm = 0.0;
    for (int j = 0; j < dim; ++j) {
        query[j] = (float)orc_rng_next_gaussian(r, 0.0, 1.0);
        qnorm += (double)query[j] * query[j];
    }
    double* centers = (double*)malloc(sizeof(double) * (size_t)n_clusters * (size_t)dim);
    for (int c = 0; c < n_clusters; ++c) {
        double* cc = centers + (size_t)c * (size_t)dim;
        for (int j = 0; j < dim; ++j) cc[j] = orc_rng_next_gaussian(r, 0.0, separation);
        double dot = 0.0;
        for (int j = 0; j < dim; ++j) dot += cc[j] * query[j];
        for (int j = 0; j < dim; ++j) cc[j] -= dot / qnorm * query[j];
    }
    int64_t row = 0;
    for (int c = 0; c < n_clusters; ++c) {
        const int64_t size = (c == 0) ? count - (int64_t)rare_cluster_size * (n_clusters - 1)
                                      : (int64_t)rare_cluster_size;
        for (int64_t i = 0; i < size; ++i, ++row) {
            cluster_of[row] = c;
            for (int j = 0; j < dim; ++j)
                cloud[(size_t)row * (size_t)dim + (size_t)j] =
                    (float)(centers[(size_t)c * (size_t)dim + (size_t)j] + orc_rng_next_gaussian(r, 0.0, sigma));
        }
    }
    free(centers);
}

int64_t orc_random_subset(orc_rng* r, int64_t n, int k, int64_t* out) {
    int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) idx[i] = i;
    const int take = (int)((int64_t)k < n ? (int64_t)k : n);
    for (int i = 0; i < take; ++i) {
        const int64_t j = i + (int64_t)orc_rng_next_below(r, (uint64_t)(n - i));
        const int64_t t = idx[i]; idx[i] = idx[j]; idx[j] = t;
    }
    for (int i = 0; i < take; ++i) out[i] = idx[i];
    free(idx);
    return take;
}

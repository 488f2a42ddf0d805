/*
 * cortex_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the Warp Cortex reference's Topological Synapse
 * hot path (/root/reference/proj, CPU-only C++20).  Every function cites the
 * reference file:line it restates.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load this library, and only as the checker:
 * the product path (paper_2601_01298_b200) never links or calls it.
 *
 * Parity pins: tests/test_oracle_pins.py checks this restatement against the
 * reference's own known-answer tests (test_synapse.cpp, test_kernels.cpp,
 * acceptance.cpp AC3/AC4) and, when oracle/_ref is built, bitwise against the
 * reference library compiled from /root/reference sources.
 *
 * Arithmetic contract (matches the reference build: g++ -O3, no -march, so no
 * FMA contraction): compile with -ffp-contract=off.  All sums run in the
 * reference's sequential order.
 */
#ifndef CORTEX_ORACLE_H
#define CORTEX_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes mirror the reference's exception taxonomy
 * (proj/include/cortex/errors.hpp:10-41). */
enum {
    ORC_OK = 0,
    ORC_CONFIG_ERROR = 1,
    ORC_CAPACITY_ERROR = 2,
    ORC_TOPOLOGY_ERROR = 3,
    ORC_SEQUENCING_ERROR = 4,
    ORC_PRECONDITION_ERROR = 5,
    ORC_CAP_ERROR = 6,
    ORC_DEGENERATE_INPUT_ERROR = 7
};

/* splitmix64 + Box-Muller generator, rng.hpp:11-48. */
typedef struct orc_rng {
    uint64_t state;
    double spare;
    int has_spare;
} orc_rng;

void orc_rng_init(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next_u64(orc_rng* r);
double orc_rng_next_unit(orc_rng* r);
uint64_t orc_rng_next_below(orc_rng* r, uint64_t n);
double orc_rng_next_gaussian(orc_rng* r, double mean, double stddev);
/* Fills n floats with (float)next_gaussian(mean, stddev), in order. */
void orc_rng_fill_gaussian_f32(orc_rng* r, float* dst, int64_t n, double mean, double stddev);

/* kernels.cpp:66-81 (softmax_impl). */
int orc_softmax(const double* scores, int64_t n, double* out);

/* kernels.cpp:94-101 (argmax): lowest index of the maximum (n >= 1). */
int orc_argmax(const float* v, int64_t n);

/* synapse.cpp:63-93. */
int orc_attention_scores_points(const float* keys, int64_t count, int dim,
                                const float* query, int64_t query_len, int n_heads,
                                double* out);

/* synapse.cpp:36-44 (centroid_of). */
void orc_centroid(const float* cloud, int64_t count, int dim, double* out);

/* synapse.cpp:103-120. */
int orc_coverage_scores_points(const float* cloud, int64_t count, int dim,
                               const int64_t* selected, int64_t n_selected, double* out);

/* synapse.cpp:216-284.  Writes min(k,count) ascending rows and their scores;
 * *out_n receives the count. */
int orc_select_landmarks_points(const float* cloud, int64_t count, int dim,
                                const double* attention, int64_t attention_len,
                                int k, double lambda,
                                int64_t* out_indices, double* out_scores, int64_t* out_n);

/* gate.cpp:27-42 gate_score: fp64 cosine with sequential sums, clamped to [-1, 1];
 * ORC_DEGENERATE_INPUT_ERROR on a zero norm. */
int orc_gate_score(const float* h_main, const float* t_side, int64_t n, double* out);

/* synapse.cpp:139-165. */
int orc_hausdorff_distance(const float* cloud, int64_t count, int dim,
                           const float* landmarks, int64_t m, int ldim, double* out);
int orc_hausdorff_to_subset(const float* cloud, int64_t count, int dim,
                            const int64_t* rows, int64_t n_rows, double* out);

/* synapse.cpp:169-214. */
int orc_mean_pairwise_reduction(const float* cloud, int64_t count, int dim,
                                const float* landmarks, int64_t m, int ldim, double* out);
int orc_mean_pairwise_reduction_subset(const float* cloud, int64_t count, int dim,
                                       const int64_t* rows, int64_t n_rows, double* out);

/* kernels.cpp:103-142 (attend). */
void orc_attend(const float* q, const float* keys, const float* values,
                int64_t n_entries, int n_heads, int d_k, float* out);

/* Batched decode oracle: kernels.cpp:103-142 attend (n_heads = 1) per
 * (agent, layer, q-head) over [synapse rows of its KV head || private rows
 * [0, tail_len[a])] (scheduler.cpp:245-262); agents [a0, a1). */
void orc_decode_attend_agents(int64_t a0, int64_t a1, int n_layers, int n_kv, int n_q, int d_k, int64_t k_syn,
                              int64_t t_cap, const float* syn_k, const float* syn_v, const float* tail_k,
                              const float* tail_v, const int32_t* tail_len, const float* q, float* out);

/* harness/bench.cpp:65-112 (make_clustered_cloud); writes count*dim floats,
 * dim query floats and count cluster ids. */
void orc_make_clustered_cloud(orc_rng* r, int64_t count, int dim, int n_clusters,
                              double separation, double sigma, int rare_cluster_size,
                              float* cloud, float* query, int32_t* cluster_of);

/* harness/bench.cpp:114-125 (random_subset); writes min(k,n) rows. */
int64_t orc_random_subset(orc_rng* r, int64_t n, int k, int64_t* out);

#ifdef __cplusplus
}
#endif

#endif /* CORTEX_ORACLE_H */

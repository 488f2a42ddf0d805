// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shims over the UNMODIFIED reference library (cortex:: from
// /root/reference/proj/src, compiled by oracle/Makefile into
// oracle/_ref/libcortex_ref.so).  Used for three things only:
//   1. pinning the C restatement (oracle/cortex_oracle.c) bit-for-bit,
//   2. generating the golden fixtures under tests/golden/,
//   3. timing the reference's own CPU path (bench.py --impl reference and the
//      cpu_baseline leg), on all host cores via std::thread over groups /
//      agents, exactly as SURVEY.md §8(d) plans.
// Nothing in the product (paper_2601_01298_b200/) links this file.
#include "cortex/errors.hpp"
#include "cortex/bench.hpp"
#include "cortex/injector.hpp"
#include "cortex/kernels.hpp"
#include "cortex/model.hpp"
#include "cortex/rng.hpp"
#include "cortex/gate.hpp"
#include "cortex/synapse.hpp"

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include <omp.h>

using namespace cortex;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const config_error& e) { g_err = e.what(); return 1; }
    catch (const capacity_error& e) { g_err = e.what(); return 2; }
    catch (const topology_error& e) { g_err = e.what(); return 3; }
    catch (const sequencing_error& e) { g_err = e.what(); return 4; }
    catch (const precondition_error& e) { g_err = e.what(); return 5; }
    catch (const cap_error& e) { g_err = e.what(); return 6; }
    catch (const degenerate_input_error& e) { g_err = e.what(); return 7; }
    catch (const std::exception& e) { g_err = e.what(); return 99; }
}

PointCloud make_cloud(const float* data, int64_t count, int dim) {
    PointCloud c;
    c.count = count;
    c.dim = dim;
    c.data.assign(data, data + static_cast<size_t>(count) * static_cast<size_t>(dim));
    return c;
}

ModelConfig make_cfg(int n_layers, int n_heads, int d_model, int64_t max_positions) {
    ModelConfig cfg;
    cfg.n_layers = n_layers;
    cfg.n_heads = n_heads;
    cfg.d_model = d_model;
    cfg.d_k = d_model / n_heads;
    cfg.max_positions = max_positions;
    return cfg;
}

// Per-group attention for GQA groups: the sum, in q-head
// order, of attention_scores_points(cloud, q_h, 1).
std::vector<double> group_attention(const PointCloud& cloud, const float* q, int n_q, int dim) {
    std::vector<double> total(static_cast<size_t>(cloud.count), 0.0);
    for (int h = 0; h < n_q; ++h) {
        const auto p = attention_scores_points(
            cloud, std::span<const float>(q + static_cast<size_t>(h) * dim, static_cast<size_t>(dim)), 1);
        for (size_t i = 0; i < total.size(); ++i) total[i] += p[i];
    }
    return total;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_softmax(const double* s, int64_t n, double* out) {
    return guarded([&] {
        auto p = kernels::softmax(std::span<const double>(s, static_cast<size_t>(n)));
        std::copy(p.begin(), p.end(), out);
    });
}

int ref_argmax(const float* v, int64_t n, int* out) {
    return guarded([&] { *out = kernels::argmax(std::span<const float>(v, static_cast<size_t>(n))); });
}

int ref_attention_scores_points(const float* keys, int64_t count, int dim, const float* q,
                                int64_t qlen, int n_heads, double* out) {
    return guarded([&] {
        auto c = make_cloud(keys, count, dim);
        auto a = attention_scores_points(c, std::span<const float>(q, static_cast<size_t>(qlen)), n_heads);
        std::copy(a.begin(), a.end(), out);
    });
}

int ref_coverage_scores_points(const float* cloud, int64_t count, int dim, const int64_t* sel,
                               int64_t n_sel, double* out) {
    return guarded([&] {
        auto c = make_cloud(cloud, count, dim);
        auto r = coverage_scores_points(c, std::span<const int64_t>(sel, static_cast<size_t>(n_sel)));
        std::copy(r.begin(), r.end(), out);
    });
}

int ref_select_landmarks_points(const float* cloud, int64_t count, int dim, const double* attn,
                                int64_t attn_len, int k, double lambda, int64_t* idx,
                                double* scores, int64_t* out_n) {
    return guarded([&] {
        auto c = make_cloud(cloud, count, dim);
        auto r = select_landmarks_points(c, std::span<const double>(attn, static_cast<size_t>(attn_len)), k, lambda);
        std::copy(r.indices.begin(), r.indices.end(), idx);
        std::copy(r.scores.begin(), r.scores.end(), scores);
        *out_n = static_cast<int64_t>(r.indices.size());
    });
}

int ref_gate_score(const float* h, const float* t, int64_t n, double* out) {
    return guarded([&] {
        *out = gate_score(std::span<const float>(h, static_cast<size_t>(n)),
                          std::span<const float>(t, static_cast<size_t>(n)));
    });
}

int ref_hausdorff_distance(const float* cloud, int64_t count, int dim, const float* lm, int64_t m,
                           int ldim, double* out) {
    return guarded([&] {
        PointCloud a = make_cloud(cloud, count, dim), b = make_cloud(lm, m, ldim);
        *out = hausdorff_distance(a, b);
    });
}

int ref_hausdorff_to_subset(const float* cloud, int64_t count, int dim, const int64_t* rows,
                            int64_t n, double* out) {
    return guarded([&] {
        auto a = make_cloud(cloud, count, dim);
        *out = hausdorff_to_subset(a, std::span<const int64_t>(rows, static_cast<size_t>(n)));
    });
}

int ref_mean_pairwise_reduction(const float* cloud, int64_t count, int dim, const float* lm,
                                int64_t m, int ldim, double* out) {
    return guarded([&] {
        PointCloud a = make_cloud(cloud, count, dim), b = make_cloud(lm, m, ldim);
        *out = mean_pairwise_reduction(a, b);
    });
}

int ref_mean_pairwise_reduction_subset(const float* cloud, int64_t count, int dim,
                                       const int64_t* rows, int64_t n, double* out) {
    return guarded([&] {
        auto a = make_cloud(cloud, count, dim);
        *out = mean_pairwise_reduction_subset(a, std::span<const int64_t>(rows, static_cast<size_t>(n)));
    });
}

int ref_attend(const float* q, const float* keys, const float* values, int64_t n_entries,
               int n_heads, int d_k, float* out) {
    return guarded([&] {
        const size_t dm = static_cast<size_t>(n_heads) * d_k;
        kernels::attend(std::span<const float>(q, dm),
                        std::span<const float>(keys, static_cast<size_t>(n_entries) * dm),
                        std::span<const float>(values, static_cast<size_t>(n_entries) * dm),
                        n_entries, n_heads, d_k, std::span<float>(out, dm));
    });
}

// ---- Rng + harness generators (rng.hpp, harness/bench.cpp) ----------------

void* ref_rng_new(uint64_t seed) { return new Rng(seed); }
void ref_rng_free(void* r) { delete static_cast<Rng*>(r); }
uint64_t ref_rng_next_u64(void* r) { return static_cast<Rng*>(r)->next_u64(); }
uint64_t ref_rng_next_below(void* r, uint64_t n) { return static_cast<Rng*>(r)->next_below(n); }
double ref_rng_next_unit(void* r) { return static_cast<Rng*>(r)->next_unit(); }
double ref_rng_next_gaussian(void* r, double mean, double sd) {
    return static_cast<Rng*>(r)->next_gaussian(mean, sd);
}

void ref_make_clustered_cloud(void* r, int64_t count, int dim, int n_clusters, double separation,
                              double sigma, int rare, float* cloud, float* query, int32_t* cluster_of) {
    auto cc = harness::make_clustered_cloud(*static_cast<Rng*>(r), count, dim, n_clusters,
                                            separation, sigma, rare);
    std::copy(cc.cloud.data.begin(), cc.cloud.data.end(), cloud);
    std::copy(cc.query.begin(), cc.query.end(), query);
    for (size_t i = 0; i < cc.cluster_of.size(); ++i) cluster_of[i] = cc.cluster_of[i];
}

int64_t ref_random_subset(void* r, int64_t n, int k, int64_t* out) {
    auto v = harness::random_subset(*static_cast<Rng*>(r), n, k);
    std::copy(v.begin(), v.end(), out);
    return static_cast<int64_t>(v.size());
}

// bench_landmarks (harness/bench.cpp:330-425): returns the report's JSON.
int ref_bench_landmarks(uint64_t seed, int n_seeds, int64_t cloud_size, int k, double lambda,
                        char* json_out, int64_t cap) {
    return guarded([&] {
        auto rep = harness::bench_landmarks(seed, n_seeds, cloud_size, k, lambda);
        const std::string s = rep.to_json().dump();
        std::strncpy(json_out, s.c_str(), static_cast<size_t>(cap - 1));
        json_out[cap - 1] = 0;
    });
}

// ---- KvCache-level path: select_landmarks (synapse.cpp:286-320) ------------
// keys/values: [n_entries][n_layers][d_model] (append_entry layout).
int ref_select_landmarks(int n_layers, int n_heads, int d_model, int64_t max_positions,
                         int64_t n_entries, const int64_t* positions, const uint8_t* origins,
                         const float* keys, const float* values, const float* query, int k,
                         double lambda, int64_t* out_source_length, int64_t* out_n,
                         int64_t* out_pos, double* out_scores, float* out_keys, float* out_values) {
    return guarded([&] {
        const ModelConfig cfg = make_cfg(n_layers, n_heads, d_model, max_positions);
        KvCache cache(cfg);
        const size_t per = static_cast<size_t>(n_layers) * d_model;
        for (int64_t i = 0; i < n_entries; ++i) {
            cache.append_entry(positions[i], origins[i] ? Origin::injected : Origin::context,
                               std::span<const float>(keys + i * per, per),
                               std::span<const float>(values + i * per, per));
        }
        auto snap = select_landmarks(cache, std::span<const float>(query, static_cast<size_t>(d_model)), k, lambda);
        *out_source_length = snap.source_length;
        *out_n = static_cast<int64_t>(snap.landmarks.size());
        for (size_t s = 0; s < snap.landmarks.size(); ++s) {
            out_pos[s] = snap.landmarks[s].source_position;
            out_scores[s] = snap.landmarks[s].hybrid_score;
            std::copy(snap.landmarks[s].keys.begin(), snap.landmarks[s].keys.end(), out_keys + s * per);
            std::copy(snap.landmarks[s].values.begin(), snap.landmarks[s].values.end(), out_values + s * per);
        }
    });
}

// ---- CPU baseline timing helpers (SURVEY.md §8(d) "CPU baseline timing plan")
// Per-group compression: attention (sum over the group's q-heads) + greedy
// selection, one std::thread per core over groups.  clouds: [G][L][dim];
// queries: [G][n_q][dim]; idx out: [G][min(k,L)].
int ref_compress_groups_mt(int n_groups, const float* clouds, int64_t L, int dim, const float* queries,
                           int n_q, int k, double lambda, int n_threads, int64_t* idx_out) {
    return guarded([&] {
        std::atomic<int> next{0};
        std::atomic<int> failed{0};
        const int64_t take = std::min<int64_t>(k, L);
        auto worker = [&] {
            omp_set_num_threads(1); // one std::thread per core; no nested teams
            for (int g = next.fetch_add(1); g < n_groups; g = next.fetch_add(1)) {
                try {
                    auto c = make_cloud(clouds + static_cast<size_t>(g) * L * dim, L, dim);
                    auto a = group_attention(c, queries + static_cast<size_t>(g) * n_q * dim, n_q, dim);
                    auto r = select_landmarks_points(c, a, k, lambda);
                    std::copy(r.indices.begin(), r.indices.end(), idx_out + static_cast<size_t>(g) * take);
                } catch (...) {
                    failed.store(1);
                }
            }
        };
        std::vector<std::thread> ts;
        for (int t = 0; t < std::max(1, n_threads); ++t) ts.emplace_back(worker);
        for (auto& t : ts) t.join();
        if (failed.load()) throw std::runtime_error("ref_compress_groups_mt: a group failed");
    });
}

// Decode attention baseline: for each agent a, each (layer, q-head h), call
// kernels::attend(n_heads=1, d_k) over [synapse rows of h's KV head || the
// agent's private rows].  Layouts (fp32): syn_k/v [n_layers][n_kv][k_syn][d_k];
// tail_k/v [N][n_layers][n_kv][T][d_k]; q/out [N][n_layers][n_q][d_k].
int ref_decode_attend_mt(int N, int n_layers, int n_kv, int n_q, int d_k, int k_syn, int T,
                         const float* syn_k, const float* syn_v, const float* tail_k,
                         const float* tail_v, const float* q, float* out, int n_threads) {
    return guarded([&] {
        std::atomic<int> next{0};
        const int qpg = n_q / n_kv;
        const int n = k_syn + T;
        auto worker = [&] {
            omp_set_num_threads(1);
            std::vector<float> kbuf(static_cast<size_t>(n) * d_k), vbuf(kbuf.size());
            for (int a = next.fetch_add(1); a < N; a = next.fetch_add(1)) {
                for (int l = 0; l < n_layers; ++l) {
                    for (int g = 0; g < n_kv; ++g) {
                        const size_t so = ((size_t)l * n_kv + g) * (size_t)k_syn * d_k;
                        const size_t to = (((size_t)a * n_layers + l) * n_kv + g) * (size_t)T * d_k;
                        std::copy(syn_k + so, syn_k + so + (size_t)k_syn * d_k, kbuf.begin());
                        std::copy(syn_v + so, syn_v + so + (size_t)k_syn * d_k, vbuf.begin());
                        std::copy(tail_k + to, tail_k + to + (size_t)T * d_k, kbuf.begin() + (size_t)k_syn * d_k);
                        std::copy(tail_v + to, tail_v + to + (size_t)T * d_k, vbuf.begin() + (size_t)k_syn * d_k);
                        for (int hh = 0; hh < qpg; ++hh) {
                            const int h = g * qpg + hh;
                            const size_t qo = (((size_t)a * n_layers + l) * n_q + h) * d_k;
                            kernels::attend(std::span<const float>(q + qo, d_k), kbuf, vbuf, n, 1, d_k,
                                            std::span<float>(out + qo, d_k));
                        }
                    }
                }
            }
        };
        std::vector<std::thread> ts;
        for (int t = 0; t < std::max(1, n_threads); ++t) ts.emplace_back(worker);
        for (auto& t : ts) t.join();
    });
}

} // extern "C"

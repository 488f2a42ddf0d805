/*
 * cortex_b200.h -- C-ABI of the B200-native Topological Synapse hot path.
 *
 * The reference (/root/reference/proj) is a C++20 library with no FFI layer;
 * its hot path is the cortex:: header API compiled into cortex_core
 * (SURVEY.md §8(b)).  This header is the drop-in boundary: one extern "C"
 * entry point per reference function on the path (the citation on each line
 * is the cortex:: declaration it replaces), plain pointers + sizes, no torch
 * or CUDA types (streams are passed as void* = cudaStream_t).  The C++ shim
 * in include/cortex/ (the .hpp headers) re-exports the exact cortex:: declarations on top
 * of these entry points, so code written against the reference links
 * unchanged.
 *
 * Error convention: every call returns cx_status.  Categories map 1:1 onto
 * the reference's exception types (proj/include/cortex/errors.hpp:10-41) and
 * validation happens before any device work, as in the reference.  A failed
 * CUDA call returns CX_DEVICE_ERROR (never one of the reference categories).
 * cx_last_error() returns the thread-local message of the last failure.
 *
 * Pointer conventions:
 *   *_host entry points and the un-suffixed reference-shaped calls take HOST
 *   pointers, are synchronous, and have the reference's semantics;
 *   *_dev entry points take DEVICE pointers and are ordered on `stream`.
 * There is no CPU fallback: without a CUDA device every compute call returns
 * CX_DEVICE_ERROR.
 */
#ifndef CORTEX_B200_H
#define CORTEX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CX_ABI_VERSION 1

typedef enum cx_status {
    CX_OK = 0,
    CX_CONFIG_ERROR = 1,           /* cortex::config_error          errors.hpp:13 */
    CX_CAPACITY_ERROR = 2,         /* cortex::capacity_error        errors.hpp:18 */
    CX_TOPOLOGY_ERROR = 3,         /* cortex::topology_error        errors.hpp:23 */
    CX_SEQUENCING_ERROR = 4,       /* cortex::sequencing_error      errors.hpp:28 */
    CX_PRECONDITION_ERROR = 5,     /* cortex::precondition_error    errors.hpp:32 */
    CX_CAP_ERROR = 6,              /* cortex::cap_error             errors.hpp:37 */
    CX_DEGENERATE_INPUT_ERROR = 7, /* cortex::degenerate_input_error errors.hpp:41 */
    CX_DEVICE_ERROR = 100,         /* CUDA failure / no device (new; never a reference type) */
    CX_INVALID_ARGUMENT = 101      /* null handle / impossible size at the C boundary (new) */
} cx_status;

typedef enum cx_origin { CX_ORIGIN_CONTEXT = 0, CX_ORIGIN_INJECTED = 1 } cx_origin; /* model.hpp:16 */

int cx_abi_version(void);
const char* cx_last_error(void);
/* Number of sm_100a kernel launches this process issued (all entry points). */
uint64_t cx_kernel_launch_count(void);

/* ======================================================================
 * Point-level synapse operations, reference semantics, HOST pointers.
 * ====================================================================== */

/* synapse.hpp:62-64 attention_scores_points(const PointCloud&, span<const float> query, int n_heads) */
cx_status cx_attention_scores_points(const float* keys, int64_t count, int dim,
                                     const float* query, int64_t query_len, int n_heads,
                                     double* out /* [count] */);

/* synapse.hpp:73-74 coverage_scores_points(const PointCloud&, span<const int64_t> selected) */
cx_status cx_coverage_scores_points(const float* cloud, int64_t count, int dim,
                                    const int64_t* selected, int64_t n_selected,
                                    double* out /* [count] */);

/* synapse.hpp:104-106 select_landmarks_points(const PointCloud&, span<const double>, int k, double lambda)
 * out_indices/out_scores must hold min(k, count) entries; *out_n receives it. */
cx_status cx_select_landmarks_points(const float* cloud, int64_t count, int dim,
                                     const double* attention, int64_t attention_len,
                                     int k, double lambda,
                                     int64_t* out_indices, double* out_scores, int64_t* out_n);

/* synapse.hpp:83-91 metrics */
cx_status cx_hausdorff_distance(const float* cloud, int64_t count, int dim,
                                const float* landmarks, int64_t m, int ldim, double* out);
cx_status cx_hausdorff_to_subset(const float* cloud, int64_t count, int dim,
                                 const int64_t* rows, int64_t n_rows, double* out);
cx_status cx_mean_pairwise_reduction(const float* cloud, int64_t count, int dim,
                                     const float* landmarks, int64_t m, int ldim, double* out);
cx_status cx_mean_pairwise_reduction_subset(const float* cloud, int64_t count, int dim,
                                            const int64_t* rows, int64_t n_rows, double* out);

/* gate.hpp:22 / gate.cpp:27-43 gate_score(h_main, t_side): fp64 cosine clamped to [-1, 1];
 * CX_DEGENERATE_INPUT_ERROR for a zero-norm input.  Host pointers; computed on the device. */
cx_status cx_gate_score(const float* h_main, const float* t_side, int64_t n, double* out);

/* kernels.hpp:31-32 softmax(span<const double>) / softmax(span<const float>)
 * (kernels.cpp:66-92): max-subtracted exp in fp64, the sum in index order;
 * CX_PRECONDITION_ERROR on empty or non-finite input.  Within 1e-15 relative of
 * the reference (CUDA exp vs glibc exp: <= 1 ulp).  out: n doubles (host). */
cx_status cx_softmax(const double* scores, int64_t n, double* out);
cx_status cx_softmax_f32(const float* scores, int64_t n, double* out);

/* kernels.hpp:35 argmax(span<const float>) (kernels.cpp:94-101): the lowest
 * index of the maximum (a NaN never wins, except at index 0);
 * CX_PRECONDITION_ERROR on empty input (the reference asserts it). */
cx_status cx_argmax(const float* v, int64_t n, int* out);

/* kernels.hpp:40-42 attend(q, keys, values, n_entries, n_heads, d_k, out)
 * fp64 accumulation like the reference (tolerance 1e-6, test_kernels.cpp:159). */
cx_status cx_attend(const float* q, const float* keys, const float* values,
                    int64_t n_entries, int n_heads, int d_k, float* out);

/* ======================================================================
 * Grouped device path (per-(layer, KV-head) groups).
 * ====================================================================== */

typedef struct cx_ctx cx_ctx; /* device workspace + default stream; one per host thread */

cx_status cx_ctx_create(int device, cx_ctx** out);
cx_status cx_ctx_destroy(cx_ctx* ctx);

/* On-box peak of the selection's exact arithmetic: unfused fp64 add / mul
 * operations per second over the whole device (independent dependency chains on
 * every SM; a few ms).  The bench uses it as the fp64 roofline of the greedy
 * selection. */
cx_status cx_probe_fp64_rate(cx_ctx* ctx, double* ops_per_s);

/* Priority lanes (SURVEY.md §8(b) threading row): the River's
 * work (injection appends, synapse pushes) goes on the highest-priority stream,
 * Stream agents' decode on a medium-priority one.  Replaces the reference's
 * river thread / per-agent std::threads (scheduler.cpp:63-113, 198). */
typedef enum cx_lane { CX_LANE_RIVER = 0, CX_LANE_STREAM = 1 } cx_lane;
cx_status cx_ctx_lane_stream(cx_ctx* ctx, int lane, void** stream, int* priority);

/* A batch of G independent selection groups.  Group g's cloud row i, column c
 * is clouds[g * group_stride + i * row_stride + c] (fp32, device).  Queries:
 * queries[(g * n_pass + p) * d_k + c].  Pass p scores columns
 * [p * col_step, p * col_step + d_k) -- col_step = d_k reproduces the
 * reference's head-concatenated MHA cloud (attention_scores_points with
 * n_heads = n_pass, synapse.cpp:63-93); col_step = 0 is the GQA group mode
 * (sum over the group's q-heads of attention_scores_points(cloud, q_h, 1)). */
typedef struct cx_groups {
    int n_groups;
    int64_t count;       /* L rows per group */
    int dim;             /* cloud width */
    const float* clouds; /* device */
    int64_t group_stride;
    int64_t row_stride;
    const float* queries; /* device, [G][n_pass][d_k] */
    int n_pass;
    int d_k;
    int col_step;
} cx_groups;

/* attention mass per row for every group: out[G][count] (device, fp64). */
cx_status cx_attention_grouped_dev(cx_ctx* ctx, const cx_groups* g, double* out, void* stream);

/* Greedy hybrid selection (synapse.cpp:216-284) for every group given its
 * attention [G][count] (device).  Outputs (device): rows [G][take] ascending,
 * scores [G][take], take = min(k, count).  flags: CX_SELECT_* below. */
#define CX_SELECT_EXACT_ONLY 1u /* disable the conservative fp32 distance filter */
#define CX_SELECT_GENERIC 2u    /* force the generic-dim kernel (testing) */
cx_status cx_select_grouped_dev(cx_ctx* ctx, const cx_groups* g, const double* attention,
                                int k, double lambda, unsigned flags,
                                int64_t* out_rows, double* out_scores, void* stream);

/* Path pinning for tests and tuning (defaults: the cost models).  Options are
 * per context and read at launch time; they never change results (every
 * pinned path is bit-exact / within tolerance like the default), only which
 * kernel configuration computes them.  CX_INVALID_ARGUMENT for an unknown
 * option or out-of-range value. */
#define CX_OPT_SELECT_CLUSTER 1     /* selection cluster size 1..16; 0 = cost model */
#define CX_OPT_SELECT_NO_SKETCH 2   /* 1 = never keep rows as the fp16 sketch */
#define CX_OPT_DECODE_IMPL 3        /* CX_DECODE_* below */
#define CX_OPT_DECODE_CTAS_PER_LH 4 /* tcgen05 decode CTAs per (layer, KV head); 0 = auto */
#define CX_OPT_HOST_UPLOAD_VALUES 5 /* 1 = host path uploads all values even if pinned */
#define CX_OPT_SELECT_IMPL 6        /* CX_SELECT_IMPL_* below */
#define CX_SELECT_IMPL_AUTO 0       /* tensor-core filter (d = 64), then CUDA-core, then generic */
#define CX_SELECT_IMPL_TC 1         /* pinned: an error if the shape does not apply */
#define CX_SELECT_IMPL_CUDA_CORE 2  /* the CUDA-core filter kernels (select64 / select128) */
#define CX_OPT_SELECT_EXCHANGE 7    /* tensor-core selection: 0 cost model, 1 thread-block clusters
                                       (DSMEM), 2 cooperative launch (global-memory exchanges),
                                       3 split: co-resident clusters + a cooperative launch for the
                                       remaining groups on the free SMs, side by side in one wave */
#define CX_OPT_HOST_STAGE_OUTPUTS 8 /* 1 = host path stages the synapse K/V on the device and copies
                                       it back even when the caller's buffers are pinned (default 0:
                                       the landmark gather writes them straight into pinned memory) */
#define CX_DECODE_AUTO 0            /* tcgen05, then v2, then the generic kernel */
#define CX_DECODE_TC 1              /* pinned: an error if the shape does not apply */
#define CX_DECODE_V2 2
#define CX_DECODE_V1 3
cx_status cx_ctx_set_option(cx_ctx* ctx, int option, int64_t value);
cx_status cx_ctx_get_option(cx_ctx* ctx, int option, int64_t* value);

/* Decision-gap monitor (SURVEY.md §7 "per-round gap monitor").  Writes, for
 * each of the n_groups groups of this ctx's most recent selection launch (the
 * last cx_select_grouped_dev / cx_compress_grouped_dev call, or the last chunk
 * of cx_compress_grouped_host), the smallest top-1 / top-2 gap of the exact
 * hybrid score over its greedy rounds, capped at 1e-10 (gaps above the cap are
 * not resolved).  The attention mass is within 1e-12 relative of the
 * reference's (CUDA vs glibc exp, tree-ordered softmax sum), which moves a
 * normalised hybrid score by a few 1e-12 when amax >> amin; a gap above 1e-11
 * therefore certifies that the reference makes the same pick in every round.
 * NaN = not monitored (the generic-dim kernel).  `out` may be host or device
 * memory; the copy is ordered on `stream`, after the selection.
 * CX_PRECONDITION_ERROR if n_groups exceeds the last launch's group count. */
cx_status cx_selection_gaps(cx_ctx* ctx, int n_groups, double* out, void* stream);

/* Landmark gather (synapse.cpp:303-318 copy, per group): dst[g][s][:] =
 * src row rows[g][s] of group g (same addressing as g->clouds, base `src`). */
cx_status cx_gather_grouped_dev(cx_ctx* ctx, const cx_groups* g, const float* src,
                                const int64_t* rows, int take, float* dst, void* stream);

/* One synapse compression: attention + selection + landmark K/V gather.
 * values: same addressing as g->clouds (separate base pointer).  Outputs
 * (device): rows/scores [G][take], syn_keys/syn_values [G][take][dim]. */
cx_status cx_compress_grouped_dev(cx_ctx* ctx, const cx_groups* g, const float* values,
                                  int k, double lambda, unsigned flags,
                                  int64_t* out_rows, double* out_scores,
                                  float* syn_keys, float* syn_values, void* stream);

/* cx_compress_grouped_dev with the synapse blocks syn_group_stride floats apart
 * (0 = take * dim): e.g. a per-KV-head view of the river cache compressed
 * straight into the decode layout [layer][kv head][k][d_k] (stride n_kv * k * d_k,
 * base + head * k * d_k), with no copy. */
cx_status cx_compress_grouped_strided_dev(cx_ctx* ctx, const cx_groups* g, const float* values,
                                          int k, double lambda, unsigned flags,
                                          int64_t* out_rows, double* out_scores,
                                          float* syn_keys, float* syn_values,
                                          int64_t syn_group_stride, void* stream);

/* One synapse compression from HOST buffers (the end-to-end call): dense
 * keys/values [G][count][dim], queries [G][n_pass][d_k] (n_pass/d_k/col_step as
 * in cx_groups); outputs (host): rows/scores [G][take], syn_keys/syn_values
 * [G][take][dim], take = min(k, count).  Groups are uploaded in chunks on a copy
 * stream so the upload of chunk i+1 overlaps the compression of chunk i (true
 * overlap needs pinned host memory).  When `values` is pinned (device-accessible),
 * only the selected value rows cross PCIe (zero-copy gather); otherwise all of
 * it is uploaded.  When syn_keys and syn_values are both pinned, the landmark
 * gather writes them in place over PCIe (no device copy, no D2H; see
 * CX_OPT_HOST_STAGE_OUTPUTS).  Synchronous: returns with outputs written.
 * Same checks, in the same order, as cx_compress_grouped_dev. */
cx_status cx_compress_grouped_host(cx_ctx* ctx, int n_groups, int64_t count, int dim,
                                   const float* keys, const float* values, const float* queries,
                                   int n_pass, int d_k, int col_step, int k, double lambda,
                                   unsigned flags, int64_t* out_rows, double* out_scores,
                                   float* syn_keys, float* syn_values);

/* ======================================================================
 * Batched decode attention of N agents against the shared synapse
 * (kernels.cpp:103-142 per (agent, layer, q-head), fp32 accumulate).
 * ====================================================================== */
typedef struct cx_decode_batch {
    int n_agents, n_layers, n_kv, n_q, d_k;
    int k_syn;                 /* synapse rows per (layer, kv head) */
    const float* syn_keys;     /* [n_layers][n_kv][k_syn][d_k] */
    const float* syn_values;
    float* tail_keys;          /* [N][n_layers][n_kv][t_cap][d_k]  private rows */
    float* tail_values;
    int t_cap;
    const int32_t* tail_len;   /* [N] rows already in each private tail */
    const float* new_keys;     /* [N][n_layers][n_kv][d_k]  appended at tail_len (or NULL) */
    const float* new_values;
    const float* q;            /* [N][n_layers][n_q][d_k] */
    float* out;                /* [N][n_layers][n_q][d_k] */
    unsigned flags;            /* CX_DECODE_* below (0 = none) */
} cx_decode_batch;

/* The caller guarantees syn_keys / syn_values were not written since the previous
 * decode step on the same stream (the synapse between two pushes): the tcgen05
 * kernel then stages the synapse while the previous step drains (programmatic
 * dependent launch); everything else still waits for the previous step. */
#define CX_DECODE_SYN_UNCHANGED 1u

/* Stream-ordered: never synchronizes.  Precondition per agent (the reference
 * KvCache's capacity check, model.cpp:124-140): 0 <= tail_len[a] <= t_cap - 1
 * when new_keys is set (room for the appended row), <= t_cap otherwise.  The
 * kernels check it on the device: an agent outside it sets
 * CX_DEVERR_TAIL_RANGE (cx_ctx_device_errors), appends nothing, and attends
 * over its rows clamped to that range (its outputs are then unspecified);
 * no write ever leaves the agent's own tail. */
cx_status cx_decode_step_dev(cx_ctx* ctx, const cx_decode_batch* b, void* stream);

/* Device-detected precondition failures of the stream-ordered *_dev calls
 * on this ctx (a bitmask, accumulated since the last clear): the reference
 * throws for these, a device kernel can only record them.  Synchronizes
 * `stream` (the stream the checked calls ran on), then writes the mask and,
 * if clear != 0, resets it.
 *   CX_DEVERR_NONFINITE   a non-finite attention score (kernels.cpp:70; the
 *                         reference's precondition_error)
 *   CX_DEVERR_TAIL_RANGE  a decode tail_len outside its range (above)
 * A ctx is meant to be driven from one stream at a time: its scratch arena,
 * side stream and this flag are shared by all of its *_dev calls. */
#define CX_DEVERR_NONFINITE 1u
#define CX_DEVERR_TAIL_RANGE 2u
cx_status cx_ctx_device_errors(cx_ctx* ctx, void* stream, unsigned* flags, int clear);

/* gate.hpp:26 / gate.cpp:45-61 decide(h_main, t_side, theta) for n_pairs (row h[i], row t[i])
 * device pairs (row strides in floats): scores[i] (NaN when degenerate), accepted[i] =
 * scores[i] >= theta, degenerate[i] = zero norm (accepted and degenerate may be NULL).
 * theta outside [-1, 1] -> CX_PRECONDITION_ERROR before any work (gate.cpp:47-48).
 * The gate fused after an agent step: h = main-model hidden states, t = thoughts. */
cx_status cx_gate_decide_dev(cx_ctx* ctx, int64_t n_pairs, int dim, const float* h, int64_t h_stride,
                             const float* t, int64_t t_stride, double theta, double* scores,
                             uint8_t* accepted, uint8_t* degenerate, void* stream);

/* ======================================================================
 * Device-resident KvCache (model.hpp:67-113) and Referential Injection.
 * Layout: keys/values [n_layers][capacity][d_model] fp32, positions int64,
 * origins u8.  Checks and error categories follow model.cpp:124-173.
 * ====================================================================== */
typedef struct cx_kvcache cx_kvcache;

cx_status cx_kvcache_create(int n_layers, int n_heads, int d_model, int d_k,
                            int64_t max_positions, int64_t capacity, cx_kvcache** out);
cx_status cx_kvcache_destroy(cx_kvcache* c);
/* deep copy (the reference KvCache is a value type): rows, positions, origins, state */
cx_status cx_kvcache_clone(const cx_kvcache* src, cx_kvcache** out);
int64_t cx_kvcache_size(const cx_kvcache* c);
int64_t cx_kvcache_context_count(const cx_kvcache* c);
int64_t cx_kvcache_last_context_position(const cx_kvcache* c);
int cx_kvcache_entry_open(const cx_kvcache* c);
int64_t cx_kvcache_capacity(const cx_kvcache* c);
/* device base pointers (layer-major) for zero-copy consumers */
float* cx_kvcache_keys_dev(cx_kvcache* c);
float* cx_kvcache_values_dev(cx_kvcache* c);
const int64_t* cx_kvcache_positions_host(const cx_kvcache* c);
const uint8_t* cx_kvcache_origins_host(const cx_kvcache* c);

cx_status cx_kvcache_begin_entry(cx_kvcache* c, int64_t position, cx_origin origin); /* model.cpp:124-140 */
cx_status cx_kvcache_write_layer(cx_kvcache* c, int layer, const float* key, const float* value,
                                 int64_t width);                                      /* model.cpp:142-152 */
cx_status cx_kvcache_end_entry(cx_kvcache* c);                                        /* model.cpp:154-159 */
cx_status cx_kvcache_append_entry(cx_kvcache* c, int64_t position, cx_origin origin,
                                  const float* keys, const float* values);            /* model.cpp:161-173 */
/* Bulk device append of `count` context entries at positions base..base+count-1
 * from a device block [n_layers][count][d_model] (a river prefill), stream-ordered.
 * Same per-entry checks and partial-append behaviour as count append_entry calls
 * (model.cpp:124-173): entries before the first failing one stay appended. */
cx_status cx_kvcache_append_context_dev(cx_kvcache* c, const float* keys, const float* values,
                                        int64_t base_position, int64_t count, void* stream);
/* copy rows [first, first+n) of one layer to host */
cx_status cx_kvcache_read(const cx_kvcache* c, int layer, int64_t first, int64_t n,
                          float* keys_out, float* values_out);

/* injector.hpp:27-35 */
typedef struct cx_injection_record {
    int64_t thought_id;
    int64_t token_count;
    int64_t virtual_position_base;
    int64_t applied_at_stream_position;
} cx_injection_record;

/* injector.hpp:46-47 inject(KvCache&, const KvBlock&, thought_id, stream_position).
 * block keys/values: [n_layers][token_count][d_model]; *_host = host pointers,
 * *_dev = device pointers ordered on stream. */
cx_status cx_inject_host(cx_kvcache* c, const float* keys, const float* values,
                         int64_t base_position, int64_t token_count, int n_layers, int d_model,
                         int64_t thought_id, int64_t stream_position, cx_injection_record* rec);
cx_status cx_inject_dev(cx_kvcache* c, const float* keys, const float* values,
                        int64_t base_position, int64_t token_count, int n_layers, int d_model,
                        int64_t thought_id, int64_t stream_position, cx_injection_record* rec,
                        void* stream);

/* ======================================================================
 * Cache-level selection (synapse.hpp:110-111 select_landmarks) and the
 * SynapseBuffer (synapse.hpp:115-135).
 * ====================================================================== */
typedef struct cx_snapshot cx_snapshot;

cx_status cx_select_landmarks(const cx_kvcache* c, const float* query, int64_t query_len, int k,
                              double lambda, cx_snapshot** out);
/* A snapshot from host data (SynapseSnapshot built by value, synapse.hpp:37-49):
 * positions/scores [count]; keys/values [count][n_layers][d_model] (may be NULL
 * when count == 0).  The K/V are copied to the device. */
cx_status cx_snapshot_create(int64_t source_length, int k_configured, int n_layers, int d_model,
                             int64_t count, const int64_t* positions, const double* scores,
                             const float* keys, const float* values, cx_snapshot** out);
cx_status cx_snapshot_destroy(cx_snapshot* s);
uint64_t cx_snapshot_version(const cx_snapshot* s);
int64_t cx_snapshot_source_length(const cx_snapshot* s);
int cx_snapshot_k_configured(const cx_snapshot* s);
int cx_snapshot_n_layers(const cx_snapshot* s);
int cx_snapshot_d_model(const cx_snapshot* s);
int64_t cx_snapshot_count(const cx_snapshot* s);
/* host copies: positions/scores [count]; keys/values [count][n_layers][d_model] */
cx_status cx_snapshot_read(const cx_snapshot* s, int64_t* positions, double* scores,
                           float* keys, float* values);
/* device views: keys/values [n_layers][count][d_model] (decode-friendly) */
const float* cx_snapshot_keys_dev(const cx_snapshot* s);
const float* cx_snapshot_values_dev(const cx_snapshot* s);

typedef struct cx_synapse_buffer cx_synapse_buffer;
cx_status cx_synapse_buffer_create(cx_synapse_buffer** out);
cx_status cx_synapse_buffer_destroy(cx_synapse_buffer* b);
/* Takes ownership of snap; stamps and returns the version (1, 2, ...). */
cx_status cx_synapse_buffer_push(cx_synapse_buffer* b, cx_snapshot* snap, uint64_t* version);
/* *out = NULL before the first push; the returned reference must be released
 * with cx_snapshot_release (shared ownership, like shared_ptr<const>). */
cx_status cx_synapse_buffer_read_latest(cx_synapse_buffer* b, const cx_snapshot** out);
cx_status cx_synapse_buffer_wait_nonempty(cx_synapse_buffer* b, int64_t timeout_ms,
                                          const cx_snapshot** out);
cx_status cx_synapse_buffer_shutdown(cx_synapse_buffer* b);
cx_status cx_snapshot_release(const cx_snapshot* s);

/* Device memory helpers for C consumers of the *_dev entry points: allocate /
 * free device bytes, and a synchronous read of device bytes ordered on `stream`. */
cx_status cx_device_alloc(size_t bytes, void** out);
cx_status cx_device_free(void* p);
cx_status cx_device_read(void* host, const void* dev, size_t bytes, void* stream);

/* ======================================================================
 * The toy transformer on the device: WeightStore,
 * forward_step batched across agents, and the kernels:: primitives it uses.
 * ====================================================================== */
typedef struct cx_weights cx_weights;
/* floats of the flat weight array, in the reference's draw order (model.cpp:49-80):
 * embedding [vocab][d], per layer {attn_norm [d], wq, wk, wv, wo [d][d], mlp_norm [d],
 * w_in [4d][d], w_out [d][4d]}, final_norm [d], unembedding [vocab][d] */
size_t cx_weights_flat_floats(int n_layers, int d_model, int vocab_size);
cx_status cx_weights_create(int n_layers, int n_heads, int d_model, int d_k, int vocab_size,
                            int64_t max_positions, double rope_base, const float* flat,
                            cx_weights** out);
cx_status cx_weights_destroy(cx_weights* w);

/* forward_step (model.hpp:130-131, model.cpp:175-235) for n_agents agents at once:
 * agent i feeds tokens[i] at positions[i] (host arrays) into caches[i] (distinct
 * caches) and gets logits [i][vocab], hidden [i][d] (after the final norm) and
 * final_query [i][d] (final layer, post RoPE) -- device outputs, any may be NULL.
 * Every agent is checked (token range, open entry, position bounds, strictly
 * increasing context positions) before any device work, with the reference's
 * error categories.  Projections, RMSNorm, RoPE and attention accumulate in fp64
 * (the reference's rounding points), so logits agree to ~1e-12 relative.
 * On a created stream the step's launch sequence is captured once per (weights,
 * batch size, 128-row chunk count, scratch) and replayed as a CUDA graph (the
 * agents' cache pointers / rows / positions / tokens go to device memory first);
 * on the default stream, or a stream the caller is capturing, the launches are
 * issued directly.  Both give the same bits. */
cx_status cx_forward_step_dev(cx_ctx* ctx, const cx_weights* w, int n_agents, cx_kvcache* const* caches,
                              const int* tokens, const int64_t* positions, float* logits,
                              float* hidden, float* final_query, void* stream);

/* kernels.hpp:14-28 (host pointers, computed on the device, synchronous):
 * matvec y = W x (fp64 accumulate), rmsnorm, add_inplace (op 0: x += y) and
 * relu_inplace (op 1), apply_rope. */
cx_status cx_matvec(const float* w, int n_out, int n_in, const float* x, float* y);
cx_status cx_rmsnorm(const float* x, const float* gain, int64_t n, double eps, float* out);
cx_status cx_elementwise(float* x, const float* y, int64_t n, int op);
cx_status cx_apply_rope(float* v, int64_t n, int64_t position, double rope_base);

/* ======================================================================
 * The River / Stream loop on the device (BASELINE
 * configs[4]): Scheduler::run's device work, scheduler.cpp:63-165.
 * River lane (greatest priority; the calling host thread): per river token the
 * token's forward_step on the river cache; every inject_every tokens a thought
 * (thought_tokens ids) is encoded at the next reserved virtual positions
 * (encode_thought) and injected before the token; every push_every tokens (when
 * the previous push has been published) a synapse push into the back buffer.
 * Stream lane (medium priority; a second host thread): each agent step is every
 * agent decoding one token against the front synapse (one CUDA-graph replay).
 * A push is published (version + 1) at the first agent step after its completion
 * event fired, and that step waits on it: agents never read a partly written
 * synapse (SynapseBuffer::push / read_latest, synapse.hpp:115-135).
 * ====================================================================== */
typedef struct cx_cortex cx_cortex;
#define CX_CORTEX_PUSH_SCHEDULER 0 /* Scheduler::push_synapse (scheduler.cpp:158-165): select_landmarks
                                      over the last layer's context keys with the river's final query
                                      (synapse.cpp:286-323), one row set for every layer and head */
#define CX_CORTEX_PUSH_GROUPS 1    /* one selection per (layer, KV head) group with the fixed
                                      river_queries (the BASELINE cfg2 decomposition, 48 groups) */
typedef struct cx_cortex_config {
    int n_agents;            /* stream agents */
    int n_q;                 /* agent query heads per layer (GQA: n_q / n_kv per KV head) */
    int t_cap;               /* agent private rows */
    int k;                   /* landmarks (per group in CX_CORTEX_PUSH_GROUPS) */
    double lambda;
    int push_every;          /* river tokens between pushes (a push waits for the previous one) */
    int inject_every;        /* river tokens between injections */
    int thought_tokens;      /* tokens per injected thought */
    int64_t virtual_base;    /* first reserved virtual position (RuntimeConfig::virtual_base) */
    int64_t max_context;     /* context rows the push mirror holds (>= the prefill) */
    int push_mode;           /* CX_CORTEX_PUSH_* */
    int gate;                /* 1: gate each thought before its injection (scheduler.cpp:272-286 decide:
                                cosine of the river's latest hidden state and the thought's last hidden
                                state >= theta; a rejected thought is not injected); 0: inject all */
    double theta;            /* gate threshold, [-1, 1] (gate.cpp:47-48) */
} cx_cortex_config;
typedef struct cx_cortex_agents {  /* device tensors, the cx_decode_batch layouts */
    float* tail_keys;
    float* tail_values;
    const int32_t* tail_len;
    const float* new_keys;
    const float* new_values;
    const float* q;
    float* out;
    const float* river_queries;     /* CX_CORTEX_PUSH_GROUPS: [n_kv][n_layers][n_q / n_kv][d_k] */
} cx_cortex_agents;
typedef struct cx_cortex_stats {
    double agent_ms, river_ms, push_ms_mean;  /* lane spans (device events) and mean push */
    int pushes, injections;
    uint64_t last_version;
    int thoughts_accepted, thoughts_rejected;  /* gate decisions of the run (gate = 1) */
} cx_cortex_stats;
/* river: the prefilled river cache (context rows only); it must outlive the runtime.
 * The first synapse is pushed and published (version 1) before this returns
 * (CX_CORTEX_PUSH_SCHEDULER: with the final query of the river's last forward_step
 * through this runtime, zeros before the first one). */
cx_status cx_cortex_create(cx_ctx* ctx, const cx_weights* w, cx_kvcache* river,
                           const cx_cortex_config* cfg, const cx_cortex_agents* agents,
                           cx_cortex** out);
/* n_river_tokens river tokens (host ids) at the next river positions, concurrently
 * with n_agent_steps agent steps.  thought_tokens: host ids, thought_tokens per
 * injection, ceil(n_river_tokens / inject_every) thoughts.
 * versions_used (host, optional): the synapse version each agent step read;
 * river_logits (device, optional): [n_river_tokens][vocab].  Audit (device,
 * optional): synapse_history [max_versions][K | V][n_layers][n_kv][k][d_k] gets
 * every version as published (at its version index); out_history
 * [n_agent_steps][agents' out]. */
cx_status cx_cortex_run(cx_cortex* rt, int n_river_tokens, const int* river_tokens, const int* thought_tokens,
                        int n_agent_steps, cx_cortex_stats* stats, uint64_t* versions_used,
                        float* river_logits, float* synapse_history, int max_versions, float* out_history);
/* the latest published synapse (keys / values [n_layers][n_kv][k][d_k], any memory) */
cx_status cx_cortex_front_synapse(const cx_cortex* rt, float* keys, float* values, uint64_t* version);
/* The gate decisions of the last cx_cortex_run (GateDecision rows, gate.hpp:14-22): up to
 * max entries of (thought_id, score (NaN when degenerate), accepted, degenerate); *n = the
 * run's decision count.  Empty when the runtime does not gate. */
cx_status cx_cortex_gate_log(const cx_cortex* rt, int64_t max, int64_t* thought_ids, double* scores,
                             uint8_t* accepted, uint8_t* degenerate, int64_t* n);
cx_status cx_cortex_destroy(cx_cortex* rt);

/* ======================================================================
 * Multi-GPU (the reference has none -- SPEC.md:15).
 * Selection groups are sharded by (layer, KV head): rank r of R owns the
 * balanced contiguous block [b_r, e_r) of the G groups (the first G % R ranks
 * one more) and runs its selections with no collective; the ONE exchange step
 * is an all-gather of the packed per-group synapse records over NVLink.
 * Decode shards by agent against local synapse replicas (no exchange).
 * NCCL is loaded at first use (dlopen libnccl.so.2); without it these calls
 * return CX_DEVICE_ERROR and cx_nccl_version() returns 0.
 * ====================================================================== */
typedef struct cx_comm cx_comm;
#define CX_COMM_ID_BYTES 128
int cx_nccl_version(void);
cx_status cx_comm_unique_id(void* id /* CX_COMM_ID_BYTES */);
/* one process per GPU (ids shared out of band, e.g. torch.distributed) */
cx_status cx_comm_init_rank(int nranks, const void* id, int rank, int device, cx_comm** out);
/* one process driving ndev GPUs (ncclCommInitAll): out[ndev]; drive the ranks'
 * collective calls between cx_comm_group_start / cx_comm_group_end */
cx_status cx_comm_init_all(int ndev, const int* devices, cx_comm** out);
cx_status cx_comm_destroy(cx_comm* c);
cx_status cx_comm_info(const cx_comm* c, int* rank, int* nranks, int* device);
cx_status cx_comm_group_start(void);
cx_status cx_comm_group_end(void);

/* Sharded compression: `local` holds exactly this rank's block of the
 * n_groups_total groups (CX_PRECONDITION_ERROR otherwise), `values` the same
 * rows' values.  Outputs (device, ALL groups, every rank): rows/scores
 * [G][take], syn_keys/syn_values [G][take][dim]; take = min(k, count).  One
 * compression of the local groups, then one all-gather; bitwise equal to a
 * single-GPU cx_compress_grouped_dev of all G groups.  dim % 4 == 0. */
cx_status cx_compress_sharded_dev(cx_ctx* ctx, cx_comm* comm, const cx_groups* local,
                                  const float* values, int n_groups_total, int k, double lambda,
                                  unsigned flags, int64_t* out_rows, double* out_scores,
                                  float* syn_keys, float* syn_values, void* stream);

/* The exchange step's record format, for callers with their own transport:
 * one record per group (rows | scores | keys | values, padded to 256 B).
 * pack: groups [g_begin, g_begin + n_groups) of the [G] arrays -> n_groups
 * consecutive records at dst.  unpack: nranks blocks of ceil(G / nranks)
 * records each (rank r's groups first in its block) -> the [G] arrays. */
size_t cx_synapse_record_bytes(int take, int dim);
cx_status cx_synapse_pack_dev(const int64_t* rows, const double* scores, const float* syn_keys,
                              const float* syn_values, int g_begin, int n_groups, int take, int dim,
                              void* dst, void* stream);
cx_status cx_synapse_unpack_dev(const void* src, int n_groups, int nranks, int take, int dim,
                                int64_t* rows, double* scores, float* syn_keys, float* syn_values,
                                void* stream);
/* the same on host memory (no device work) */
cx_status cx_synapse_pack_host(const int64_t* rows, const double* scores, const float* syn_keys,
                               const float* syn_values, int g_begin, int n_groups, int take, int dim,
                               void* dst);
cx_status cx_synapse_unpack_host(const void* src, int n_groups, int nranks, int take, int dim,
                                 int64_t* rows, double* scores, float* syn_keys, float* syn_values);

/* Accepted-thought K/V to the river GPU (drain_injections, scheduler.cpp:139-156
 * consumes them there with cx_inject_dev): a KvBlock [n_layers][T][d_model]
 * keys + values as one NCCL send / receive pair. */
cx_status cx_thought_send_dev(cx_comm* comm, const float* keys, const float* values,
                              int64_t token_count, int n_layers, int d_model, int river_rank,
                              void* stream);
cx_status cx_thought_recv_dev(cx_comm* comm, float* keys, float* values, int64_t token_count,
                              int n_layers, int d_model, int src_rank, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CORTEX_B200_H */

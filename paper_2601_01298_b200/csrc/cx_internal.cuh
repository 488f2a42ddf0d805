// cx_internal.cuh -- shared plumbing for the sm_100a synapse kernels and the
// C-ABI (include/cortex_b200.h).  Host-side errors are C++ exceptions carrying
// a cx_status; every extern "C" entry point catches them at the boundary.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "cortex_b200.h"

namespace cx {

struct Failure : std::runtime_error {
    cx_status st;
    Failure(cx_status s, const std::string& m) : std::runtime_error(m), st(s) {}
};

[[noreturn]] inline void fail(cx_status s, const std::string& m) { throw Failure(s, m); }

#define CX_CUDA(call)                                                                         \
    do {                                                                                      \
        cudaError_t cx_e_ = (call);                                                           \
        if (cx_e_ != cudaSuccess)                                                             \
            ::cx::fail(CX_DEVICE_ERROR, std::string(#call) + ": " + cudaGetErrorString(cx_e_)); \
    } while (0)

// Counts every kernel launch issued by this library (cx_kernel_launch_count).
extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }
inline void check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(CX_DEVICE_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
    count_launch();
}

void set_last_error(const std::string& m);

// Raises a kernel's dynamic shared memory limit (and, for clusters > 8, allows the
// non-portable size) once per (kernel, device) and size, not on every launch.
void kernel_smem_attr(const void* fn, size_t bytes, bool nonportable_cluster = false);
template <class K>
inline void kernel_smem(K* fn, size_t bytes, bool nonportable_cluster = false) {
    kernel_smem_attr(reinterpret_cast<const void*>(fn), bytes, nonportable_cluster);
}

// Path pinning for tests and tuning (cx_ctx_set_option; defaults = the cost models).
struct Options {
    int select_cluster = 0;      // CX_OPT_SELECT_CLUSTER: force the selection cluster size (0 = cost model)
    int select_no_sketch = 0;    // CX_OPT_SELECT_NO_SKETCH: never use the fp16 sketch row mode
    int select_impl = 0;         // CX_OPT_SELECT_IMPL: CX_SELECT_IMPL_{AUTO,TC,CUDA_CORE}
    int select_exchange = 0;     // CX_OPT_SELECT_EXCHANGE: 0 cost model, 1 clusters (DSMEM), 2 cooperative
    int decode_impl = 0;         // CX_OPT_DECODE_IMPL: CX_DECODE_{AUTO,TC,V2,V1}
    int decode_ctas_per_lh = 0;  // CX_OPT_DECODE_CTAS_PER_LH: tcgen05 decode CTAs per (layer, KV head) (0 = auto)
    int host_upload_values = 0;  // CX_OPT_HOST_UPLOAD_VALUES: host path uploads all values even when pinned
    int host_stage_outputs = 0;  // CX_OPT_HOST_STAGE_OUTPUTS: host path copies the synapse back even when pinned
};

// One NVTX range per C-ABI call (named after the entry point) and per runtime phase: an
// attached Nsight tool shows the boundary calls and the River / Stream work on the timeline;
// without a tool the push / pop are a few-ns no-op (NVTX v3 is header-only, no link-time
// dependency).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Runs f inside an NVTX range named `name`, mapping exceptions to cx_status (the C boundary).
template <class F>
cx_status guard(const char* name, F&& f) {
    NvtxRange range(name);
    try {
        f();
        return CX_OK;
    } catch (const Failure& e) {
        set_last_error(e.what());
        return e.st;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return CX_DEVICE_ERROR;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return CX_DEVICE_ERROR;
    }
}

// Grow-only device arena; one per cx_ctx.  take() hands out 256-byte aligned
// slices that stay valid until reset() (called at the start of each entry point).
struct Arena {
    char* base = nullptr;
    size_t cap = 0;
    size_t used = 0;
    void reserve(size_t bytes) {
        if (bytes <= cap) return;
        if (base) cudaFree(base);
        base = nullptr;
        cap = 0;
        size_t want = bytes + (bytes >> 2);
        CX_CUDA(cudaMalloc(&base, want));
        cap = want;
    }
    void reset() { used = 0; }
    template <class T>
    T* take(size_t n) {
        size_t off = (used + 255) & ~size_t(255);
        size_t bytes = n * sizeof(T);
        if (off + bytes > cap) fail(CX_DEVICE_ERROR, "workspace arena overflow (reserve too small)");
        used = off + bytes;
        return reinterpret_cast<T*>(base + off);
    }
};

// Sizing pass: counts bytes a sequence of take() calls needs.
struct ArenaPlan {
    size_t used = 0;
    template <class T>
    void take(size_t n) { used = ((used + 255) & ~size_t(255)) + n * sizeof(T); }
};

}  // namespace cx

struct cx_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;  // used by the host-pointer (reference-shaped) calls
    cudaStream_t side = nullptr;    // fork target (centroid alongside attention)
    cudaStream_t lane[2] = {nullptr, nullptr};  // CX_LANE_RIVER (highest priority), CX_LANE_STREAM (medium)
    int lane_prio[2] = {0, 0};
    cudaStream_t copy = nullptr;    // host-path uploads (cx_compress_grouped_host)
    char* hbuf = nullptr;           // host-path device staging (grow-only, separate from the arena)
    size_t hcap = 0;
    std::vector<cudaEvent_t> hev;   // per-chunk upload events
    std::vector<cudaEvent_t> pev;   // per-chunk prologue (centroid + attention) events
    cx_ctx* aux = nullptr;          // host path: prologue context (own stream, arena, flag)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cx::Arena arena;                // device scratch
    int* d_flag = nullptr;          // device-side error flag (softmax non-finite, ...)
    double* gaps = nullptr;         // decision-gap monitor: [gaps_n] of the last selection (device)
    int gaps_cap = 0, gaps_n = 0;
    int num_sms = 0;
    unsigned* fw_counters = nullptr;  // forward_step attention: per (agent, head) chunk counters (kept zero)
    int fw_counters_n = 0;
    // forward_step: the agents' batch lives in device memory (one H2D copy per step from a pinned
    // staging ring), so a step's launch sequence is the same for every token and replays as a
    // captured CUDA graph, keyed by everything the launches bake in
    static constexpr int kFwRing = 16;
    void* fw_dev = nullptr;                   // the batch (device)
    void* fw_host = nullptr;                  // [kFwRing] batches (pinned)
    cudaEvent_t fw_ev[kFwRing] = {};          // staging slot i is reusable once fw_ev[i] has fired
    int fw_slot = 0;
    struct FwGraph {
        const void* key[10];
        int nb, n_chunks;
        cudaGraphExec_t exec;
        uint64_t launches;
    };
    std::vector<FwGraph> fw_graphs;
    cx::Options opt;                // cx_ctx_set_option
    std::mutex mu;
};

// Device KvCache (model.hpp:67-113): storage in HBM, host-checked append protocol.
struct cx_kvcache {
    int n_layers, n_heads, d_model, d_k;
    int64_t max_positions;
    int64_t capacity = 0;
    float* keys = nullptr;    // [n_layers][capacity][d_model]
    float* values = nullptr;
    std::vector<int64_t> positions;
    std::vector<uint8_t> origins;
    int64_t last_context_position = -1;
    int64_t context_count = 0;
    bool entry_open = false;
    int layers_written = 0;
    cudaStream_t stream = nullptr;  // ordering for all of this cache's device work
    cudaEvent_t ev = nullptr;       // cross-stream ordering with appends on caller streams
};

// Weights in the reference's draw order (model.cpp:49-80): embedding [vocab][d],
// per layer {attn_norm [d], wq, wk, wv, wo [d][d], mlp_norm [d], w_in [dff][d],
// w_out [d][dff]}, final_norm [d], unembedding [vocab][d].
struct cx_weights {
    int n_layers = 0, n_heads = 0, d_model = 0, d_k = 0, vocab = 0;
    int64_t max_positions = 0;
    double rope_base = 10000.0;
    float* buf = nullptr;
    size_t per_layer = 0;
    size_t emb = 0, layers = 0, final_norm = 0, unemb = 0;  // offsets (floats)
    size_t attn_norm(int l) const { return layers + (size_t)l * per_layer; }
    size_t wq(int l) const { return attn_norm(l) + d_model; }
    size_t wk(int l) const { return wq(l) + (size_t)d_model * d_model; }
    size_t wv(int l) const { return wk(l) + (size_t)d_model * d_model; }
    size_t wo(int l) const { return wv(l) + (size_t)d_model * d_model; }
    size_t mlp_norm(int l) const { return wo(l) + (size_t)d_model * d_model; }
    size_t w_in(int l) const { return mlp_norm(l) + d_model; }
    size_t w_out(int l) const { return w_in(l) + (size_t)4 * d_model * d_model; }
};

namespace cx {

// KvCache stream ordering and growth (capi.cu)
void kv_before(cx_kvcache* c, cudaStream_t s);  // s waits for the cache's pending work
void kv_after(cx_kvcache* c, cudaStream_t s);   // the cache's stream waits for s
void kv_grow(cx_kvcache* c, int64_t need);      // capacity >= need rows (copies, synchronous)

// Thread-local default context for the reference-shaped host calls.
cx_ctx* default_ctx();

// Device error flags written by kernels (bitmask in ctx->d_flag).
enum : int {
    FLAG_NONFINITE = 1,    // CX_DEVERR_NONFINITE: a non-finite attention score (softmax precondition)
    FLAG_TAIL_RANGE = 2,   // CX_DEVERR_TAIL_RANGE: decode tail_len outside [0, t_cap - append]
};
static_assert(FLAG_NONFINITE == CX_DEVERR_NONFINITE && FLAG_TAIL_RANGE == CX_DEVERR_TAIL_RANGE, "flag bits");

// ---- launch helpers implemented in the .cu files ----------------------------
struct GroupView {  // device-side view of cx_groups
    int G;
    int64_t L;
    int dim;
    const float* X;
    int64_t gstride, rstride;
    const float* Q;
    int P, d_k, col_step;
};

// attention mass: out[G][L]; uses arena scratch (scores [G][P][L] + sums [G][P]).
void attention_grouped(cx_ctx* ctx, const GroupView& g, double* out, cudaStream_t s);
// bytes of arena scratch attention_grouped needs
void plan_attention(ArenaPlan& p, const GroupView& g);

// selection-monitor scratch per (group, round): one candidate per cluster CTA (<= 16)
constexpr int kGapRecStride = 16;
// the landmark K/V gather (A5) a selection may do itself once its picks are sorted:
// syn_k[g][s] = keys row rows[g][s], syn_v[g][s] = values row (values in the keys' group
// layout); blocks syn_gs floats apart.  Either output may be null.
struct SynGather {
    const float* values;
    float* syn_k;
    float* syn_v;
    int64_t syn_gs;
};
// greedy selection for all groups.  rows/scores out [G][take] ascending.  Returns true when
// the selection also did the gather `gat` (the tensor-core path); otherwise the caller gathers.
bool select_grouped(cx_ctx* ctx, const GroupView& g, const double* attn, int k, double lambda,
                    unsigned flags, int64_t* rows, double* scores, cudaStream_t s,
                    const double* centroids = nullptr /* [G][dim], computed here when null */,
                    const SynGather* gat = nullptr);
// d = 128 instantiation (select128.cu): the reference-mode cloud of a 2-head MHA cache
bool select128_launch(const GroupView& g, const Options& o, const double* attn, const double* cen, int take,
                      double lambda, unsigned flags, int64_t* pick_rows, double* pick_scores, int64_t* rows, double* scores,
                      double* gaps, double* gap_rec, cudaStream_t s);
int select128_wave(int64_t L, int G);
// gate.cpp:27-61 for n (h, t) pairs (row strides in floats): score (NaN when degenerate),
// accepted = score >= theta, degenerate = zero norm
void gate_decide(const float* h, int64_t hs, const float* t, int64_t ts, int64_t n, int dim, double theta,
                 double* score, uint8_t* accepted, uint8_t* degenerate, cudaStream_t s);
// groups per selection wave for G groups of L rows (dim 64), 0 if not on chip
int select64_wave(int64_t L, int G);
// centroid_of for every group (synapse.cpp:36-44), bit-exact sequential sums
void centroid_launch(const GroupView& g, double* cen, cudaStream_t s);
void plan_select(ArenaPlan& p, const GroupView& g, int k);
// d = 64 with the tensor-core filter and TMEM-resident rows (select_tc.cu); false when it
// does not apply
bool select_tc_launch(const GroupView& g, const Options& o, const double* attn, const double* cen, int take,
                      double lambda, unsigned flags, int64_t* pick_rows, double* pick_scores, int64_t* rows,
                      double* scores, double* gaps, void* scratch, cudaStream_t s,
                      const SynGather* gat = nullptr, bool* gathered = nullptr);
int select_tc_wave(int64_t L, int G);
size_t select_tc_scratch(int G);  // bytes of scratch select_tc_launch may use
// dim-64 fast path (select64.cu); false when it does not apply
bool select64_launch(const GroupView& g, const Options& o, const double* attn, const double* cen, int take,
                     double lambda, unsigned flags, int64_t* pick_rows, double* pick_scores, int64_t* rows, double* scores,
                     double* gaps, double* gap_rec, cudaStream_t s);

// gather selected rows from a (values or keys) tensor with the group addressing.
void gather_rows(const GroupView& g, const float* src, const int64_t* rows, int take, float* dst,
                 cudaStream_t s);
// keys and values in one launch; destination group blocks dst_gstride floats apart
void gather_rows2(const GroupView& g, const float* src0, const float* src1, const int64_t* rows, int take, float* dst0,
                  float* dst1, int64_t dst_gstride, cudaStream_t s);

// coverage_scores_points with a non-empty selection (one group).
void coverage_selected(const GroupView& g, const int64_t* sel, int64_t n_sel, double* out,
                       cudaStream_t s);
// centroid + centroid-distance coverage (one group).
void coverage_centroid(cx_ctx* ctx, const GroupView& g, double* out, cudaStream_t s);

// metrics (one cloud): sq-dist min/max reduction and pairwise means.
void hausdorff(const float* cloud, int64_t count, int dim, const float* lm, int64_t m,
               const int64_t* rows, double* out_worst_sq, cudaStream_t s);
// doubles of scratch mean_pairwise needs at out_sum (the sum, then its working space)
size_t mean_pairwise_scratch(int64_t count, int dim);
void mean_pairwise(const float* pts, int64_t count, int dim, const int64_t* rows, double* out_sum,
                   cudaStream_t s);

// kernels::softmax / argmax (kernels.cpp:66-101), one vector per call
void softmax_fp64(const double* s, int64_t n, double* out, int* flag, cudaStream_t st);
void argmax_f32(const float* v, int64_t n, int* out, cudaStream_t st);
// attend (reference-shaped, fp64 accumulate)
void attend_fp64_ws(const float* q, const float* k, const float* v, int64_t n, int H, int dk,
                    double* w /* [H][n] scratch */, float* out, cudaStream_t s);
// batched decode step (fp32 accumulate)
void decode_step(cx_ctx* ctx, const cx_decode_batch& b, cudaStream_t s);
// tcgen05 variant (decode_tc.cu); false when the shape does not apply
bool decode_tc_launch(cx_ctx* ctx, const cx_decode_batch& b, cudaStream_t s);

// KV append: copies block [n_layers][T][d_model] (device) into the cache
// arrays at rows [dst_row, dst_row+T) of every layer.
void kv_append_rows(float* cache_k, float* cache_v, int64_t capacity, int n_layers, int d_model,
                    const float* blk_k, const float* blk_v, int64_t T, int64_t dst_row,
                    cudaStream_t s);

}  // namespace cx

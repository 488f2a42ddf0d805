// cortex_runtime.cu -- the River / Stream loop on the device (SURVEY.md §8(f) row 2,
// BASELINE configs[4]): Scheduler::run's device work (scheduler.cpp:63-165) behind
// the C-ABI.
//
// River lane (the device's greatest stream priority; driven by the calling thread),
// per river token:
//   * every inject_every tokens, drain_injections (scheduler.cpp:139-156): a thought is
//     encoded context-blind at reserved virtual positions (encode_thought,
//     injector.cpp:36-68, on a scratch cache) and appended to the river cache (inject,
//     :70-94) -- the token attends over it;
//   * the token's forward_step on the river KvCache (model.cpp:175-235), which also
//     appends its row to a contiguous mirror of the context rows (context_key_cloud's
//     compaction, synapse.cpp:48-61, kept incrementally);
//   * every push_every tokens, push_synapse (scheduler.cpp:158-165) into the BACK
//     buffer, in the decode layout [layer][kv][k][d_k]: either the reference's
//     select_landmarks over the last layer with the river's final query
//     (CX_CORTEX_PUSH_SCHEDULER, synapse.cpp:286-323) or one selection per (layer,
//     KV head) (CX_CORTEX_PUSH_GROUPS).
// Stream lane (medium priority; a second host thread, so agent steps are issued at
// their own pace as the reference's agent threads run, scheduler.cpp:198): each agent
// step is N agents x every layer decoding one token against the FRONT synapse
// (append + attend, decode_tc.cu), one CUDA-graph replay per step (a graph per buffer).
// Publication (SynapseBuffer::push / read_latest, synapse.hpp:115-135): a push becomes
// the front at the first agent step after its completion event fired (a non-blocking
// query), and that step waits on the event: an agent step never reads a partly written
// synapse.  A push into a buffer first waits for the last agent step that read it.
// Versions are 1, 2, ...; each host thread runs at most kAhead steps ahead of its lane.
#include <algorithm>
#include <exception>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "cx_internal.cuh"

struct cx_cortex {
    cx_ctx* ctx = nullptr;
    const cx_weights* w = nullptr;
    cx_kvcache* river = nullptr;
    cx_cortex_config cfg{};
    cx_cortex_agents ag{};
    int n_layers = 0, n_kv = 0, d_k = 0, d_model = 0;
    cudaStream_t rs = nullptr, ss = nullptr;  // river / stream lanes (ctx-owned)
    // synapse double buffer [2][K | V][layer][kv][k][d_k]
    float* syn = nullptr;
    size_t syn_floats = 0;  // one K (or V) block
    // the river's CONTEXT rows, contiguous ([layer][ctx_cap][d_model], context_key_cloud's
    // compaction kept incrementally: every new river row is appended here too), so pushes
    // read them with plain strides although injected rows interleave in the river cache
    float* ctx_k = nullptr;
    float* ctx_v = nullptr;
    int64_t ctx_cap = 0, ctx_n = 0;
    int64_t* rows = nullptr;  // compress outputs [n_kv][n_layers][k]
    double* scores = nullptr;
    int front = -1;
    uint64_t version = 0, front_version = 0;
    bool inflight = false;
    int inflight_buf = 0;
    cudaEvent_t push_start = nullptr, push_done = nullptr, reader_done[2] = {nullptr, nullptr};
    cudaGraphExec_t agent_graph[2] = {nullptr, nullptr};
    cx_kvcache* scratch = nullptr;  // encode_thought
    float* dev_out = nullptr;       // river logits (one token)
    int64_t virtual_next = 0;
    int64_t position = 0;  // next river position
    double push_ms_sum = 0.0;
    int pushes = 0, injections = 0;
    cudaEvent_t t0 = nullptr, t_river = nullptr, t_stream = nullptr;
    float* fq = nullptr;      // the river's last final query [d_model] (CX_CORTEX_PUSH_SCHEDULER)
    double* attn = nullptr;   // push attention [ctx_cap]
    std::mutex mu;            // front / version / inflight, shared by the two host threads
    cudaEvent_t rev[8] = {}, aev[8] = {};  // per-lane step completion rings (host throttle)
    // the thought gate (cfg.gate): the river's latest hidden state and the thought's last one
    // [2][d_model], the device decision, its pinned host copy, the run's log
    float* hid = nullptr;
    double* g_score = nullptr;      // device: score, then accepted / degenerate bytes
    double* g_host = nullptr;       // pinned: score, flags
    struct GateRec {
        int64_t id;
        double score;
        uint8_t accepted, degenerate;
    };
    std::vector<GateRec> gate_log;
    int accepted = 0, rejected = 0;
};

namespace cx {
namespace {

constexpr int kAhead = 4;  // steps a host thread may run ahead of its lane

// syn[l][h][s][:] = mirror[l][rows[s]][h * d_k : (h + 1) * d_k] for every layer and head
// (select_landmarks' per-layer landmark K/V, synapse.cpp:303-318, in the decode layout)
__global__ void cortex_gather_kernel(const float* __restrict__ ck, const float* __restrict__ cv, int64_t ctx_cap,
                                     int d_model, int n_kv, int d_k, const int64_t* __restrict__ rows, int k,
                                     float* __restrict__ sk, float* __restrict__ sv) {
    const int s = blockIdx.x, l = blockIdx.y;
    const int64_t row = rows[s];
    const float4* srck = reinterpret_cast<const float4*>(ck + ((size_t)l * ctx_cap + row) * d_model);
    const float4* srcv = reinterpret_cast<const float4*>(cv + ((size_t)l * ctx_cap + row) * d_model);
    for (int c4 = threadIdx.x; c4 < d_model / 4; c4 += blockDim.x) {
        const int c = c4 * 4, h = c / d_k, j = c % d_k;
        const size_t o = (((size_t)l * n_kv + h) * k + s) * d_k + j;
        *reinterpret_cast<float4*>(sk + o) = srck[c4];
        *reinterpret_cast<float4*>(sv + o) = srcv[c4];
    }
}

void make_events(cx_cortex* r) {
    for (int i = 0; i < kAhead; ++i) {
        CX_CUDA(cudaEventCreateWithFlags(&r->rev[i], cudaEventDisableTiming));
        CX_CUDA(cudaEventCreateWithFlags(&r->aev[i], cudaEventDisableTiming));
    }
    CX_CUDA(cudaEventCreate(&r->push_start));
    CX_CUDA(cudaEventCreate(&r->push_done));
    CX_CUDA(cudaEventCreateWithFlags(&r->reader_done[0], cudaEventDisableTiming));
    CX_CUDA(cudaEventCreateWithFlags(&r->reader_done[1], cudaEventDisableTiming));
    CX_CUDA(cudaEventCreate(&r->t0));
    CX_CUDA(cudaEventCreate(&r->t_river));
    CX_CUDA(cudaEventCreate(&r->t_stream));
}

cx_decode_batch agent_batch(cx_cortex* r, int buf) {
    cx_decode_batch b{};
    b.n_agents = r->cfg.n_agents;
    b.n_layers = r->n_layers;
    b.n_kv = r->n_kv;
    b.n_q = r->cfg.n_q;
    b.d_k = r->d_k;
    b.k_syn = r->cfg.k;
    b.syn_keys = r->syn + (size_t)(2 * buf) * r->syn_floats;
    b.syn_values = r->syn + (size_t)(2 * buf + 1) * r->syn_floats;
    b.tail_keys = r->ag.tail_keys;
    b.tail_values = r->ag.tail_values;
    b.t_cap = r->cfg.t_cap;
    b.tail_len = r->ag.tail_len;
    b.new_keys = r->ag.new_keys;
    b.new_values = r->ag.new_values;
    b.q = r->ag.q;
    b.out = r->ag.out;
    b.flags = CX_DECODE_SYN_UNCHANGED;  // between publishes the front buffer is never written
    return b;
}

// push_synapse (scheduler.cpp:158-165) of the context rows so far -> syn[buf]
void push(cx_cortex* r, int buf) {
    cx::NvtxRange range("cortex push_synapse");
    const int64_t L = r->ctx_n;
    // the last agent step that read this buffer is done with it
    CX_CUDA(cudaStreamWaitEvent(r->rs, r->reader_done[buf], 0));
    CX_CUDA(cudaEventRecord(r->push_start, r->rs));
    const int k = r->cfg.k;
    float* sk_buf = r->syn + (size_t)(2 * buf) * r->syn_floats;
    float* sv_buf = r->syn + (size_t)(2 * buf + 1) * r->syn_floats;
    if (r->cfg.push_mode == CX_CORTEX_PUSH_SCHEDULER) {
        // select_landmarks(cache, last_query, k, lambda) (synapse.cpp:286-323): the last
        // layer's context keys, MHA attention with the river's final query, one row set
        cx_groups g{};
        g.n_groups = 1;
        g.count = L;
        g.dim = r->d_model;
        g.clouds = r->ctx_k + (size_t)(r->n_layers - 1) * r->ctx_cap * r->d_model;
        g.group_stride = r->ctx_cap * r->d_model;
        g.row_stride = r->d_model;
        g.queries = r->fq;
        g.n_pass = r->n_kv;
        g.d_k = r->d_k;
        g.col_step = r->d_k;
        cx_status st = cx_attention_grouped_dev(r->ctx, &g, r->attn, r->rs);
        if (st == CX_OK) st = cx_select_grouped_dev(r->ctx, &g, r->attn, k, r->cfg.lambda, 0u, r->rows, r->scores, r->rs);
        if (st != CX_OK) fail(st, cx_last_error());
        cortex_gather_kernel<<<dim3((unsigned)k, (unsigned)r->n_layers), 128, 0, r->rs>>>(
            r->ctx_k, r->ctx_v, r->ctx_cap, r->d_model, r->n_kv, r->d_k, r->rows, k, sk_buf, sv_buf);
        CX_CUDA(cudaGetLastError());
        count_launch();
    } else {
        const int qpg = r->cfg.n_q / r->n_kv;
        for (int h = 0; h < r->n_kv; ++h) {
            cx_groups g{};
            g.n_groups = r->n_layers;
            g.count = L;
            g.dim = r->d_k;
            g.clouds = r->ctx_k + (size_t)h * r->d_k;
            g.group_stride = r->ctx_cap * r->d_model;
            g.row_stride = r->d_model;
            g.queries = r->ag.river_queries + (size_t)h * r->n_layers * qpg * r->d_k;
            g.n_pass = qpg;
            g.d_k = r->d_k;
            g.col_step = 0;  // GQA: every query of the group against the head's d_k columns
            const cx_status st = cx_compress_grouped_strided_dev(
                r->ctx, &g, r->ctx_v + (size_t)h * r->d_k, k, r->cfg.lambda, 0u, r->rows + (size_t)h * r->n_layers * k,
                r->scores + (size_t)h * r->n_layers * k, sk_buf + (size_t)h * k * r->d_k, sv_buf + (size_t)h * k * r->d_k,
                (int64_t)r->n_kv * k * r->d_k, r->rs);
            if (st != CX_OK) fail(st, cx_last_error());
        }
    }
    CX_CUDA(cudaEventRecord(r->push_done, r->rs));
}

// read_latest at an agent step boundary: a landed push becomes the front buffer
// (caller holds r->mu).  `wait`: block until the inflight push lands (end of a run).
void publish_if_landed(cx_cortex* r, bool wait, float* history, int max_versions) {
    if (!r->inflight) return;
    if (wait) {
        CX_CUDA(cudaEventSynchronize(r->push_done));
    } else {
        const cudaError_t q = cudaEventQuery(r->push_done);
        if (q == cudaErrorNotReady) return;
        CX_CUDA(q);
    }
    float ms = 0.f;
    CX_CUDA(cudaEventElapsedTime(&ms, r->push_start, r->push_done));
    r->push_ms_sum += ms;
    r->pushes += 1;
    CX_CUDA(cudaStreamWaitEvent(r->ss, r->push_done, 0));
    CX_CUDA(cudaEventRecord(r->reader_done[r->front], r->ss));  // the old front: readers done after this
    r->front = r->inflight_buf;
    r->front_version = ++r->version;
    r->inflight = false;
    if (history && (int64_t)r->front_version < max_versions)  // audit: the published bytes
        CX_CUDA(cudaMemcpyAsync(history + (size_t)r->front_version * 2 * r->syn_floats,
                                r->syn + (size_t)(2 * r->front) * r->syn_floats, sizeof(float) * 2 * r->syn_floats,
                                cudaMemcpyDeviceToDevice, r->ss));
}

// the river cache's row `row` (every layer) -> the context mirror's next row
void mirror_row(cx_cortex* r, int64_t row) {
    if (r->ctx_n >= r->ctx_cap) fail(CX_CAPACITY_ERROR, "cortex: context mirror full (max_context)");
    cx_kvcache* kc = r->river;
    const size_t dm = (size_t)r->d_model;
    CX_CUDA(cudaMemcpy2DAsync(r->ctx_k + r->ctx_n * dm, r->ctx_cap * dm * sizeof(float), kc->keys + row * dm,
                              kc->capacity * dm * sizeof(float), dm * sizeof(float), r->n_layers,
                              cudaMemcpyDeviceToDevice, r->rs));
    CX_CUDA(cudaMemcpy2DAsync(r->ctx_v + r->ctx_n * dm, r->ctx_cap * dm * sizeof(float), kc->values + row * dm,
                              kc->capacity * dm * sizeof(float), dm * sizeof(float), r->n_layers,
                              cudaMemcpyDeviceToDevice, r->rs));
    r->ctx_n += 1;
}

// drain_injections: encode the thought at the next virtual positions, append it to the river
void inject_thought(cx_cortex* r, const int* thought, int64_t thought_id, int64_t stream_position) {
    cx::NvtxRange range("cortex drain_injections");
    const int T = r->cfg.thought_tokens;
    cx_kvcache* sc = r->scratch;
    // a fresh scratch cache per thought (encode_thought's KvCache scratch(cfg))
    sc->positions.clear();
    sc->origins.clear();
    sc->last_context_position = -1;
    sc->context_count = 0;
    for (int t = 0; t < T; ++t) {
        const int64_t pos = r->virtual_next + t;
        // the last token's hidden state is the thought's t_side (encode_thought's last_hidden)
        float* h = (r->cfg.gate && t == T - 1) ? r->hid + r->d_model : nullptr;
        const cx_status st = cx_forward_step_dev(r->ctx, r->w, 1, &sc, thought + t, &pos, nullptr, h, nullptr, r->rs);
        if (st != CX_OK) fail(st, cx_last_error());
    }
    // the scratch cache holds exactly T rows per layer ([layer][T][d] when its capacity is T)
    if (sc->capacity != T) fail(CX_DEVICE_ERROR, "cortex: the scratch cache must hold exactly the thought's rows");
    if (r->cfg.gate) {
        // decide(river hidden, thought hidden, theta) (gate.cpp:45-61) on the device; the host
        // needs the verdict (a rejected thought leaves the river cache unchanged), so the river
        // lane is synchronised once per thought
        uint8_t* flags = reinterpret_cast<uint8_t*>(r->g_score + 1);
        const cx_status gs = cx_gate_decide_dev(r->ctx, 1, r->d_model, r->hid, r->d_model, r->hid + r->d_model,
                                                r->d_model, r->cfg.theta, r->g_score, flags, flags + 1, r->rs);
        if (gs != CX_OK) fail(gs, cx_last_error());
        CX_CUDA(cudaMemcpyAsync(r->g_host, r->g_score, 2 * sizeof(double), cudaMemcpyDeviceToHost, r->rs));
        CX_CUDA(cudaStreamSynchronize(r->rs));
        const uint8_t* hf = reinterpret_cast<const uint8_t*>(r->g_host + 1);
        r->gate_log.push_back({thought_id, r->g_host[0], hf[0], hf[1]});
        if (!hf[0]) {  // rejected (scheduler.cpp:299-302): not injected, the virtual range is reused
            r->rejected += 1;
            return;
        }
        r->accepted += 1;
    }
    cx_injection_record rec{};
    const cx_status st = cx_inject_dev(r->river, sc->keys, sc->values, r->virtual_next, T, r->n_layers, r->d_model,
                                       thought_id, stream_position, &rec, r->rs);
    if (st != CX_OK) fail(st, cx_last_error());
    r->virtual_next += T;
    r->injections += 1;
}

}  // namespace
}  // namespace cx

using namespace cx;

extern "C" cx_status cx_cortex_create(cx_ctx* ctx, const cx_weights* w, cx_kvcache* river, const cx_cortex_config* cfg,
                                      const cx_cortex_agents* agents, cx_cortex** out) {
    return guard(__func__, [&] {
        if (!ctx || !w || !river || !cfg || !agents || !out) fail(CX_INVALID_ARGUMENT, "null argument");
        if (cfg->n_agents < 1 || cfg->k < 1 || cfg->push_every < 1 || cfg->inject_every < 1 || cfg->thought_tokens < 1 ||
            cfg->t_cap < 1 || cfg->n_q < river->n_heads || cfg->n_q % river->n_heads != 0)
            fail(CX_CONFIG_ERROR, "cortex: bad configuration");
        if (cfg->lambda < 0.0 || cfg->lambda > 1.0) fail(CX_CONFIG_ERROR, "select_landmarks: lambda must be in [0,1]");
        if (cfg->push_mode != CX_CORTEX_PUSH_SCHEDULER && cfg->push_mode != CX_CORTEX_PUSH_GROUPS)
            fail(CX_CONFIG_ERROR, "cortex: unknown push_mode");
        if (cfg->push_mode == CX_CORTEX_PUSH_GROUPS && !agents->river_queries)
            fail(CX_INVALID_ARGUMENT, "cortex: CX_CORTEX_PUSH_GROUPS needs river_queries");
        if (cfg->virtual_base <= river->last_context_position || cfg->virtual_base >= river->max_positions)
            fail(CX_CONFIG_ERROR, "cortex: virtual_base must lie between the river and max_positions");
        if (river->entry_open) fail(CX_SEQUENCING_ERROR, "cortex: river cache has an open entry");
        if (river->context_count != (int64_t)river->positions.size())
            fail(CX_PRECONDITION_ERROR, "cortex: the river cache must hold only context rows at creation");
        if (river->context_count < cfg->k) fail(CX_PRECONDITION_ERROR, "cortex: fewer context rows than k");
        if (cfg->gate && (cfg->theta < -1.0 || cfg->theta > 1.0))
            fail(CX_PRECONDITION_ERROR, "decide: theta must be in [-1,1]");
        auto r = std::make_unique<cx_cortex>();
        r->ctx = ctx;
        r->w = w;
        r->river = river;
        r->cfg = *cfg;
        r->ag = *agents;
        r->n_layers = river->n_layers;
        r->n_kv = river->n_heads;
        r->d_k = river->d_k;
        r->d_model = river->d_model;
        int prio = 0;
        void* st = nullptr;
        if (cx_ctx_lane_stream(ctx, CX_LANE_RIVER, &st, &prio) != CX_OK) fail(CX_DEVICE_ERROR, cx_last_error());
        r->rs = (cudaStream_t)st;
        if (cx_ctx_lane_stream(ctx, CX_LANE_STREAM, &st, &prio) != CX_OK) fail(CX_DEVICE_ERROR, cx_last_error());
        r->ss = (cudaStream_t)st;
        r->syn_floats = (size_t)r->n_layers * r->n_kv * cfg->k * r->d_k;
        CX_CUDA(cudaMalloc(&r->syn, sizeof(float) * 4 * r->syn_floats));
        CX_CUDA(cudaMemset(r->syn, 0, sizeof(float) * 4 * r->syn_floats));
        CX_CUDA(cudaMalloc(&r->rows, sizeof(int64_t) * r->n_kv * r->n_layers * cfg->k));
        CX_CUDA(cudaMalloc(&r->scores, sizeof(double) * r->n_kv * r->n_layers * cfg->k));
        CX_CUDA(cudaMalloc(&r->dev_out, sizeof(float) * std::max(4096, w->vocab)));
        CX_CUDA(cudaMalloc(&r->fq, sizeof(float) * r->d_model));
        CX_CUDA(cudaMemset(r->fq, 0, sizeof(float) * r->d_model));
        // gate buffers; the river hidden starts at zero (no river token yet: a degenerate,
        // rejected decision, as decide() gives a zero-norm input)
        CX_CUDA(cudaMalloc(&r->hid, sizeof(float) * 2 * r->d_model));
        CX_CUDA(cudaMemset(r->hid, 0, sizeof(float) * 2 * r->d_model));
        CX_CUDA(cudaMalloc(&r->g_score, 2 * sizeof(double)));
        CX_CUDA(cudaMallocHost(&r->g_host, 2 * sizeof(double)));
        // the context mirror (the river holds only context rows, checked above)
        r->ctx_cap = std::max<int64_t>(cfg->max_context, river->context_count);
        CX_CUDA(cudaMalloc(&r->ctx_k, sizeof(float) * r->n_layers * r->ctx_cap * r->d_model));
        CX_CUDA(cudaMalloc(&r->ctx_v, sizeof(float) * r->n_layers * r->ctx_cap * r->d_model));
        CX_CUDA(cudaMalloc(&r->attn, sizeof(double) * r->ctx_cap));
        CX_CUDA(cudaStreamSynchronize(river->stream));
        {
            const size_t dm = (size_t)r->d_model;
            const int64_t n = river->context_count;
            CX_CUDA(cudaMemcpy2DAsync(r->ctx_k, r->ctx_cap * dm * sizeof(float), river->keys,
                                      river->capacity * dm * sizeof(float), n * dm * sizeof(float), r->n_layers,
                                      cudaMemcpyDeviceToDevice, r->rs));
            CX_CUDA(cudaMemcpy2DAsync(r->ctx_v, r->ctx_cap * dm * sizeof(float), river->values,
                                      river->capacity * dm * sizeof(float), n * dm * sizeof(float), r->n_layers,
                                      cudaMemcpyDeviceToDevice, r->rs));
            r->ctx_n = n;
        }
        make_events(r.get());
        CX_CUDA(cudaEventRecord(r->reader_done[0], r->ss));
        CX_CUDA(cudaEventRecord(r->reader_done[1], r->ss));
        cx_kvcache* sc = nullptr;
        if (cx_kvcache_create(r->n_layers, r->n_kv, r->d_model, r->d_k, river->max_positions, cfg->thought_tokens, &sc) !=
            CX_OK)
            fail(CX_DEVICE_ERROR, cx_last_error());
        r->scratch = sc;
        r->virtual_next = cfg->virtual_base;
        r->position = river->last_context_position + 1;
        // the agent step, captured once per synapse buffer (decode_tc: one launch)
        for (int buf = 0; buf < 2; ++buf) {
            cx_decode_batch b = agent_batch(r.get(), buf);
            cudaGraph_t g = nullptr;
            CX_CUDA(cudaStreamBeginCapture(r->ss, cudaStreamCaptureModeThreadLocal));
            const cx_status st2 = cx_decode_step_dev(ctx, &b, r->ss);
            cudaGraph_t g2 = nullptr;
            const cudaError_t e = cudaStreamEndCapture(r->ss, &g2);
            g = g2;
            if (st2 != CX_OK) fail(st2, cx_last_error());
            CX_CUDA(e);
            CX_CUDA(cudaGraphInstantiate(&r->agent_graph[buf], g, 0));
            cudaGraphDestroy(g);
        }
        // the first synapse: pushed and published before the loop (Scheduler::run pushes
        // once the prompt is in, scheduler.cpp:63-113)
        push(r.get(), 0);
        CX_CUDA(cudaEventSynchronize(r->push_done));
        r->front = 0;
        r->version = r->front_version = 1;
        CX_CUDA(cudaStreamWaitEvent(r->ss, r->push_done, 0));
        *out = r.release();
    });
}

namespace cx {
namespace {

// the stream lane: n_steps agent steps, each a graph replay against the front synapse
void agent_lane(cx_cortex* r, int n_steps, uint64_t* versions_used, float* out_history, float* history,
                int max_versions) {
    CX_CUDA(cudaSetDevice(r->ctx->device));
    const size_t n_out = (size_t)r->cfg.n_agents * r->n_layers * r->cfg.n_q * r->d_k;
    for (int s = 0; s < n_steps; ++s) {
        cx::NvtxRange range("cortex agent step");
        if (s >= kAhead) CX_CUDA(cudaEventSynchronize(r->aev[s % kAhead]));
        uint64_t ver = 0;
        {
            std::lock_guard<std::mutex> lk(r->mu);
            publish_if_landed(r, false, history, max_versions);
            CX_CUDA(cudaGraphLaunch(r->agent_graph[r->front], r->ss));
            ver = r->front_version;
        }
        count_launch();
        if (out_history)  // audit: what the agents computed at this step
            CX_CUDA(cudaMemcpyAsync(out_history + (size_t)s * n_out, r->ag.out, sizeof(float) * n_out,
                                    cudaMemcpyDeviceToDevice, r->ss));
        CX_CUDA(cudaEventRecord(r->aev[s % kAhead], r->ss));
        if (versions_used) versions_used[s] = ver;
    }
}

// the river lane: n_tokens river tokens with their injections and pushes
void river_lane(cx_cortex* r, int n_tokens, const int* river_tokens, const int* thought_tokens, float* river_logits) {
    const int V = r->w->vocab, inj = r->cfg.inject_every;
    for (int t = 0; t < n_tokens; ++t) {
        cx::NvtxRange range("cortex river token");
        if (t >= kAhead) CX_CUDA(cudaEventSynchronize(r->rev[t % kAhead]));
        if (r->position >= r->cfg.virtual_base)  // scheduler.cpp step_token
            fail(CX_CAPACITY_ERROR, "river stream reached the reserved virtual range");
        // drain_injections: the thought is in the river before this token
        if (t % inj == 0)
            inject_thought(r, thought_tokens + (size_t)(t / inj) * r->cfg.thought_tokens, t / inj, r->position - 1);
        cx_kvcache* kc = r->river;
        const int64_t pos = r->position;
        const cx_status st =
            cx_forward_step_dev(r->ctx, r->w, 1, &kc, river_tokens + t, &pos, r->dev_out, r->cfg.gate ? r->hid : nullptr,
                                r->fq, r->rs);
        if (st != CX_OK) fail(st, cx_last_error());
        r->position += 1;
        mirror_row(r, (int64_t)kc->positions.size() - 1);  // the new context row
        if (river_logits)
            CX_CUDA(cudaMemcpyAsync(river_logits + (size_t)t * V, r->dev_out, sizeof(float) * V,
                                    cudaMemcpyDeviceToDevice, r->rs));
        CX_CUDA(cudaEventRecord(r->rev[t % kAhead], r->rs));
        if ((t + 1) % r->cfg.push_every == 0) {  // (now + 1) % synapse_push_period == 0
            int buf = -1;
            {
                std::lock_guard<std::mutex> lk(r->mu);
                if (!r->inflight) buf = 1 - r->front;
            }
            if (buf >= 0) {
                push(r, buf);  // the agent lane never touches the back buffer
                std::lock_guard<std::mutex> lk(r->mu);
                r->inflight = true;
                r->inflight_buf = buf;
            }
        }
    }
}

}  // namespace
}  // namespace cx

extern "C" cx_status cx_cortex_run(cx_cortex* r, int n_tokens, const int* river_tokens, const int* thought_tokens,
                                   int n_agent_steps, cx_cortex_stats* stats, uint64_t* versions_used,
                                   float* river_logits, float* synapse_history, int max_versions, float* out_history) {
    return guard(__func__, [&] {
        if (!r || (n_tokens > 0 && (!river_tokens || !thought_tokens))) fail(CX_INVALID_ARGUMENT, "null argument");
        if (n_tokens < 0 || n_agent_steps < 0) fail(CX_INVALID_ARGUMENT, "negative step count");
        for (int t = 0; t < n_tokens; ++t)
            if (river_tokens[t] < 0 || river_tokens[t] >= r->w->vocab)
                fail(CX_PRECONDITION_ERROR, "river token outside vocabulary");
        const int64_t n_th = (int64_t)((n_tokens + r->cfg.inject_every - 1) / r->cfg.inject_every) * r->cfg.thought_tokens;
        for (int64_t i = 0; i < n_th; ++i)  // scheduler.cpp:67-74
            if (thought_tokens[i] < 0 || thought_tokens[i] >= r->w->vocab)
                fail(CX_PRECONDITION_ERROR, "script token outside vocabulary");
        r->push_ms_sum = 0.0;
        r->pushes = 0;
        r->injections = 0;
        r->accepted = r->rejected = 0;
        r->gate_log.clear();
        if (synapse_history && (int64_t)r->front_version < max_versions)  // the version published before the run
            CX_CUDA(cudaMemcpyAsync(synapse_history + (size_t)r->front_version * 2 * r->syn_floats,
                                    r->syn + (size_t)(2 * r->front) * r->syn_floats, sizeof(float) * 2 * r->syn_floats,
                                    cudaMemcpyDeviceToDevice, r->ss));
        CX_CUDA(cudaEventRecord(r->t0, r->ss));
        CX_CUDA(cudaStreamWaitEvent(r->rs, r->t0, 0));
        std::exception_ptr agent_err;
        std::thread agents;
        if (n_agent_steps > 0)
            agents = std::thread([&] {
                try {
                    agent_lane(r, n_agent_steps, versions_used, out_history, synapse_history, max_versions);
                } catch (...) {
                    agent_err = std::current_exception();
                }
            });
        std::exception_ptr river_err;
        try {
            river_lane(r, n_tokens, river_tokens, thought_tokens, river_logits);
        } catch (...) {
            river_err = std::current_exception();
        }
        if (agents.joinable()) agents.join();
        if (river_err) std::rethrow_exception(river_err);
        if (agent_err) std::rethrow_exception(agent_err);
        CX_CUDA(cudaEventRecord(r->t_stream, r->ss));
        CX_CUDA(cudaEventRecord(r->t_river, r->rs));
        CX_CUDA(cudaEventSynchronize(r->t_stream));
        CX_CUDA(cudaEventSynchronize(r->t_river));
        {
            std::lock_guard<std::mutex> lk(r->mu);  // a push still in flight at the end lands now
            publish_if_landed(r, true, synapse_history, max_versions);
        }
        CX_CUDA(cudaStreamSynchronize(r->ss));
        if (stats) {
            float a = 0.f, b = 0.f;
            CX_CUDA(cudaEventElapsedTime(&a, r->t0, r->t_stream));
            CX_CUDA(cudaEventElapsedTime(&b, r->t0, r->t_river));
            stats->agent_ms = a;
            stats->river_ms = b;
            stats->pushes = r->pushes;
            stats->injections = r->injections;
            stats->push_ms_mean = r->pushes ? r->push_ms_sum / r->pushes : 0.0;
            stats->last_version = r->version;
            stats->thoughts_accepted = r->accepted;
            stats->thoughts_rejected = r->rejected;
        }
    });
}

// the synapse of the front buffer (the latest published version) -> device copies
extern "C" cx_status cx_cortex_front_synapse(const cx_cortex* r, float* keys, float* values, uint64_t* version) {
    return guard(__func__, [&] {
        if (!r) fail(CX_INVALID_ARGUMENT, "null runtime");
        CX_CUDA(cudaStreamSynchronize(r->ss));
        if (keys)
            CX_CUDA(cudaMemcpy(keys, r->syn + (size_t)(2 * r->front) * r->syn_floats, sizeof(float) * r->syn_floats,
                               cudaMemcpyDefault));
        if (values)
            CX_CUDA(cudaMemcpy(values, r->syn + (size_t)(2 * r->front + 1) * r->syn_floats, sizeof(float) * r->syn_floats,
                               cudaMemcpyDefault));
        if (version) *version = r->front_version;
    });
}

extern "C" cx_status cx_cortex_gate_log(const cx_cortex* r, int64_t max, int64_t* thought_ids, double* scores,
                                        uint8_t* accepted, uint8_t* degenerate, int64_t* n) {
    return guard(__func__, [&] {
        if (!r || !n) fail(CX_INVALID_ARGUMENT, "null argument");
        const int64_t m = std::min<int64_t>(max, (int64_t)r->gate_log.size());
        for (int64_t i = 0; i < m; ++i) {
            if (thought_ids) thought_ids[i] = r->gate_log[i].id;
            if (scores) scores[i] = r->gate_log[i].score;
            if (accepted) accepted[i] = r->gate_log[i].accepted;
            if (degenerate) degenerate[i] = r->gate_log[i].degenerate;
        }
        *n = (int64_t)r->gate_log.size();
    });
}

extern "C" cx_status cx_cortex_destroy(cx_cortex* r) {
    return guard(__func__, [&] {
        if (!r) return;
        cudaStreamSynchronize(r->ss);
        cudaStreamSynchronize(r->rs);
        for (auto g : r->agent_graph)
            if (g) cudaGraphExecDestroy(g);
        for (int i = 0; i < kAhead; ++i) {
            if (r->rev[i]) cudaEventDestroy(r->rev[i]);
            if (r->aev[i]) cudaEventDestroy(r->aev[i]);
        }
        for (cudaEvent_t e : {r->push_start, r->push_done, r->reader_done[0], r->reader_done[1], r->t0, r->t_river,
                              r->t_stream})
            if (e) cudaEventDestroy(e);
        if (r->scratch) cx_kvcache_destroy(r->scratch);
        cudaFree(r->syn);
        cudaFree(r->rows);
        cudaFree(r->scores);
        cudaFree(r->dev_out);
        cudaFree(r->ctx_k);
        cudaFree(r->ctx_v);
        cudaFree(r->fq);
        cudaFree(r->attn);
        cudaFree(r->hid);
        cudaFree(r->g_score);
        if (r->g_host) cudaFreeHost(r->g_host);
        delete r;
    });
}

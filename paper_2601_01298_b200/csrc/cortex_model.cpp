// cortex_model.cpp -- the cortex:: model drop-in (include/cortex/model.hpp,
// injector.hpp encode_thought, kernels.hpp projections) over the C-ABI.
//
// WeightStore::init must reproduce the reference's parameters bit for bit (the
// same seeded stream, model.cpp:49-80), so it keeps the reference's draw order;
// everything that computes -- forward_step, encode_thought, the kernels::
// primitives -- runs on the device (forward.cu).
#include <cmath>
#include <mutex>
#include <stdexcept>

#include "cortex/errors.hpp"
#include "cortex/injector.hpp"
#include "cortex/kernels.hpp"
#include "cortex/model.hpp"
#include "cortex/rng.hpp"
#include "cortex_b200.h"

namespace cortex {

namespace {

void ck(cx_status st) {
    if (st == CX_OK) return;
    const std::string msg = cx_last_error();
    switch (st) {
        case CX_CONFIG_ERROR: throw config_error(msg);
        case CX_CAPACITY_ERROR: throw capacity_error(msg);
        case CX_TOPOLOGY_ERROR: throw topology_error(msg);
        case CX_SEQUENCING_ERROR: throw sequencing_error(msg);
        case CX_PRECONDITION_ERROR: throw precondition_error(msg);
        case CX_CAP_ERROR: throw cap_error(msg);
        case CX_DEGENERATE_INPUT_ERROR: throw degenerate_input_error(msg);
        default: throw device_error(msg);
    }
}

void fill(Rng& rng, std::vector<float>& dst, size_t n, double mean, double stddev) {
    dst.resize(n);
    for (size_t i = 0; i < n; ++i) dst[i] = static_cast<float>(rng.next_gaussian(mean, stddev));
}

// one device context per host thread for the reference-shaped (synchronous) model calls
struct ThreadCtx {
    cx_ctx* ctx = nullptr;
    void* stream = nullptr;
    float* dev = nullptr;  // outputs: logits | hidden | final_query
    size_t cap = 0;
    ~ThreadCtx() = default;  // leaked at thread exit (the runtime may be gone)
};
thread_local ThreadCtx t_model;

ThreadCtx& model_ctx() {
    if (!t_model.ctx) {
        ck(cx_ctx_create(0, &t_model.ctx));
        int prio = 0;
        ck(cx_ctx_lane_stream(t_model.ctx, CX_LANE_STREAM, &t_model.stream, &prio));
    }
    return t_model;
}

}  // namespace

// ---- WeightStore (model.cpp:49-87) -------------------------------------------
WeightStore WeightStore::init(const ModelConfig& cfg) {
    cfg.validate();
    WeightStore w;
    w.cfg_ = cfg;
    Rng rng(cfg.seed);
    const size_t d = static_cast<size_t>(cfg.d_model), dff = static_cast<size_t>(cfg.d_ff());
    const size_t vocab = static_cast<size_t>(cfg.vocab_size);
    const double proj_std = 1.0 / std::sqrt(static_cast<double>(d));
    const double mlp_out_std = 1.0 / std::sqrt(static_cast<double>(dff));
    // draw order: embedding, per layer {attn_norm, wq, wk, wv, wo, mlp_norm, w_in, w_out},
    // final_norm, unembedding
    fill(rng, w.embedding_, vocab * d, 0.0, 1.0);
    w.layers_.resize(static_cast<size_t>(cfg.n_layers));
    for (auto& lw : w.layers_) {
        fill(rng, lw.attn_norm, d, 1.0, 0.02);
        fill(rng, lw.wq, d * d, 0.0, proj_std);
        fill(rng, lw.wk, d * d, 0.0, proj_std);
        fill(rng, lw.wv, d * d, 0.0, proj_std);
        fill(rng, lw.wo, d * d, 0.0, proj_std);
        fill(rng, lw.mlp_norm, d, 1.0, 0.02);
        fill(rng, lw.w_in, dff * d, 0.0, proj_std);
        fill(rng, lw.w_out, d * dff, 0.0, mlp_out_std);
    }
    fill(rng, w.final_norm_, d, 1.0, 0.02);
    fill(rng, w.unembedding_, vocab * d, 0.0, proj_std);
    const int64_t per_layer = static_cast<int64_t>(2 * d + 4 * d * d + dff * d + d * dff);
    w.parameter_count_ = static_cast<int64_t>(2 * vocab * d + d) + static_cast<int64_t>(cfg.n_layers) * per_layer;
    return w;
}

std::span<const float> WeightStore::embedding_row(int token) const {
    return {embedding_.data() + static_cast<size_t>(token) * static_cast<size_t>(cfg_.d_model),
            static_cast<size_t>(cfg_.d_model)};
}

cx_weights* WeightStore::device_handle() const {
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (!dev_) {
        // the flat array in the reference's draw order (cx_weights_flat_floats)
        std::vector<float> flat;
        flat.reserve(cx_weights_flat_floats(cfg_.n_layers, cfg_.d_model, cfg_.vocab_size));
        auto put = [&](const std::vector<float>& v) { flat.insert(flat.end(), v.begin(), v.end()); };
        put(embedding_);
        for (const auto& lw : layers_) {
            put(lw.attn_norm); put(lw.wq); put(lw.wk); put(lw.wv); put(lw.wo);
            put(lw.mlp_norm); put(lw.w_in); put(lw.w_out);
        }
        put(final_norm_);
        put(unembedding_);
        cx_weights* h = nullptr;
        ck(cx_weights_create(cfg_.n_layers, cfg_.n_heads, cfg_.d_model, cfg_.d_k, cfg_.vocab_size, cfg_.max_positions,
                             cfg_.rope_base, flat.data(), &h));
        dev_ = std::shared_ptr<cx_weights>(h, [](cx_weights* p) { cx_weights_destroy(p); });
    }
    return dev_.get();
}

// ---- forward_step (model.cpp:175-235) on the device ---------------------------
StepResult forward_step(const WeightStore& w, KvCache& cache, int token, int64_t position) {
    const ModelConfig& cfg = w.config();
    ThreadCtx& t = model_ctx();
    const size_t need = static_cast<size_t>(cfg.vocab_size + 2 * cfg.d_model);
    cx_weights* dw = w.device_handle();
    if (t.cap < need) {
        if (t.dev) cx_device_free(t.dev);
        t.dev = nullptr;
        ck(cx_device_alloc(need * sizeof(float), reinterpret_cast<void**>(&t.dev)));
        t.cap = need;
    }
    cx_kvcache* kc = cache.device_handle();
    ck(cx_forward_step_dev(t.ctx, dw, 1, &kc, &token, &position, t.dev, t.dev + cfg.vocab_size,
                           t.dev + cfg.vocab_size + cfg.d_model, t.stream));
    StepResult r;
    r.logits.resize(static_cast<size_t>(cfg.vocab_size));
    r.hidden_last.resize(static_cast<size_t>(cfg.d_model));
    r.final_query.resize(static_cast<size_t>(cfg.d_model));
    std::vector<float> host(need);
    ck(cx_device_read(host.data(), t.dev, need * sizeof(float), t.stream));
    std::copy(host.begin(), host.begin() + cfg.vocab_size, r.logits.begin());
    std::copy(host.begin() + cfg.vocab_size, host.begin() + cfg.vocab_size + cfg.d_model, r.hidden_last.begin());
    std::copy(host.begin() + cfg.vocab_size + cfg.d_model, host.end(), r.final_query.begin());
    return r;
}

std::vector<int> generate_greedy(const WeightStore& w, std::span<const int> prompt, int n_new) {
    if (prompt.empty()) throw precondition_error("empty prompt");
    KvCache cache(w.config());
    std::vector<int> out(prompt.begin(), prompt.end());
    int64_t pos = 0;
    StepResult last;
    for (int t : prompt) last = forward_step(w, cache, t, pos++);
    for (int i = 0; i < n_new; ++i) {
        const int t = kernels::argmax(last.logits);
        out.push_back(t);
        last = forward_step(w, cache, t, pos++);
    }
    return out;
}

std::vector<int> tokenize_bytes(std::string_view text) {
    std::vector<int> out;
    out.reserve(text.size());
    for (char c : text) out.push_back(static_cast<int>(static_cast<unsigned char>(c)));
    return out;
}

std::string detokenize_bytes(std::span<const int> tokens) {
    std::string out;
    out.reserve(tokens.size());
    for (int t : tokens) out.push_back(static_cast<char>(static_cast<unsigned char>(t)));
    return out;
}

// ---- encode_thought (injector.cpp:36-68): the device forward pass on a scratch cache
KvBlock encode_thought(const WeightStore& w, std::span<const int> thought_tokens, int64_t virtual_position_base) {
    if (thought_tokens.empty()) throw precondition_error("encode_thought: empty thought");
    const ModelConfig& cfg = w.config();
    if (virtual_position_base < 0 ||
        virtual_position_base + static_cast<int64_t>(thought_tokens.size()) > cfg.max_positions)
        throw capacity_error("encode_thought: virtual positions beyond max_positions");
    KvCache scratch(cfg);
    StepResult last;
    int64_t pos = virtual_position_base;
    for (int t : thought_tokens) last = forward_step(w, scratch, t, pos++);
    KvBlock block;
    block.base_position = virtual_position_base;
    block.token_count = static_cast<int64_t>(thought_tokens.size());
    block.n_layers = cfg.n_layers;
    block.d_model = cfg.d_model;
    for (int l = 0; l < cfg.n_layers; ++l) {
        auto lk = scratch.layer_keys(l);
        auto lv = scratch.layer_values(l);
        block.keys.insert(block.keys.end(), lk.begin(), lk.end());
        block.values.insert(block.values.end(), lv.begin(), lv.end());
    }
    block.last_hidden = last.hidden_last;
    return block;
}

// ---- kernels.hpp projections (kernels.cpp:12-62) on the device ----------------
namespace kernels {
void matvec(std::span<const float> w, int n_out, int n_in, std::span<const float> x, std::span<float> y) {
    ck(cx_matvec(w.data(), n_out, n_in, x.data(), y.data()));
}
void rmsnorm(std::span<const float> x, std::span<const float> gain, std::span<float> out, double eps) {
    ck(cx_rmsnorm(x.data(), gain.data(), static_cast<int64_t>(x.size()), eps, out.data()));
}
void add_inplace(std::span<float> x, std::span<const float> y) {
    ck(cx_elementwise(x.data(), y.data(), static_cast<int64_t>(x.size()), 0));
}
void relu_inplace(std::span<float> x) { ck(cx_elementwise(x.data(), nullptr, static_cast<int64_t>(x.size()), 1)); }
void apply_rope(std::span<float> v, int64_t position, double rope_base) {
    ck(cx_apply_rope(v.data(), static_cast<int64_t>(v.size()), position, rope_base));
}
}  // namespace kernels

}  // namespace cortex

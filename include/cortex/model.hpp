// cortex/model.hpp -- B200 drop-in for proj/include/cortex/model.hpp (Origin,
// LayerWeights, WeightStore, KvCache, StepResult, forward_step, generate_greedy,
// the byte tokenizer).  KvCache storage lives in HBM (cx_kvcache,
// [n_layers][capacity][d_model] fp32); key()/value()/layer_keys() return spans
// over a host mirror that is kept in step with host-side appends and re-synced
// from the device after device-side appends.  WeightStore keeps the reference's
// host vectors (same seeded draw order) plus a device copy created on first use;
// forward_step runs on the device (cx_forward_step_dev).
#pragma once

#include "cortex/config.hpp"

#include <cstdint>
#include <memory>
#include <span>
#include <string>
#include <string_view>
#include <vector>

struct cx_kvcache;
struct cx_weights;

namespace cortex {

enum class Origin : uint8_t { context, injected };

struct LayerWeights {
    std::vector<float> attn_norm;       // d_model
    std::vector<float> wq, wk, wv, wo;  // d_model x d_model, row-major
    std::vector<float> mlp_norm;        // d_model
    std::vector<float> w_in;            // d_ff x d_model
    std::vector<float> w_out;           // d_model x d_ff
};

class WeightStore {
public:
    static WeightStore init(const ModelConfig& cfg);

    const ModelConfig& config() const { return cfg_; }
    const LayerWeights& layer(int l) const { return layers_[static_cast<size_t>(l)]; }
    std::span<const float> embedding_row(int token) const;
    const std::vector<float>& final_norm() const { return final_norm_; }
    const std::vector<float>& unembedding() const { return unembedding_; }

    int64_t parameter_count() const { return parameter_count_; }
    int64_t total_bytes() const { return parameter_count_ * 4; }

    // ---- B200 extension: the device copy (created on first use, shared by copies)
    cx_weights* device_handle() const;

private:
    WeightStore() = default;

    ModelConfig cfg_;
    std::vector<float> embedding_;
    std::vector<LayerWeights> layers_;
    std::vector<float> final_norm_;
    std::vector<float> unembedding_;
    int64_t parameter_count_ = 0;
    mutable std::shared_ptr<cx_weights> dev_;
};

class KvCache {
public:
    explicit KvCache(const ModelConfig& cfg);
    ~KvCache();
    KvCache(KvCache&& o) noexcept;
    KvCache& operator=(KvCache&& o) noexcept;
    KvCache(const KvCache& o);             // deep copy on the device (cx_kvcache_clone)
    KvCache& operator=(const KvCache& o);

    const ModelConfig& config() const { return cfg_; }
    int64_t size() const;
    int64_t position(int64_t i) const;
    Origin origin(int64_t i) const;
    int64_t last_context_position() const;
    int64_t context_count() const;

    std::span<const float> key(int layer, int64_t i) const;
    std::span<const float> value(int layer, int64_t i) const;
    std::span<const float> layer_keys(int layer) const;
    std::span<const float> layer_values(int layer) const;

    int64_t kv_bytes() const;
    static int64_t entry_bytes(const ModelConfig& cfg);

    bool entry_open() const;

    void begin_entry(int64_t position, Origin origin);
    void write_layer(int layer, std::span<const float> key, std::span<const float> value);
    void end_entry();
    void append_entry(int64_t position, Origin origin, std::span<const float> keys,
                      std::span<const float> values);

    // ---- B200 extensions -------------------------------------------------
    cx_kvcache* device_handle() const { return h_; }
    // Call after appending through the device API so spans re-sync.
    void invalidate_host_mirror() const { mirror_rows_ = 0; }

private:
    void sync_mirror() const;

    ModelConfig cfg_;
    cx_kvcache* h_ = nullptr;
    mutable std::vector<std::vector<float>> hk_, hv_;  // per layer, rows [0, mirror_rows_)
    mutable int64_t mirror_rows_ = 0;
    std::vector<int> layer_rows_;  // rows mirrored per layer while an entry is open
};

struct StepResult {
    std::vector<float> logits;       // vocab_size
    std::vector<float> hidden_last;  // d_model, after the final norm
    std::vector<float> final_query;  // d_model, final-layer post-RoPE query
};

StepResult forward_step(const WeightStore& w, KvCache& cache, int token, int64_t position);

std::vector<int> generate_greedy(const WeightStore& w, std::span<const int> prompt, int n_new);

std::vector<int> tokenize_bytes(std::string_view text);
std::string detokenize_bytes(std::span<const int> tokens);

}  // namespace cortex

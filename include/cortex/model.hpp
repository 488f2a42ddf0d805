// cortex/model.hpp -- B200 drop-in for the KvCache part of
// proj/include/cortex/model.hpp:16,67-113.  Storage lives in HBM (cx_kvcache,
// [n_layers][capacity][d_model] fp32); key()/value()/layer_keys() return spans
// over a host mirror that is kept in step with host-side appends and re-synced
// from the device after device-side appends (inject_dev, decode appends).
// WeightStore / forward_step (dense model compute) are out of scope
// (SURVEY.md §8(f) "next").
#pragma once

#include "cortex/config.hpp"

#include <cstdint>
#include <span>
#include <vector>

struct cx_kvcache;

namespace cortex {

enum class Origin : uint8_t { context, injected };

class KvCache {
public:
    explicit KvCache(const ModelConfig& cfg);
    ~KvCache();
    KvCache(KvCache&& o) noexcept;
    KvCache& operator=(KvCache&& o) noexcept;
    KvCache(const KvCache&) = delete;
    KvCache& operator=(const KvCache&) = delete;

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

}  // namespace cortex

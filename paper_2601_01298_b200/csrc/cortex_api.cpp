// cortex_api.cpp -- the C++ cortex:: drop-in shim (include/cortex/*.hpp) over
// the C-ABI (include/cortex_b200.h).  Code written against the reference's
// synapse / KvCache / inject / attend / gate API links against libcortex_b200.so
// unchanged; every compute call runs the sm_100a kernels.  cx_status codes are
// rethrown as the reference's exception types (errors.hpp).
#include "cortex/config.hpp"
#include "cortex/errors.hpp"
#include "cortex/gate.hpp"
#include "cortex/injector.hpp"
#include "cortex/kernels.hpp"
#include "cortex/model.hpp"
#include "cortex/synapse.hpp"
#include "cortex_b200.h"

#include <charconv>
#include <cmath>
#include <limits>
#include <sstream>
#include <unordered_map>

namespace cortex {

namespace {

void throw_status(cx_status st) {
    const std::string msg = cx_last_error();
    switch (st) {
        case CX_OK: return;
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

inline void ck(cx_status st) {
    if (st != CX_OK) throw_status(st);
}

// nlohmann::json's number format: shortest round-trip, integral values keep ".0".
std::string json_double(double v) {
    if (!std::isfinite(v)) return "null";
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof(buf), v);
    std::string s(buf, r.ptr);
    if (s.find_first_of(".eE") == std::string::npos) s += ".0";
    return s;
}

}  // namespace

// ---- config.hpp (model.cpp:12-35) ------------------------------------------
void ModelConfig::validate() const {
    if (n_layers < 1 || n_heads < 1 || d_model < 1 || d_k < 1) throw config_error("model dimensions must be positive");
    if (n_heads * d_k != d_model) throw config_error("d_model must equal n_heads * d_k exactly");
    if (d_k % 2 != 0) throw config_error("d_k must be even for pairwise rotation");
    if (vocab_size < 1) throw config_error("vocab_size must be positive");
    if (max_positions < 1) throw config_error("max_positions must be positive");
    if (!(rope_base > 0.0)) throw config_error("rope_base must be positive");
}

void RuntimeConfig::validate(const ModelConfig& mc) const {
    if (k < 1) throw config_error("k must be >= 1");
    if (lambda < 0.0 || lambda > 1.0) throw config_error("lambda must be in [0,1]");
    if (theta < -1.0 || theta > 1.0) throw config_error("theta must be in [-1,1]");
    if (max_stream_agents < 0) throw config_error("max_stream_agents must be >= 0");
    if (thought_budget < 1) throw config_error("thought_budget must be >= 1");
    if (synapse_push_period < 1) throw config_error("synapse_push_period must be >= 1");
    if (river_budget < 0) throw config_error("river_budget must be >= 0");
    const int64_t base = virtual_base(mc);
    if (base < 1 || base >= mc.max_positions) throw config_error("reserved virtual base out of range");
}

// ---- KvCache (model.hpp) ---------------------------------------------------
KvCache::KvCache(const ModelConfig& cfg) : cfg_(cfg) {
    cfg.validate();
    ck(cx_kvcache_create(cfg.n_layers, cfg.n_heads, cfg.d_model, cfg.d_k, cfg.max_positions, 64, &h_));
    hk_.resize(static_cast<size_t>(cfg.n_layers));
    hv_.resize(static_cast<size_t>(cfg.n_layers));
}

KvCache::~KvCache() {
    if (h_) cx_kvcache_destroy(h_);
}

KvCache::KvCache(KvCache&& o) noexcept
    : cfg_(o.cfg_), h_(o.h_), hk_(std::move(o.hk_)), hv_(std::move(o.hv_)), mirror_rows_(o.mirror_rows_),
      layer_rows_(std::move(o.layer_rows_)) {
    o.h_ = nullptr;
}

KvCache::KvCache(const KvCache& o)
    : cfg_(o.cfg_), hk_(o.hk_), hv_(o.hv_), mirror_rows_(o.mirror_rows_), layer_rows_(o.layer_rows_) {
    ck(cx_kvcache_clone(o.h_, &h_));
}

KvCache& KvCache::operator=(const KvCache& o) {
    if (this != &o) {
        KvCache tmp(o);
        *this = std::move(tmp);
    }
    return *this;
}

KvCache& KvCache::operator=(KvCache&& o) noexcept {
    if (this != &o) {
        if (h_) cx_kvcache_destroy(h_);
        cfg_ = o.cfg_;
        h_ = o.h_;
        hk_ = std::move(o.hk_);
        hv_ = std::move(o.hv_);
        mirror_rows_ = o.mirror_rows_;
        layer_rows_ = std::move(o.layer_rows_);
        o.h_ = nullptr;
    }
    return *this;
}

int64_t KvCache::size() const { return cx_kvcache_size(h_); }
int64_t KvCache::position(int64_t i) const { return cx_kvcache_positions_host(h_)[i]; }
Origin KvCache::origin(int64_t i) const { return static_cast<Origin>(cx_kvcache_origins_host(h_)[i]); }
int64_t KvCache::last_context_position() const { return cx_kvcache_last_context_position(h_); }
int64_t KvCache::context_count() const { return cx_kvcache_context_count(h_); }
bool KvCache::entry_open() const { return cx_kvcache_entry_open(h_) != 0; }
int64_t KvCache::entry_bytes(const ModelConfig& cfg) { return static_cast<int64_t>(cfg.n_layers) * 2 * cfg.d_model * 4; }
int64_t KvCache::kv_bytes() const { return size() * entry_bytes(cfg_); }

void KvCache::sync_mirror() const {
    // rows appended through the host API are mirrored eagerly; anything else
    // (device-side appends) is read back here.
    if (entry_open()) return;  // mid-entry: per-layer rows are already mirrored
    const int64_t n = size();
    if (mirror_rows_ >= n) return;
    const size_t d = static_cast<size_t>(cfg_.d_model);
    for (int l = 0; l < cfg_.n_layers; ++l) {
        auto& k = hk_[static_cast<size_t>(l)];
        auto& v = hv_[static_cast<size_t>(l)];
        k.resize(static_cast<size_t>(n) * d);
        v.resize(static_cast<size_t>(n) * d);
        ck(cx_kvcache_read(h_, l, mirror_rows_, n - mirror_rows_, k.data() + mirror_rows_ * d,
                           v.data() + mirror_rows_ * d));
    }
    mirror_rows_ = n;
}

std::span<const float> KvCache::key(int layer, int64_t i) const {
    sync_mirror();
    const auto& k = hk_[static_cast<size_t>(layer)];
    return {k.data() + static_cast<size_t>(i) * cfg_.d_model, static_cast<size_t>(cfg_.d_model)};
}

std::span<const float> KvCache::value(int layer, int64_t i) const {
    sync_mirror();
    const auto& v = hv_[static_cast<size_t>(layer)];
    return {v.data() + static_cast<size_t>(i) * cfg_.d_model, static_cast<size_t>(cfg_.d_model)};
}

std::span<const float> KvCache::layer_keys(int layer) const {
    sync_mirror();
    const auto& k = hk_[static_cast<size_t>(layer)];
    return {k.data(), k.size()};
}

std::span<const float> KvCache::layer_values(int layer) const {
    sync_mirror();
    const auto& v = hv_[static_cast<size_t>(layer)];
    return {v.data(), v.size()};
}

void KvCache::begin_entry(int64_t position, Origin origin) {
    sync_mirror();
    ck(cx_kvcache_begin_entry(h_, position, static_cast<cx_origin>(origin)));
}

void KvCache::write_layer(int layer, std::span<const float> key, std::span<const float> value) {
    if (key.size() != value.size()) throw precondition_error("write_layer: key/value width mismatch");
    ck(cx_kvcache_write_layer(h_, layer, key.data(), value.data(), static_cast<int64_t>(key.size())));
    auto& k = hk_[static_cast<size_t>(layer)];
    auto& v = hv_[static_cast<size_t>(layer)];
    k.insert(k.end(), key.begin(), key.end());
    v.insert(v.end(), value.begin(), value.end());
    if (layer == cfg_.n_layers - 1) mirror_rows_ = size();
}

void KvCache::end_entry() { ck(cx_kvcache_end_entry(h_)); }

void KvCache::append_entry(int64_t position, Origin origin, std::span<const float> keys,
                           std::span<const float> values) {
    const size_t d = static_cast<size_t>(cfg_.d_model);
    if (keys.size() != d * cfg_.n_layers || values.size() != d * cfg_.n_layers)
        throw precondition_error("append_entry: keys/values must hold n_layers * d_model floats");
    sync_mirror();
    ck(cx_kvcache_append_entry(h_, position, static_cast<cx_origin>(origin), keys.data(), values.data()));
    for (int l = 0; l < cfg_.n_layers; ++l) {
        auto& k = hk_[static_cast<size_t>(l)];
        auto& v = hv_[static_cast<size_t>(l)];
        k.insert(k.end(), keys.begin() + l * d, keys.begin() + (l + 1) * d);
        v.insert(v.end(), values.begin() + l * d, values.begin() + (l + 1) * d);
    }
    mirror_rows_ = size();
}

// ---- synapse.hpp -------------------------------------------------------------
ContextCloud context_key_cloud(const KvCache& cache, int layer) {
    const ModelConfig& cfg = cache.config();
    ContextCloud out;
    out.cloud.dim = cfg.d_model;
    for (int64_t i = 0; i < cache.size(); ++i) {
        if (cache.origin(i) != Origin::context) continue;
        auto key = cache.key(layer, i);
        out.cloud.data.insert(out.cloud.data.end(), key.begin(), key.end());
        out.entry_index.push_back(i);
        out.positions.push_back(cache.position(i));
        ++out.cloud.count;
    }
    return out;
}

std::vector<double> attention_scores_points(const PointCloud& keys, std::span<const float> query, int n_heads) {
    std::vector<double> out(static_cast<size_t>(keys.count));
    ck(cx_attention_scores_points(keys.data.data(), keys.count, keys.dim, query.data(),
                                  static_cast<int64_t>(query.size()), n_heads, out.data()));
    return out;
}

std::vector<double> attention_scores(const KvCache& cache, std::span<const float> query, int layer) {
    auto ctx = context_key_cloud(cache, layer);
    if (ctx.cloud.count == 0) throw precondition_error("attention_scores: cache has no context entries");
    return attention_scores_points(ctx.cloud, query, cache.config().n_heads);
}

std::vector<double> coverage_scores_points(const PointCloud& cloud, std::span<const int64_t> selected) {
    std::vector<double> out(static_cast<size_t>(cloud.count), 0.0);
    ck(cx_coverage_scores_points(cloud.data.data(), cloud.count, cloud.dim, selected.data(),
                                 static_cast<int64_t>(selected.size()), out.data()));
    return out;
}

std::vector<double> coverage_scores(const KvCache& cache, std::span<const int64_t> selected_positions, int layer) {
    auto ctx = context_key_cloud(cache, layer);
    std::unordered_map<int64_t, int64_t> row_of;
    for (int64_t r = 0; r < ctx.cloud.count; ++r) row_of[ctx.positions[static_cast<size_t>(r)]] = r;
    std::vector<int64_t> rows;
    rows.reserve(selected_positions.size());
    for (int64_t p : selected_positions) {
        auto it = row_of.find(p);
        if (it == row_of.end()) throw precondition_error("coverage_scores: position is not a context entry");
        rows.push_back(it->second);
    }
    return coverage_scores_points(ctx.cloud, rows);
}

double hausdorff_distance(const PointCloud& cloud, const PointCloud& landmarks) {
    double out = 0.0;
    ck(cx_hausdorff_distance(cloud.data.data(), cloud.count, cloud.dim, landmarks.data.data(), landmarks.count,
                             landmarks.dim, &out));
    return out;
}

double hausdorff_to_subset(const PointCloud& cloud, std::span<const int64_t> rows) {
    double out = 0.0;
    ck(cx_hausdorff_to_subset(cloud.data.data(), cloud.count, cloud.dim, rows.data(), static_cast<int64_t>(rows.size()),
                              &out));
    return out;
}

double mean_pairwise_reduction(const PointCloud& cloud, const PointCloud& landmarks) {
    double out = 0.0;
    ck(cx_mean_pairwise_reduction(cloud.data.data(), cloud.count, cloud.dim, landmarks.data.data(), landmarks.count,
                                  landmarks.dim, &out));
    return out;
}

double mean_pairwise_reduction_subset(const PointCloud& cloud, std::span<const int64_t> rows) {
    double out = 0.0;
    ck(cx_mean_pairwise_reduction_subset(cloud.data.data(), cloud.count, cloud.dim, rows.data(),
                                         static_cast<int64_t>(rows.size()), &out));
    return out;
}

SelectionResult select_landmarks_points(const PointCloud& cloud, std::span<const double> attention, int k,
                                        double lambda) {
    const int64_t cap = std::max<int64_t>(0, std::min<int64_t>(k, cloud.count));
    SelectionResult r;
    r.indices.resize(static_cast<size_t>(cap));
    r.scores.resize(static_cast<size_t>(cap));
    int64_t n = 0;
    ck(cx_select_landmarks_points(cloud.data.data(), cloud.count, cloud.dim, attention.data(),
                                  static_cast<int64_t>(attention.size()), k, lambda, r.indices.data(), r.scores.data(),
                                  &n));
    r.indices.resize(static_cast<size_t>(n));
    r.scores.resize(static_cast<size_t>(n));
    return r;
}

SynapseSnapshot select_landmarks(const KvCache& cache, std::span<const float> query, int k, double lambda) {
    cx_snapshot* h = nullptr;
    ck(cx_select_landmarks(cache.device_handle(), query.data(), static_cast<int64_t>(query.size()), k, lambda, &h));
    SynapseSnapshot snap;
    snap.device = std::shared_ptr<const cx_snapshot>(h, [](const cx_snapshot* p) { cx_snapshot_release(p); });
    snap.source_length = cx_snapshot_source_length(h);
    snap.k_configured = cx_snapshot_k_configured(h);
    snap.n_layers = cx_snapshot_n_layers(h);
    snap.d_model = cx_snapshot_d_model(h);
    const int64_t n = cx_snapshot_count(h);
    if (n > 0) {
        const size_t per = static_cast<size_t>(snap.n_layers) * snap.d_model;
        std::vector<int64_t> pos(static_cast<size_t>(n));
        std::vector<double> sc(static_cast<size_t>(n));
        std::vector<float> ks(static_cast<size_t>(n) * per), vs(ks.size());
        ck(cx_snapshot_read(h, pos.data(), sc.data(), ks.data(), vs.data()));
        snap.landmarks.resize(static_cast<size_t>(n));
        for (int64_t s = 0; s < n; ++s) {
            auto& lm = snap.landmarks[static_cast<size_t>(s)];
            lm.source_position = pos[static_cast<size_t>(s)];
            lm.hybrid_score = sc[static_cast<size_t>(s)];
            lm.keys.assign(ks.begin() + s * per, ks.begin() + (s + 1) * per);
            lm.values.assign(vs.begin() + s * per, vs.begin() + (s + 1) * per);
        }
    }
    return snap;
}

std::string SynapseSnapshot::to_json() const {
    // synapse.cpp:322-335: nlohmann object (sorted keys), compact dump
    std::ostringstream os;
    os << "{\"hybrid_scores\":[";
    for (size_t i = 0; i < landmarks.size(); ++i) os << (i ? "," : "") << json_double(landmarks[i].hybrid_score);
    os << "],\"positions\":[";
    for (size_t i = 0; i < landmarks.size(); ++i) os << (i ? "," : "") << landmarks[i].source_position;
    os << "],\"source_length\":" << source_length << ",\"version\":" << version << "}";
    return os.str();
}

// SynapseBuffer (synapse.cpp:337-362): version-stamped latest-value slot.
// Snapshots are immutable after push; the device K/V travel inside them.
uint64_t SynapseBuffer::push(SynapseSnapshot snap) {
    auto owned = std::make_shared<SynapseSnapshot>(std::move(snap));
    std::lock_guard<std::mutex> lk(mu_);
    owned->version = ++version_;
    latest_ = std::move(owned);
    cv_.notify_all();
    return version_;
}

std::shared_ptr<const SynapseSnapshot> SynapseBuffer::read_latest() const {
    std::lock_guard<std::mutex> lk(mu_);
    return latest_;
}

std::shared_ptr<const SynapseSnapshot> SynapseBuffer::wait_nonempty(std::chrono::milliseconds timeout) const {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait_for(lk, timeout, [&] { return latest_ != nullptr || shutdown_; });
    return latest_;
}

void SynapseBuffer::shutdown() {
    std::lock_guard<std::mutex> lk(mu_);
    shutdown_ = true;
    cv_.notify_all();
}

// ---- kernels.hpp ---------------------------------------------------------------
namespace kernels {
std::vector<double> softmax(std::span<const double> scores) {
    std::vector<double> out(scores.size());
    ck(cx_softmax(scores.data(), static_cast<int64_t>(scores.size()), out.data()));
    return out;
}

std::vector<double> softmax(std::span<const float> scores) {
    std::vector<double> out(scores.size());
    ck(cx_softmax_f32(scores.data(), static_cast<int64_t>(scores.size()), out.data()));
    return out;
}

int argmax(std::span<const float> v) {
    int out = 0;
    ck(cx_argmax(v.data(), static_cast<int64_t>(v.size()), &out));
    return out;
}

void attend(std::span<const float> q, std::span<const float> keys, std::span<const float> values, int64_t n_entries,
            int n_heads, int d_k, std::span<float> out) {
    ck(cx_attend(q.data(), keys.data(), values.data(), n_entries, n_heads, d_k, out.data()));
}
}  // namespace kernels

// ---- injector.hpp --------------------------------------------------------------
std::span<const float> KvBlock::key(int layer, int64_t t) const {
    const size_t d = static_cast<size_t>(d_model);
    return {keys.data() + (static_cast<size_t>(layer) * static_cast<size_t>(token_count) + static_cast<size_t>(t)) * d,
            d};
}

std::span<const float> KvBlock::value(int layer, int64_t t) const {
    const size_t d = static_cast<size_t>(d_model);
    return {values.data() + (static_cast<size_t>(layer) * static_cast<size_t>(token_count) + static_cast<size_t>(t)) * d,
            d};
}

std::string InjectionRecord::csv_header() {
    return "thought_id,token_count,virtual_position_base,applied_at_stream_position";
}

std::string InjectionRecord::csv_row() const {
    std::ostringstream os;
    os << thought_id << ',' << token_count << ',' << virtual_position_base << ',' << applied_at_stream_position;
    return os.str();
}

InjectionRecord inject(KvCache& river_cache, const KvBlock& block, int64_t thought_id, int64_t stream_position) {
    cx_injection_record r{};
    const cx_status st = cx_inject_host(river_cache.device_handle(), block.keys.data(), block.values.data(),
                                        block.base_position, block.token_count, block.n_layers, block.d_model,
                                        thought_id, stream_position, &r);
    river_cache.invalidate_host_mirror();  // rows appended on the device (also on a partial append)
    ck(st);
    InjectionRecord rec;
    rec.thought_id = r.thought_id;
    rec.token_count = r.token_count;
    rec.virtual_position_base = r.virtual_position_base;
    rec.applied_at_stream_position = r.applied_at_stream_position;
    return rec;
}

VirtualPositionPlanner::VirtualPositionPlanner(int64_t reserved_start, int64_t max_positions)
    : start_(reserved_start), limit_(max_positions) {
    if (reserved_start < 0 || reserved_start >= max_positions)
        throw config_error("planner: reserved_start out of range");
}

int64_t VirtualPositionPlanner::reserve(int64_t token_count) {
    if (token_count < 1) throw precondition_error("planner: token_count must be >= 1");
    const int64_t base = start_ + taken_;
    if (base + token_count > limit_) throw capacity_error("planner: reserved virtual range exhausted");
    taken_ += token_count;
    return base;
}

// ---- gate.cpp:12-61 -------------------------------------------------------
std::string GateDecision::csv_header() { return "thought_id,score,theta,accepted"; }

std::string GateDecision::csv_row() const {  // gate.cpp:14-25 (precision 17, "nan" when degenerate)
    std::ostringstream os;
    os.precision(17);
    os << thought_id << ',';
    if (degenerate)
        os << "nan";
    else
        os << score;
    os << ',' << threshold << ',' << (accepted ? 1 : 0);
    return os.str();
}

double gate_score(std::span<const float> h_main, std::span<const float> t_side) {
    if (h_main.size() != t_side.size()) throw precondition_error("gate_score: width mismatch");
    double s = 0.0;
    ck(cx_gate_score(h_main.data(), t_side.data(), (int64_t)h_main.size(), &s));
    return s;
}

GateDecision decide(std::span<const float> h_main, std::span<const float> t_side, double theta, int64_t thought_id) {
    if (theta < -1.0 || theta > 1.0) throw precondition_error("decide: theta must be in [-1,1]");
    GateDecision d;
    d.threshold = theta;
    d.thought_id = thought_id;
    try {
        d.score = gate_score(h_main, t_side);
        d.accepted = d.score >= theta;
    } catch (const degenerate_input_error&) {
        d.score = std::numeric_limits<double>::quiet_NaN();
        d.degenerate = true;
        d.accepted = false;
    }
    return d;
}

}  // namespace cortex

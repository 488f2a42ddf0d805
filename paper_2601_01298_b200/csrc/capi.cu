// capi.cu -- the extern "C" boundary (include/cortex_b200.h).
//
// Validation mirrors the reference's checks and their ORDER (each is cited),
// happens before any device work, and maps each reference exception type onto
// its cx_status.  The reference-shaped calls take host pointers and are
// synchronous (H2D -> sm_100a kernels -> D2H on the calling thread's context
// stream); the *_dev calls are stream-ordered and never synchronize.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <map>
#include <memory>

#include "cx_internal.cuh"

namespace cx {

std::atomic<uint64_t> g_launches{0};
static thread_local std::string t_last_error;
void set_last_error(const std::string& m) { t_last_error = m; }

void kernel_smem_attr(const void* fn, size_t bytes, bool nonportable_cluster) {
    struct Key {
        const void* fn;
        int dev;
        bool operator<(const Key& o) const { return fn != o.fn ? fn < o.fn : dev < o.dev; }
    };
    struct Set {
        size_t bytes = 0;
        bool nonportable = false;
    };
    static std::mutex mu;
    static std::map<Key, Set> done;  // attributes already set per (kernel, device)
    int dev = 0;
    CX_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    Set& st = done[{fn, dev}];
    if (st.bytes < bytes) {
        CX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        st.bytes = bytes;
    }
    if (nonportable_cluster && !st.nonportable) {
        CX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        st.nonportable = true;
    }
}

namespace {

void require_device() {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        fail(CX_DEVICE_ERROR, "no CUDA device: the B200 path has no CPU fallback");
}

void ctx_init(cx_ctx* c, int device) {
    require_device();
    c->device = device;
    CX_CUDA(cudaSetDevice(device));
    int lo = 0, hi = 0;
    CX_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CX_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CX_CUDA(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    // priority lanes: lo is the least urgent value, hi the most (numerically smaller)
    c->lane_prio[CX_LANE_RIVER] = hi;
    c->lane_prio[CX_LANE_STREAM] = (lo + hi) / 2 == hi && lo != hi ? hi + 1 : (lo + hi) / 2;
    CX_CUDA(cudaStreamCreateWithPriority(&c->lane[CX_LANE_RIVER], cudaStreamNonBlocking, c->lane_prio[CX_LANE_RIVER]));
    CX_CUDA(cudaStreamCreateWithPriority(&c->lane[CX_LANE_STREAM], cudaStreamNonBlocking, c->lane_prio[CX_LANE_STREAM]));
    CX_CUDA(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
    CX_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CX_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    CX_CUDA(cudaMalloc(&c->d_flag, sizeof(int)));
    CX_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
}

struct CtxHolder {
    cx_ctx* ctx = nullptr;
    ~CtxHolder() {
        // contexts are intentionally leaked at thread exit: the CUDA runtime may
        // already be torn down during process exit.
    }
};
thread_local CtxHolder t_ctx;

}  // namespace

cx_ctx* default_ctx() {
    if (!t_ctx.ctx) {
        int dev = 0;
        require_device();
        CX_CUDA(cudaGetDevice(&dev));
        auto* c = new cx_ctx();
        ctx_init(c, dev);
        t_ctx.ctx = c;
    }
    return t_ctx.ctx;
}

// ---- small helpers -----------------------------------------------------------

static void h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes) CX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
}
static void d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes) CX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
}

static void check_flag_and_sync(cx_ctx* c) {
    int flag = 0;
    CX_CUDA(cudaMemcpyAsync(&flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CX_CUDA(cudaStreamSynchronize(c->stream));
    if (flag & FLAG_NONFINITE) fail(CX_PRECONDITION_ERROR, "softmax: non-finite input");
}

static GroupView single_group(const float* d_cloud, int64_t count, int dim) {
    GroupView g{};
    g.G = 1;
    g.L = count;
    g.dim = dim;
    g.X = d_cloud;
    g.gstride = count * dim;
    g.rstride = dim;
    return g;
}

static GroupView view_of(const cx_groups* gr) {
    GroupView g{};
    g.G = gr->n_groups;
    g.L = gr->count;
    g.dim = gr->dim;
    g.X = gr->clouds;
    g.gstride = gr->group_stride;
    g.rstride = gr->row_stride;
    g.Q = gr->queries;
    g.P = gr->n_pass;
    g.d_k = gr->d_k;
    g.col_step = gr->col_step;
    return g;
}

static void validate_groups(const cx_groups* gr, bool need_queries) {
    if (!gr) fail(CX_INVALID_ARGUMENT, "null cx_groups");
    if (gr->n_groups < 0 || gr->count < 0 || gr->dim < 1) fail(CX_INVALID_ARGUMENT, "bad group shape");
    if (gr->count > 0 && gr->n_groups > 0 && !gr->clouds) fail(CX_INVALID_ARGUMENT, "null clouds");
    if (need_queries) {
        // attention_scores_points checks (synapse.cpp:66-70), per group
        if (gr->count == 0) fail(CX_PRECONDITION_ERROR, "attention_scores: empty candidate set");
        if (gr->n_pass < 1 || gr->d_k < 1) fail(CX_PRECONDITION_ERROR, "attention_scores: bad head count");
        if ((int64_t)(gr->n_pass - 1) * gr->col_step + gr->d_k > gr->dim)
            fail(CX_PRECONDITION_ERROR, "attention_scores: query width mismatch");
        if (!gr->queries) fail(CX_INVALID_ARGUMENT, "null queries");
    }
}

}  // namespace cx

using namespace cx;

// ============================================================================
// misc
// ============================================================================
extern "C" int cx_abi_version(void) { return CX_ABI_VERSION; }
extern "C" const char* cx_last_error(void) { return t_last_error.c_str(); }
extern "C" uint64_t cx_kernel_launch_count(void) { return g_launches.load(); }

extern "C" cx_status cx_ctx_create(int device, cx_ctx** out) {
    return guard(__func__, [&] {
        if (!out) fail(CX_INVALID_ARGUMENT, "null out");
        auto* c = new cx_ctx();
        try {
            ctx_init(c, device);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

extern "C" cx_status cx_ctx_destroy(cx_ctx* c) {
    return guard(__func__, [&] {
        if (!c) return;
        cudaStreamSynchronize(c->stream);
        cudaStreamSynchronize(c->side);
        if (c->arena.base) cudaFree(c->arena.base);
        if (c->fw_counters) cudaFree(c->fw_counters);
        for (auto& fg : c->fw_graphs) cudaGraphExecDestroy(fg.exec);
        for (cudaEvent_t e : c->fw_ev)
            if (e) cudaEventDestroy(e);
        if (c->fw_dev) cudaFree(c->fw_dev);
        if (c->fw_host) cudaFreeHost(c->fw_host);
        if (c->d_flag) cudaFree(c->d_flag);
        if (c->gaps) cudaFree(c->gaps);
        cudaEventDestroy(c->ev_fork);
        cudaEventDestroy(c->ev_join);
        cudaStreamSynchronize(c->copy);
        cudaStreamDestroy(c->copy);
        for (cudaEvent_t e : c->hev) cudaEventDestroy(e);
        for (cudaEvent_t e : c->pev) cudaEventDestroy(e);
        if (c->aux) cx_ctx_destroy(c->aux);
        if (c->hbuf) cudaFree(c->hbuf);
        for (cudaStream_t& l : c->lane) {
            cudaStreamSynchronize(l);
            cudaStreamDestroy(l);
        }
        cudaStreamDestroy(c->side);
        cudaStreamDestroy(c->stream);
        delete c;
    });
}

extern "C" cx_status cx_ctx_lane_stream(cx_ctx* c, int lane, void** stream, int* priority) {
    return guard(__func__, [&] {
        if (!c || !stream) fail(CX_INVALID_ARGUMENT, "null pointer");
        if (lane != CX_LANE_RIVER && lane != CX_LANE_STREAM) fail(CX_INVALID_ARGUMENT, "unknown lane");
        *stream = (void*)c->lane[lane];
        if (priority) *priority = c->lane_prio[lane];
    });
}

// ============================================================================
// point-level, reference-shaped (host pointers)
// ============================================================================
extern "C" cx_status cx_attention_scores_points(const float* keys, int64_t count, int dim, const float* query,
                                                int64_t query_len, int n_heads, double* out) {
    return guard(__func__, [&] {
        // synapse.cpp:66-70, in order
        if (count == 0) fail(CX_PRECONDITION_ERROR, "attention_scores: empty candidate set");
        if (query_len != (int64_t)dim) fail(CX_PRECONDITION_ERROR, "attention_scores: query width mismatch");
        if (n_heads < 1 || dim % n_heads != 0) fail(CX_PRECONDITION_ERROR, "attention_scores: bad head count");
        if (count < 0 || !keys || !query || !out) fail(CX_INVALID_ARGUMENT, "null pointer / negative count");
        cx_ctx* c = default_ctx();
        std::lock_guard<std::mutex> lk(c->mu);
        GroupView g = single_group(nullptr, count, dim);
        g.P = n_heads;
        g.d_k = dim / n_heads;
        g.col_step = g.d_k;
        ArenaPlan pl;
        pl.take<float>((size_t)count * dim);
        pl.take<float>((size_t)dim);
        pl.take<double>((size_t)count);
        plan_attention(pl, g);
        c->arena.reserve(pl.used);
        c->arena.reset();
        float* dk = c->arena.take<float>((size_t)count * dim);
        float* dq = c->arena.take<float>((size_t)dim);
        double* dout = c->arena.take<double>((size_t)count);
        g.X = dk;
        g.Q = dq;
        CX_CUDA(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
        h2d(dk, keys, sizeof(float) * count * dim, c->stream);
        h2d(dq, query, sizeof(float) * dim, c->stream);
        attention_grouped(c, g, dout, c->stream);
        d2h(out, dout, sizeof(double) * count, c->stream);
        check_flag_and_sync(c);
    });
}

extern "C" cx_status cx_coverage_scores_points(const float* cloud, int64_t count, int dim, const int64_t* selected,
                                               int64_t n_selected, double* out) {
    return guard(__func__, [&] {
        if (count == 0) return;  // synapse.cpp:105-106 (empty output)
        if (count < 0 || dim < 1 || !cloud || !out || (n_selected > 0 && !selected))
            fail(CX_INVALID_ARGUMENT, "null pointer / bad shape");
        cx_ctx* c = default_ctx();
        std::lock_guard<std::mutex> lk(c->mu);
        ArenaPlan pl;
        pl.take<float>((size_t)count * dim);
        pl.take<int64_t>((size_t)std::max<int64_t>(1, n_selected));
        pl.take<double>((size_t)count);
        pl.take<double>((size_t)dim);
        c->arena.reserve(pl.used);
        c->arena.reset();
        float* dc = c->arena.take<float>((size_t)count * dim);
        int64_t* ds = c->arena.take<int64_t>((size_t)std::max<int64_t>(1, n_selected));
        double* dout = c->arena.take<double>((size_t)count);
        h2d(dc, cloud, sizeof(float) * count * dim, c->stream);
        GroupView g = single_group(dc, count, dim);
        if (n_selected == 0) {
            coverage_centroid(c, g, dout, c->stream);
        } else {
            h2d(ds, selected, sizeof(int64_t) * n_selected, c->stream);
            coverage_selected(g, ds, n_selected, dout, c->stream);
        }
        d2h(out, dout, sizeof(double) * count, c->stream);
        CX_CUDA(cudaStreamSynchronize(c->stream));
    });
}

extern "C" cx_status cx_select_landmarks_points(const float* cloud, int64_t count, int dim, const double* attention,
                                                int64_t attention_len, int k, double lambda, int64_t* out_indices,
                                                double* out_scores, int64_t* out_n) {
    return guard(__func__, [&] {
        // synapse.cpp:219-223, in order
        if (k < 1) fail(CX_CONFIG_ERROR, "select_landmarks: k must be >= 1");
        if (lambda < 0.0 || lambda > 1.0) fail(CX_CONFIG_ERROR, "select_landmarks: lambda must be in [0,1]");
        if (attention_len != count) fail(CX_PRECONDITION_ERROR, "select_landmarks: attention length mismatch");
        const int64_t take = std::min<int64_t>(k, count);
        if (out_n) *out_n = std::max<int64_t>(0, take);
        if (count <= 0) return;
        if (dim < 1 || !cloud || !attention || !out_indices || !out_scores)
            fail(CX_INVALID_ARGUMENT, "null pointer / bad shape");
        cx_ctx* c = default_ctx();
        std::lock_guard<std::mutex> lk(c->mu);
        GroupView g = single_group(nullptr, count, dim);
        ArenaPlan pl;
        pl.take<float>((size_t)count * dim);
        pl.take<double>((size_t)count);
        pl.take<int64_t>((size_t)take);
        pl.take<double>((size_t)take);
        plan_select(pl, g, k);
        c->arena.reserve(pl.used);
        c->arena.reset();
        float* dc = c->arena.take<float>((size_t)count * dim);
        double* da = c->arena.take<double>((size_t)count);
        int64_t* dr = c->arena.take<int64_t>((size_t)take);
        double* dsc = c->arena.take<double>((size_t)take);
        g.X = dc;
        h2d(dc, cloud, sizeof(float) * count * dim, c->stream);
        h2d(da, attention, sizeof(double) * count, c->stream);
        select_grouped(c, g, da, k, lambda, 0u, dr, dsc, c->stream);
        d2h(out_indices, dr, sizeof(int64_t) * take, c->stream);
        d2h(out_scores, dsc, sizeof(double) * take, c->stream);
        CX_CUDA(cudaStreamSynchronize(c->stream));
    });
}

namespace {

// shared implementation of hausdorff_* (synapse.cpp:139-165)
void hausdorff_impl(const float* cloud, int64_t count, int dim, const float* lm, int64_t m, const int64_t* rows,
                    double* out) {
    cx_ctx* c = default_ctx();
    std::lock_guard<std::mutex> lk(c->mu);
    ArenaPlan pl;
    pl.take<float>((size_t)count * dim);
    pl.take<float>((size_t)(rows ? 1 : m) * dim);
    pl.take<int64_t>((size_t)(rows ? m : 1));
    pl.take<double>(1);
    c->arena.reserve(pl.used);
    c->arena.reset();
    float* dc = c->arena.take<float>((size_t)count * dim);
    float* dl = c->arena.take<float>((size_t)(rows ? 1 : m) * dim);
    int64_t* dr = c->arena.take<int64_t>((size_t)(rows ? m : 1));
    double* dw = c->arena.take<double>(1);
    h2d(dc, cloud, sizeof(float) * count * dim, c->stream);
    if (rows) h2d(dr, rows, sizeof(int64_t) * m, c->stream);
    else h2d(dl, lm, sizeof(float) * m * dim, c->stream);
    hausdorff(dc, count, dim, rows ? nullptr : dl, m, rows ? dr : nullptr, dw, c->stream);
    double worst = 0.0;
    d2h(&worst, dw, sizeof(double), c->stream);
    CX_CUDA(cudaStreamSynchronize(c->stream));
    *out = std::sqrt(worst);
}

// mean pairwise distance over a point set (synapse.cpp:169-191)
double mean_pairwise_impl(cx_ctx* c, const float* d_pts, int64_t count, int dim, const int64_t* d_rows, int64_t n) {
    if (n < 2) return 0.0;
    double* dsum = c->arena.take<double>(mean_pairwise_scratch(n, dim));
    mean_pairwise(d_pts, n, dim, d_rows, dsum, c->stream);
    double sum = 0.0;
    d2h(&sum, dsum, sizeof(double), c->stream);
    CX_CUDA(cudaStreamSynchronize(c->stream));
    const double pairs = (double)n * (double)(n - 1) / 2.0;
    return sum / pairs;
}

}  // namespace

extern "C" cx_status cx_hausdorff_distance(const float* cloud, int64_t count, int dim, const float* landmarks,
                                           int64_t m, int ldim, double* out) {
    return guard(__func__, [&] {
        if (count == 0 || m == 0) fail(CX_PRECONDITION_ERROR, "hausdorff_distance: empty point set");
        if (dim != ldim) fail(CX_PRECONDITION_ERROR, "hausdorff_distance: dimension mismatch");
        if (!cloud || !landmarks || !out || count < 0 || m < 0) fail(CX_INVALID_ARGUMENT, "null pointer");
        hausdorff_impl(cloud, count, dim, landmarks, m, nullptr, out);
    });
}

extern "C" cx_status cx_hausdorff_to_subset(const float* cloud, int64_t count, int dim, const int64_t* rows,
                                            int64_t n_rows, double* out) {
    return guard(__func__, [&] {
        if (n_rows == 0) fail(CX_PRECONDITION_ERROR, "hausdorff: empty landmark set");
        if (!out || !rows || n_rows < 0 || count < 0) fail(CX_INVALID_ARGUMENT, "null pointer");
        if (count == 0) { *out = 0.0; return; }
        hausdorff_impl(cloud, count, dim, nullptr, n_rows, rows, out);
    });
}

extern "C" cx_status cx_mean_pairwise_reduction(const float* cloud, int64_t count, int dim, const float* landmarks,
                                                int64_t m, int ldim, double* out) {
    return guard(__func__, [&] {
        if (m < 2) fail(CX_PRECONDITION_ERROR, "mean_pairwise_reduction: need >= 2 landmarks");
        if (count < 2) fail(CX_PRECONDITION_ERROR, "mean_pairwise_reduction: need >= 2 cloud points");
        if (!cloud || !landmarks || !out) fail(CX_INVALID_ARGUMENT, "null pointer");
        cx_ctx* c = default_ctx();
        std::lock_guard<std::mutex> lk(c->mu);
        ArenaPlan pl;
        pl.take<float>((size_t)count * dim);
        pl.take<float>((size_t)m * ldim);
        pl.take<double>(std::max(mean_pairwise_scratch(count, dim), mean_pairwise_scratch(m, ldim)));
        c->arena.reserve(pl.used);
        c->arena.reset();
        float* dc = c->arena.take<float>((size_t)count * dim);
        float* dl = c->arena.take<float>((size_t)m * ldim);
        h2d(dc, cloud, sizeof(float) * count * dim, c->stream);
        h2d(dl, landmarks, sizeof(float) * m * ldim, c->stream);
        const size_t mark = c->arena.used;
        const double cm = mean_pairwise_impl(c, dc, count, dim, nullptr, count);
        if (cm == 0.0) { *out = 0.0; return; }
        c->arena.used = mark;
        const double lmean = mean_pairwise_impl(c, dl, m, ldim, nullptr, m);
        *out = 1.0 - lmean / cm;
    });
}

extern "C" cx_status cx_mean_pairwise_reduction_subset(const float* cloud, int64_t count, int dim, const int64_t* rows,
                                                       int64_t n_rows, double* out) {
    return guard(__func__, [&] {
        if (n_rows < 2) fail(CX_PRECONDITION_ERROR, "mean_pairwise_reduction: need >= 2 landmarks");
        if (count < 2) fail(CX_PRECONDITION_ERROR, "mean_pairwise_reduction: need >= 2 cloud points");
        if (!cloud || !rows || !out) fail(CX_INVALID_ARGUMENT, "null pointer");
        cx_ctx* c = default_ctx();
        std::lock_guard<std::mutex> lk(c->mu);
        ArenaPlan pl;
        pl.take<float>((size_t)count * dim);
        pl.take<int64_t>((size_t)n_rows);
        pl.take<double>(std::max(mean_pairwise_scratch(count, dim), mean_pairwise_scratch(n_rows, dim)));
        c->arena.reserve(pl.used);
        c->arena.reset();
        float* dc = c->arena.take<float>((size_t)count * dim);
        int64_t* dr = c->arena.take<int64_t>((size_t)n_rows);
        h2d(dc, cloud, sizeof(float) * count * dim, c->stream);
        h2d(dr, rows, sizeof(int64_t) * n_rows, c->stream);
        const size_t mark = c->arena.used;
        const double cm = mean_pairwise_impl(c, dc, count, dim, nullptr, count);
        if (cm == 0.0) { *out = 0.0; return; }
        c->arena.used = mark;
        const double lmean = mean_pairwise_impl(c, dc, count, dim, dr, n_rows);
        *out = 1.0 - lmean / cm;
    });
}

extern "C" cx_status cx_attend(const float* q, const float* keys, const float* values, int64_t n_entries, int n_heads,
                               int d_k, float* out) {
    return guard(__func__, [&] {
        if (n_heads < 1 || d_k < 1 || n_entries < 1) fail(CX_PRECONDITION_ERROR, "attend: bad shape");
        if (!q || !keys || !values || !out) fail(CX_INVALID_ARGUMENT, "null pointer");
        const int64_t dm = (int64_t)n_heads * d_k;
        cx_ctx* c = default_ctx();
        std::lock_guard<std::mutex> lk(c->mu);
        ArenaPlan pl;
        pl.take<float>((size_t)dm);
        pl.take<float>((size_t)n_entries * dm);
        pl.take<float>((size_t)n_entries * dm);
        pl.take<double>((size_t)n_heads * n_entries);
        pl.take<float>((size_t)dm);
        c->arena.reserve(pl.used);
        c->arena.reset();
        float* dq = c->arena.take<float>((size_t)dm);
        float* dk = c->arena.take<float>((size_t)n_entries * dm);
        float* dv = c->arena.take<float>((size_t)n_entries * dm);
        double* dw = c->arena.take<double>((size_t)n_heads * n_entries);
        float* dout = c->arena.take<float>((size_t)dm);
        h2d(dq, q, sizeof(float) * dm, c->stream);
        h2d(dk, keys, sizeof(float) * n_entries * dm, c->stream);
        h2d(dv, values, sizeof(float) * n_entries * dm, c->stream);
        attend_fp64_ws(dq, dk, dv, n_entries, n_heads, d_k, dw, dout, c->stream);
        d2h(out, dout, sizeof(float) * dm, c->stream);
        CX_CUDA(cudaStreamSynchronize(c->stream));
    });
}

// kernels::softmax (kernels.cpp:66-92): precondition_error on empty or non-finite input
extern "C" cx_status cx_softmax(const double* scores, int64_t n, double* out) {
    return guard(__func__, [&] {
        if (n < 1) fail(CX_PRECONDITION_ERROR, "softmax: empty input");
        if (!scores || !out) fail(CX_INVALID_ARGUMENT, "null pointer");
        cx_ctx* c = default_ctx();
        std::lock_guard<std::mutex> lk(c->mu);
        ArenaPlan pl;
        pl.take<double>((size_t)n);
        pl.take<double>((size_t)n);
        c->arena.reserve(pl.used);
        c->arena.reset();
        double* ds = c->arena.take<double>((size_t)n);
        double* dout = c->arena.take<double>((size_t)n);
        CX_CUDA(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
        h2d(ds, scores, sizeof(double) * n, c->stream);
        softmax_fp64(ds, n, dout, c->d_flag, c->stream);
        d2h(out, dout, sizeof(double) * n, c->stream);
        check_flag_and_sync(c);
    });
}

// the float overload widens first (kernels.cpp:89-92)
extern "C" cx_status cx_softmax_f32(const float* scores, int64_t n, double* out) {
    return guard(__func__, [&] {
        if (n < 1) fail(CX_PRECONDITION_ERROR, "softmax: empty input");
        if (!scores || !out) fail(CX_INVALID_ARGUMENT, "null pointer");
        std::vector<double> w(scores, scores + n);
        const cx_status st = cx_softmax(w.data(), n, out);
        if (st != CX_OK) fail(st, cx_last_error());
    });
}

// kernels::argmax (kernels.cpp:94-101); the reference asserts a non-empty input
extern "C" cx_status cx_argmax(const float* v, int64_t n, int* out) {
    return guard(__func__, [&] {
        if (n < 1) fail(CX_PRECONDITION_ERROR, "argmax: empty input");
        if (!v || !out) fail(CX_INVALID_ARGUMENT, "null pointer");
        cx_ctx* c = default_ctx();
        std::lock_guard<std::mutex> lk(c->mu);
        ArenaPlan pl;
        pl.take<float>((size_t)n);
        pl.take<int>(1);
        c->arena.reserve(pl.used);
        c->arena.reset();
        float* dv = c->arena.take<float>((size_t)n);
        int* di = c->arena.take<int>(1);
        h2d(dv, v, sizeof(float) * n, c->stream);
        argmax_f32(dv, n, di, c->stream);
        d2h(out, di, sizeof(int), c->stream);
        CX_CUDA(cudaStreamSynchronize(c->stream));
    });
}

// gate.cpp:27-43 gate_score for one (h_main, t_side) pair, on the device
extern "C" cx_status cx_gate_score(const float* h_main, const float* t_side, int64_t n, double* out) {
    return guard(__func__, [&] {
        if (n < 1) fail(CX_DEGENERATE_INPUT_ERROR, "gate_score: zero-norm input");  // empty: both norms 0
        if (!h_main || !t_side || !out) fail(CX_INVALID_ARGUMENT, "null pointer");
        cx_ctx* c = default_ctx();
        std::lock_guard<std::mutex> lk(c->mu);
        ArenaPlan pl;
        pl.take<float>((size_t)n);
        pl.take<float>((size_t)n);
        pl.take<double>(1);
        pl.take<uint8_t>(1);
        c->arena.reserve(pl.used);
        c->arena.reset();
        float* dh = c->arena.take<float>((size_t)n);
        float* dt = c->arena.take<float>((size_t)n);
        double* ds = c->arena.take<double>(1);
        uint8_t* dd = c->arena.take<uint8_t>(1);
        h2d(dh, h_main, sizeof(float) * n, c->stream);
        h2d(dt, t_side, sizeof(float) * n, c->stream);
        gate_decide(dh, 0, dt, 0, 1, (int)n, 0.0, ds, nullptr, dd, c->stream);
        uint8_t deg = 0;
        d2h(out, ds, sizeof(double), c->stream);
        d2h(&deg, dd, 1, c->stream);
        CX_CUDA(cudaStreamSynchronize(c->stream));
        if (deg) fail(CX_DEGENERATE_INPUT_ERROR, "gate_score: zero-norm input");
    });
}

// gate.cpp:45-61 decide for n_pairs rows of h / t on the device (the gate fused after an
// agent step: h = the main model's last hidden states, t = the side agents' thoughts)
extern "C" cx_status cx_gate_decide_dev(cx_ctx* c, int64_t n_pairs, int dim, const float* h, int64_t h_stride,
                                        const float* t, int64_t t_stride, double theta, double* scores,
                                        uint8_t* accepted, uint8_t* degenerate, void* stream) {
    return guard(__func__, [&] {
        if (theta < -1.0 || theta > 1.0) fail(CX_PRECONDITION_ERROR, "decide: theta must be in [-1,1]");
        if (!c) fail(CX_INVALID_ARGUMENT, "null ctx");
        if (n_pairs < 0 || dim < 0) fail(CX_PRECONDITION_ERROR, "gate: bad shape");
        if (n_pairs == 0) return;
        if (!h || !t || !scores) fail(CX_INVALID_ARGUMENT, "null pointer");
        gate_decide(h, h_stride, t, t_stride, n_pairs, dim, theta, scores, accepted, degenerate, (cudaStream_t)stream);
    });
}

// ============================================================================
// grouped device path
// ============================================================================
extern "C" cx_status cx_attention_grouped_dev(cx_ctx* c, const cx_groups* gr, double* out, void* stream) {
    return guard(__func__, [&] {
        if (!c || !out) fail(CX_INVALID_ARGUMENT, "null ctx/out");
        validate_groups(gr, true);
        GroupView g = view_of(gr);
        ArenaPlan pl;
        plan_attention(pl, g);
        c->arena.reserve(pl.used);
        c->arena.reset();
        attention_grouped(c, g, out, (cudaStream_t)stream);
    });
}

extern "C" cx_status cx_select_grouped_dev(cx_ctx* c, const cx_groups* gr, const double* attention, int k,
                                           double lambda, unsigned flags, int64_t* out_rows, double* out_scores,
                                           void* stream) {
    return guard(__func__, [&] {
        if (k < 1) fail(CX_CONFIG_ERROR, "select_landmarks: k must be >= 1");
        if (lambda < 0.0 || lambda > 1.0) fail(CX_CONFIG_ERROR, "select_landmarks: lambda must be in [0,1]");
        if (!c) fail(CX_INVALID_ARGUMENT, "null ctx");
        validate_groups(gr, false);
        if (gr->count == 0 || gr->n_groups == 0) return;
        if (!attention || !out_rows || !out_scores) fail(CX_INVALID_ARGUMENT, "null pointer");
        GroupView g = view_of(gr);
        ArenaPlan pl;
        plan_select(pl, g, k);
        c->arena.reserve(pl.used);
        c->arena.reset();
        select_grouped(c, g, attention, k, lambda, flags, out_rows, out_scores, (cudaStream_t)stream);
    });
}

extern "C" cx_status cx_ctx_set_option(cx_ctx* c, int option, int64_t value) {
    return guard(__func__, [&] {
        if (!c) fail(CX_INVALID_ARGUMENT, "null ctx");
        auto in = [&](int64_t lo, int64_t hi) {
            if (value < lo || value > hi) fail(CX_INVALID_ARGUMENT, "ctx_set_option: value out of range");
            return (int)value;
        };
        switch (option) {
            case CX_OPT_SELECT_CLUSTER: c->opt.select_cluster = in(0, 16); break;
            case CX_OPT_SELECT_NO_SKETCH: c->opt.select_no_sketch = in(0, 1); break;
            case CX_OPT_DECODE_IMPL: c->opt.decode_impl = in(CX_DECODE_AUTO, CX_DECODE_V1); break;
            case CX_OPT_DECODE_CTAS_PER_LH: c->opt.decode_ctas_per_lh = in(0, 1 << 16); break;
            case CX_OPT_HOST_UPLOAD_VALUES: c->opt.host_upload_values = in(0, 1); break;
            case CX_OPT_HOST_STAGE_OUTPUTS: c->opt.host_stage_outputs = in(0, 1); break;
            case CX_OPT_SELECT_IMPL: c->opt.select_impl = in(CX_SELECT_IMPL_AUTO, CX_SELECT_IMPL_CUDA_CORE); break;
            case CX_OPT_SELECT_EXCHANGE: c->opt.select_exchange = in(0, 3); break;
            default: fail(CX_INVALID_ARGUMENT, "ctx_set_option: unknown option");
        }
        if (c->aux) c->aux->opt = c->opt;  // the host path's prologue context follows
    });
}

extern "C" cx_status cx_ctx_get_option(cx_ctx* c, int option, int64_t* value) {
    return guard(__func__, [&] {
        if (!c || !value) fail(CX_INVALID_ARGUMENT, "null ctx/value");
        switch (option) {
            case CX_OPT_SELECT_CLUSTER: *value = c->opt.select_cluster; break;
            case CX_OPT_SELECT_NO_SKETCH: *value = c->opt.select_no_sketch; break;
            case CX_OPT_DECODE_IMPL: *value = c->opt.decode_impl; break;
            case CX_OPT_DECODE_CTAS_PER_LH: *value = c->opt.decode_ctas_per_lh; break;
            case CX_OPT_HOST_UPLOAD_VALUES: *value = c->opt.host_upload_values; break;
            case CX_OPT_HOST_STAGE_OUTPUTS: *value = c->opt.host_stage_outputs; break;
            case CX_OPT_SELECT_IMPL: *value = c->opt.select_impl; break;
            case CX_OPT_SELECT_EXCHANGE: *value = c->opt.select_exchange; break;
            default: fail(CX_INVALID_ARGUMENT, "ctx_get_option: unknown option");
        }
    });
}

extern "C" cx_status cx_ctx_device_errors(cx_ctx* c, void* stream, unsigned* flags, int clear) {
    return guard(__func__, [&] {
        if (!c || !flags) fail(CX_INVALID_ARGUMENT, "null ctx/flags");
        int f = 0;
        cudaStream_t s = (cudaStream_t)stream;
        CX_CUDA(cudaMemcpyAsync(&f, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
        if (clear) CX_CUDA(cudaMemsetAsync(c->d_flag, 0, sizeof(int), s));
        CX_CUDA(cudaStreamSynchronize(s));
        *flags = (unsigned)f;
    });
}

extern "C" cx_status cx_selection_gaps(cx_ctx* c, int n_groups, double* out, void* stream) {
    return guard(__func__, [&] {
        if (!c || !out) fail(CX_INVALID_ARGUMENT, "null ctx/out");
        if (n_groups < 0 || n_groups > c->gaps_n)
            fail(CX_PRECONDITION_ERROR, "selection_gaps: more groups than the last selection launch");
        if (n_groups == 0) return;
        CX_CUDA(cudaMemcpyAsync(out, c->gaps, sizeof(double) * (size_t)n_groups, cudaMemcpyDefault,
                                (cudaStream_t)stream));
    });
}

extern "C" cx_status cx_gather_grouped_dev(cx_ctx* c, const cx_groups* gr, const float* src, const int64_t* rows,
                                           int take, float* dst, void* stream) {
    return guard(__func__, [&] {
        if (!c) fail(CX_INVALID_ARGUMENT, "null ctx");
        validate_groups(gr, false);
        if (take < 0) fail(CX_INVALID_ARGUMENT, "negative take");
        if (take == 0 || gr->n_groups == 0) return;
        if (!src || !rows || !dst) fail(CX_INVALID_ARGUMENT, "null pointer");
        gather_rows(view_of(gr), src, rows, take, dst, (cudaStream_t)stream);
    });
}

namespace {

// attention || centroid, selection, landmark gather for the groups of `gr` (validated)
void compress_impl(cx_ctx* c, const cx_groups* gr, const float* values, int k, double lambda, unsigned flags,
                   int64_t* out_rows, double* out_scores, float* syn_keys, float* syn_values, void* stream,
                   int64_t syn_gstride = 0) {
    {
        GroupView g = view_of(gr);
        const int take = (int)std::min<int64_t>(k, g.L);
        ArenaPlan pl;
        pl.take<double>((size_t)g.G * g.L);
        pl.take<double>((size_t)g.G * g.dim);
        plan_attention(pl, g);
        plan_select(pl, g, k);
        c->arena.reserve(pl.used);
        c->arena.reset();
        cudaStream_t s = (cudaStream_t)stream;
        double* attn = c->arena.take<double>((size_t)g.G * g.L);
        double* cen = c->arena.take<double>((size_t)g.G * g.dim);
        // fork: the centroids (A2, a latency-bound serial sum per coordinate)
        // run on the side stream while the attention mass (A3) runs on `s`
#ifdef CX_EXPERIMENTS
        // timing only (results invalid): 1 = skip the centroids, 2 = skip the attention mass, 3 = both
        const int skip_pro = getenv("CX_EXP_PROLOGUE") ? atoi(getenv("CX_EXP_PROLOGUE")) : 0;
#else
        const int skip_pro = 0;
#endif
        CX_CUDA(cudaEventRecord(c->ev_fork, s));
        CX_CUDA(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
        if (skip_pro != 1 && skip_pro != 3) centroid_launch(g, cen, c->side);
        CX_CUDA(cudaEventRecord(c->ev_join, c->side));
        const size_t mark = c->arena.used;
        if (skip_pro != 2 && skip_pro != 3) attention_grouped(c, g, attn, s);
        c->arena.used = mark;  // attention scratch is dead once `attn` is written (stream-ordered)
        CX_CUDA(cudaStreamWaitEvent(s, c->ev_join, 0));
        const int64_t gs = syn_gstride > 0 ? syn_gstride : (int64_t)take * g.dim;
        const SynGather gat{values, syn_keys, values ? syn_values : nullptr, gs};
        if (select_grouped(c, g, attn, k, lambda, flags, out_rows, out_scores, s, cen, &gat))
            return;  // the selection kernel gathered the landmark rows itself
        if (syn_keys && syn_values && values)  // keys and values in one launch
            gather_rows2(g, g.X, values, out_rows, take, syn_keys, syn_values, gs, s);
        else if (syn_keys)
            gather_rows2(g, g.X, nullptr, out_rows, take, syn_keys, nullptr, gs, s);
        else if (syn_values && values)
            gather_rows2(g, values, nullptr, out_rows, take, syn_values, nullptr, gs, s);
    }
}

}  // namespace

extern "C" cx_status cx_compress_grouped_dev(cx_ctx* c, const cx_groups* gr, const float* values, int k, double lambda,
                                             unsigned flags, int64_t* out_rows, double* out_scores, float* syn_keys,
                                             float* syn_values, void* stream) {
    return guard(__func__, [&] {
        if (k < 1) fail(CX_CONFIG_ERROR, "select_landmarks: k must be >= 1");
        if (lambda < 0.0 || lambda > 1.0) fail(CX_CONFIG_ERROR, "select_landmarks: lambda must be in [0,1]");
        if (!c) fail(CX_INVALID_ARGUMENT, "null ctx");
        validate_groups(gr, true);
        if (!out_rows || !out_scores) fail(CX_INVALID_ARGUMENT, "null outputs");
        compress_impl(c, gr, values, k, lambda, flags, out_rows, out_scores, syn_keys, syn_values, stream);
    });
}

// the same with the synapse blocks syn_group_stride floats apart (0: take * dim), e.g. straight
// into the decode layout [layer][kv head][k][d_k] from a per-head view of the river cache
extern "C" cx_status cx_compress_grouped_strided_dev(cx_ctx* c, const cx_groups* gr, const float* values, int k,
                                                     double lambda, unsigned flags, int64_t* out_rows,
                                                     double* out_scores, float* syn_keys, float* syn_values,
                                                     int64_t syn_group_stride, void* stream) {
    return guard(__func__, [&] {
        if (k < 1) fail(CX_CONFIG_ERROR, "select_landmarks: k must be >= 1");
        if (lambda < 0.0 || lambda > 1.0) fail(CX_CONFIG_ERROR, "select_landmarks: lambda must be in [0,1]");
        if (!c) fail(CX_INVALID_ARGUMENT, "null ctx");
        validate_groups(gr, true);
        if (!out_rows || !out_scores) fail(CX_INVALID_ARGUMENT, "null outputs");
        const int64_t take = std::min<int64_t>(k, gr->count);
        if (syn_group_stride != 0 && syn_group_stride < take * gr->dim)
            fail(CX_INVALID_ARGUMENT, "syn_group_stride smaller than a group's take * dim");
        compress_impl(c, gr, values, k, lambda, flags, out_rows, out_scores, syn_keys, syn_values, stream,
                      syn_group_stride);
    });
}

extern "C" cx_status cx_compress_grouped_host(cx_ctx* c, int n_groups, int64_t count, int dim, const float* keys,
                                              const float* values, const float* queries, int n_pass, int d_k,
                                              int col_step, int k, double lambda, unsigned flags, int64_t* out_rows,
                                              double* out_scores, float* syn_keys, float* syn_values) {
    return guard(__func__, [&] {
        if (k < 1) fail(CX_CONFIG_ERROR, "select_landmarks: k must be >= 1");
        if (lambda < 0.0 || lambda > 1.0) fail(CX_CONFIG_ERROR, "select_landmarks: lambda must be in [0,1]");
        if (!c) fail(CX_INVALID_ARGUMENT, "null ctx");
        cx_groups all{};
        all.n_groups = n_groups;
        all.count = count;
        all.dim = dim;
        all.clouds = keys;
        all.group_stride = count * dim;
        all.row_stride = dim;
        all.queries = queries;
        all.n_pass = n_pass;
        all.d_k = d_k;
        all.col_step = col_step;
        validate_groups(&all, true);
        if (!out_rows || !out_scores || !values) fail(CX_INVALID_ARGUMENT, "null pointer");
        if (n_groups == 0) return;
        const int take = (int)std::min<int64_t>(k, count);
        const size_t in_g = (size_t)count * dim, q_g = (size_t)n_pass * d_k, o_g = (size_t)take * dim;
        // Values are only read at the selected rows (2% at cfg2).  When the caller's buffer is
        // pinned (device-accessible through UVA) the landmark gather reads those rows straight
        // from host memory over PCIe instead of uploading every value row.
        const float* vdev = nullptr;
        {
            cudaPointerAttributes pa{};
            if (cudaPointerGetAttributes(&pa, values) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
                pa.devicePointer != nullptr && !c->opt.host_upload_values)
                vdev = reinterpret_cast<const float*>(pa.devicePointer);
            cudaGetLastError();
        }
        // Likewise the synapse K/V: when both output buffers are pinned, the landmark gather
        // writes the rows straight into them (posted PCIe writes, overlapping the gather's
        // reads) instead of a device copy plus a 4 MB D2H after the selection.
        float* hsk = nullptr;
        float* hsv = nullptr;
        if (syn_keys && syn_values && !c->opt.host_stage_outputs) {
            cudaPointerAttributes ka{}, va{};
            if (cudaPointerGetAttributes(&ka, syn_keys) == cudaSuccess && ka.type == cudaMemoryTypeHost &&
                ka.devicePointer != nullptr && cudaPointerGetAttributes(&va, syn_values) == cudaSuccess &&
                va.type == cudaMemoryTypeHost && va.devicePointer != nullptr) {
                hsk = reinterpret_cast<float*>(ka.devicePointer);
                hsv = reinterpret_cast<float*>(va.devicePointer);
            }
            cudaGetLastError();
        }
        // device staging: keys | values | queries | rows | scores | syn_k | syn_v (256-B aligned slices)
        auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
        const size_t b_k = al(sizeof(float) * in_g * n_groups), b_q = al(sizeof(float) * q_g * n_groups);
        const size_t b_r = al(sizeof(int64_t) * take * n_groups), b_s = al(sizeof(double) * take * n_groups);
        const size_t b_o = al(sizeof(float) * o_g * n_groups);
        const size_t b_a = al(sizeof(double) * (size_t)count * n_groups), b_c = al(sizeof(double) * dim * n_groups);
        const size_t need = 2 * b_k + b_q + b_r + b_s + 2 * b_o + b_a + b_c;
        if (need > c->hcap) {
            if (c->hbuf) {
                CX_CUDA(cudaStreamSynchronize(c->stream));
                cudaFree(c->hbuf);
            }
            c->hbuf = nullptr;
            c->hcap = 0;
            CX_CUDA(cudaMalloc(&c->hbuf, need));
            c->hcap = need;
        }
        char* p = c->hbuf;
        float* dk = reinterpret_cast<float*>(p); p += b_k;
        float* dv = reinterpret_cast<float*>(p); p += b_k;
        float* dq = reinterpret_cast<float*>(p); p += b_q;
        int64_t* dr = reinterpret_cast<int64_t*>(p); p += b_r;
        double* ds = reinterpret_cast<double*>(p); p += b_s;
        float* dsk = reinterpret_cast<float*>(p); p += b_o;
        float* dsv = reinterpret_cast<float*>(p); p += b_o;
        if (hsk) {  // gather destinations: the caller's pinned buffers
            dsk = hsk;
            dsv = hsv;
        }
        double* dattn = reinterpret_cast<double*>(p); p += b_a;
        double* dcen = reinterpret_cast<double*>(p);
        // Chunks of groups, one selection wave each (the cost model's co-resident clusters:
        // 22 on B200 at L=8192), so chunking costs no compute; the remainder goes FIRST so
        // that the only exposed upload is the smallest one.
        // When the tensor-core selection of ALL groups is one wave (cfg2: the split plan), the
        // uploads are chunked only for the prologues (centroid + attention of a chunk run as soon
        // as it lands) and ONE selection over every group follows the last prologue: PCIe +
        // one selection, instead of a pipeline of per-wave selections (the selection's latency
        // does not depend on how many of the co-resident groups it runs).
        const bool one_wave = dim == 64 && select_tc_wave(count, n_groups) >= n_groups && c->opt.select_impl != CX_SELECT_IMPL_CUDA_CORE;
        const int w = one_wave ? (n_groups + 3) / 4 : dim == 64 ? select64_wave(count, n_groups) : 0;
        const int WAVE = w > 0 ? w : 15;
        std::vector<int> start;
#ifdef CX_EXPERIMENTS
        const char* ch = getenv("CX_E2E_CHUNKS");  // tuning only: explicit chunk sizes "a,b,c"
#else
        const char* ch = nullptr;
#endif
        if (ch) {
            int g0 = 0;
            for (const char* q = ch; *q && g0 < n_groups;) {
                const int n = std::max(1, atoi(q));
                start.push_back(g0);
                g0 += n;
                while (*q && *q != ',') ++q;
                if (*q == ',') ++q;
            }
            if (start.empty()) start.push_back(0);
            if (g0 < n_groups) start.push_back(g0);  // the rest as one chunk
        } else {
            for (int g0 = 0, first = n_groups % WAVE ? n_groups % WAVE : WAVE; g0 < n_groups; g0 += (g0 ? WAVE : first))
                start.push_back(g0);
        }
        const int nch = (int)start.size();
        start.push_back(n_groups);
        while ((int)c->hev.size() < nch) {
            cudaEvent_t e, f;
            CX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            CX_CUDA(cudaEventCreateWithFlags(&f, cudaEventDisableTiming));
            c->hev.push_back(e);
            c->pev.push_back(f);
        }
        // The prologue of each chunk (centroid + attention mass: latency-bound, few SMs)
        // runs on a second context while the previous chunk's selection holds the rest
        // of the GPU; scratch is sized once for the largest chunk.
        if (!c->aux) {
            auto* a = new cx_ctx();
            try {
                ctx_init(a, c->device);
            } catch (...) {
                delete a;
                throw;
            }
            c->aux = a;
        }
        cx_ctx* x = c->aux;
        x->opt = c->opt;
        {
            int maxg = 0;
            for (int i = 0; i < nch; ++i) maxg = std::max(maxg, start[i + 1] - start[i]);
            cx_groups gm = all;
            gm.n_groups = maxg;
            GroupView vm = view_of(&gm);
            ArenaPlan pa, ps;
            plan_attention(pa, vm);
            if (one_wave) {
                const GroupView va = view_of(&all);
                plan_select(ps, va, k);
            } else {
                plan_select(ps, vm, k);
            }
            CX_CUDA(cudaStreamSynchronize(x->stream));
            x->arena.reserve(pa.used);
            CX_CUDA(cudaStreamSynchronize(c->stream));
            c->arena.reserve(ps.used);
        }
        CX_CUDA(cudaMemsetAsync(x->d_flag, 0, sizeof(int), x->stream));
        CX_CUDA(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
        for (int i = 0; i < nch; ++i) {  // all uploads queued on the copy stream
            const int g0 = start[i], ng = start[i + 1] - g0;
            CX_CUDA(cudaMemcpyAsync(dk + g0 * in_g, keys + g0 * in_g, sizeof(float) * in_g * ng, cudaMemcpyHostToDevice, c->copy));
            if (!vdev)
                CX_CUDA(cudaMemcpyAsync(dv + g0 * in_g, values + g0 * in_g, sizeof(float) * in_g * ng, cudaMemcpyHostToDevice,
                                        c->copy));
            CX_CUDA(cudaMemcpyAsync(dq + g0 * q_g, queries + g0 * q_g, sizeof(float) * q_g * ng, cudaMemcpyHostToDevice, c->copy));
            CX_CUDA(cudaEventRecord(c->hev[i], c->copy));
        }
        for (int i = 0; i < nch; ++i) {  // prologues: as soon as each upload lands
            const int g0 = start[i], ng = start[i + 1] - g0;
            CX_CUDA(cudaStreamWaitEvent(x->stream, c->hev[i], 0));
            cx_groups gi = all;
            gi.n_groups = ng;
            gi.clouds = dk + g0 * in_g;
            gi.queries = dq + g0 * q_g;
            const GroupView g = view_of(&gi);
            centroid_launch(g, dcen + (size_t)g0 * dim, x->stream);
            x->arena.reset();
            attention_grouped(x, g, dattn + (size_t)g0 * count, x->stream);
            CX_CUDA(cudaEventRecord(c->pev[i], x->stream));
        }
        if (one_wave) {  // every prologue, then one selection + gather over all groups
            for (int i = 0; i < nch; ++i) CX_CUDA(cudaStreamWaitEvent(c->stream, c->pev[i], 0));
            cx_groups ga = all;
            ga.clouds = dk;
            ga.queries = dq;
            const GroupView g = view_of(&ga);
            c->arena.reset();
            const SynGather gat{vdev ? vdev : dv, dsk, dsv, (int64_t)o_g};
            if (!select_grouped(c, g, dattn, k, lambda, flags, dr, ds, c->stream, dcen, &gat))
                gather_rows2(g, g.X, vdev ? vdev : dv, dr, take, dsk, dsv, (int64_t)o_g, c->stream);  // K and V, one launch
        }
        for (int i = 0; i < nch && !one_wave; ++i) {  // selection + gather of chunk i after its prologue
            const int g0 = start[i], ng = start[i + 1] - g0;
            CX_CUDA(cudaStreamWaitEvent(c->stream, c->pev[i], 0));
            cx_groups gi = all;
            gi.n_groups = ng;
            gi.clouds = dk + g0 * in_g;
            gi.queries = dq + g0 * q_g;
            const GroupView g = view_of(&gi);
            c->arena.reset();
            select_grouped(c, g, dattn + (size_t)g0 * count, k, lambda, flags, dr + (size_t)g0 * take,
                           ds + (size_t)g0 * take, c->stream, dcen + (size_t)g0 * dim);
            gather_rows(g, g.X, dr + (size_t)g0 * take, take, dsk + g0 * o_g, c->stream);
            gather_rows(g, (vdev ? vdev : dv) + g0 * in_g, dr + (size_t)g0 * take, take, dsv + g0 * o_g, c->stream);
        }
        CX_CUDA(cudaMemcpyAsync(out_rows, dr, sizeof(int64_t) * take * n_groups, cudaMemcpyDeviceToHost, c->stream));
        CX_CUDA(cudaMemcpyAsync(out_scores, ds, sizeof(double) * take * n_groups, cudaMemcpyDeviceToHost, c->stream));
        if (syn_keys && !hsk)
            CX_CUDA(cudaMemcpyAsync(syn_keys, dsk, sizeof(float) * o_g * n_groups, cudaMemcpyDeviceToHost, c->stream));
        if (syn_values && !hsk)
            CX_CUDA(cudaMemcpyAsync(syn_values, dsv, sizeof(float) * o_g * n_groups, cudaMemcpyDeviceToHost, c->stream));
        check_flag_and_sync(x);  // non-finite attention input -> precondition_error (kernels.cpp:70)
        check_flag_and_sync(c);
    });
}

extern "C" cx_status cx_decode_step_dev(cx_ctx* c, const cx_decode_batch* b, void* stream) {
    return guard(__func__, [&] {
        if (!c || !b) fail(CX_INVALID_ARGUMENT, "null ctx/batch");
        if (b->n_agents < 0 || b->n_layers < 1 || b->n_kv < 1 || b->n_q < b->n_kv || b->n_q % b->n_kv != 0 ||
            b->d_k < 1 || b->k_syn < 0 || b->t_cap < 1)
            fail(CX_PRECONDITION_ERROR, "decode_step: bad shape");
        if (b->n_q / b->n_kv > 8) fail(CX_PRECONDITION_ERROR, "decode_step: more than 8 q-heads per KV head");
        if (b->n_agents == 0) return;
        if ((b->k_syn > 0 && (!b->syn_keys || !b->syn_values)) || !b->tail_keys || !b->tail_values || !b->tail_len ||
            !b->q || !b->out)
            fail(CX_INVALID_ARGUMENT, "null pointer");  // an empty synapse (k_syn = 0) may pass NULL
        if ((b->new_keys == nullptr) != (b->new_values == nullptr))
            fail(CX_INVALID_ARGUMENT, "new_keys/new_values must both be set or both NULL");
        decode_step(c, *b, (cudaStream_t)stream);
    });
}

// ============================================================================
// device KvCache (model.hpp:67-113)
// ============================================================================

namespace cx {
// Appends may run on a caller stream s.  Before: s waits for the cache's own pending work
// (a regrow's copies).  After: the cache's stream waits for s, so a later regrow, read or
// selection (all on c->stream) is ordered after the append.
void kv_before(cx_kvcache* c, cudaStream_t s) {
    if (s == c->stream) return;
    CX_CUDA(cudaEventRecord(c->ev, c->stream));
    CX_CUDA(cudaStreamWaitEvent(s, c->ev, 0));
}
void kv_after(cx_kvcache* c, cudaStream_t s) {
    if (s == c->stream) return;
    CX_CUDA(cudaEventRecord(c->ev, s));
    CX_CUDA(cudaStreamWaitEvent(c->stream, c->ev, 0));
}

void kv_grow(cx_kvcache* c, int64_t need) {
    if (need <= c->capacity) return;
    // the first allocation is exactly the requested capacity; growth doubles (at least 64 rows)
    int64_t cap = c->capacity == 0 ? need : std::max<int64_t>(need, std::max<int64_t>(64, c->capacity * 2));
    const size_t per_layer_old = (size_t)c->capacity * c->d_model;
    const size_t per_layer_new = (size_t)cap * c->d_model;
    float *nk = nullptr, *nv = nullptr;
    CX_CUDA(cudaMalloc(&nk, sizeof(float) * per_layer_new * c->n_layers));
    CX_CUDA(cudaMalloc(&nv, sizeof(float) * per_layer_new * c->n_layers));
    const int64_t rows = (int64_t)c->positions.size();
    if (c->keys && rows > 0) {
        for (int l = 0; l < c->n_layers; ++l) {
            CX_CUDA(cudaMemcpyAsync(nk + l * per_layer_new, c->keys + l * per_layer_old,
                                    sizeof(float) * rows * c->d_model, cudaMemcpyDeviceToDevice, c->stream));
            CX_CUDA(cudaMemcpyAsync(nv + l * per_layer_new, c->values + l * per_layer_old,
                                    sizeof(float) * rows * c->d_model, cudaMemcpyDeviceToDevice, c->stream));
        }
    }
    CX_CUDA(cudaStreamSynchronize(c->stream));
    if (c->keys) cudaFree(c->keys);
    if (c->values) cudaFree(c->values);
    c->keys = nk;
    c->values = nv;
    c->capacity = cap;
}
}  // namespace cx

namespace {


// model.cpp:124-140 (begin_entry) checks + host-side bookkeeping
void kv_begin(cx_kvcache* c, int64_t position, cx_origin origin) {
    if (c->entry_open) fail(CX_SEQUENCING_ERROR, "cache entry already open");
    if (position < 0 || position >= c->max_positions)
        fail(CX_CAPACITY_ERROR, "position " + std::to_string(position) + " outside max_positions " +
                                    std::to_string(c->max_positions));
    if (origin == CX_ORIGIN_CONTEXT && position <= c->last_context_position)
        fail(CX_PRECONDITION_ERROR, "context positions must be strictly increasing");
    kv_grow(c, (int64_t)c->positions.size() + 1);
    c->positions.push_back(position);
    c->origins.push_back((uint8_t)origin);
    if (origin == CX_ORIGIN_CONTEXT) {
        c->last_context_position = position;
        ++c->context_count;
    }
    c->entry_open = true;
    c->layers_written = 0;
}

}  // namespace

extern "C" cx_status cx_kvcache_create(int n_layers, int n_heads, int d_model, int d_k, int64_t max_positions,
                                       int64_t capacity, cx_kvcache** out) {
    return guard(__func__, [&] {
        // ModelConfig::validate (model.cpp:12-21), the parts KvCache depends on
        if (n_layers < 1 || n_heads < 1 || d_model < 1 || d_k < 1) fail(CX_CONFIG_ERROR, "model dimensions must be positive");
        if (n_heads * d_k != d_model) fail(CX_CONFIG_ERROR, "d_model must equal n_heads * d_k exactly");
        if (d_k % 2 != 0) fail(CX_CONFIG_ERROR, "d_k must be even for pairwise rotation");
        if (max_positions < 1) fail(CX_CONFIG_ERROR, "max_positions must be positive");
        if (!out) fail(CX_INVALID_ARGUMENT, "null out");
        require_device();
        auto* c = new cx_kvcache();
        c->n_layers = n_layers;
        c->n_heads = n_heads;
        c->d_model = d_model;
        c->d_k = d_k;
        c->max_positions = max_positions;
        try {
            CX_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
            CX_CUDA(cudaEventCreateWithFlags(&c->ev, cudaEventDisableTiming));
            kv_grow(c, std::max<int64_t>(1, capacity));
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

// value semantics of the reference KvCache (model.hpp:67-113 is copyable): a deep copy
extern "C" cx_status cx_kvcache_clone(const cx_kvcache* src, cx_kvcache** out) {
    return guard(__func__, [&] {
        if (!src || !out) fail(CX_INVALID_ARGUMENT, "null cache/out");
        cx_kvcache* c = nullptr;
        const cx_status st = cx_kvcache_create(src->n_layers, src->n_heads, src->d_model, src->d_k, src->max_positions,
                                               std::max<int64_t>(1, src->capacity), &c);
        if (st != CX_OK) fail(st, cx_last_error());
        try {
            CX_CUDA(cudaStreamSynchronize(src->stream));  // the source's pending appends
            const int64_t rows = (int64_t)src->positions.size() + (src->entry_open ? 1 : 0);
            if (rows > 0)
                for (int l = 0; l < src->n_layers; ++l) {
                    const size_t o_src = (size_t)l * src->capacity * src->d_model;
                    const size_t o_dst = (size_t)l * c->capacity * c->d_model;
                    CX_CUDA(cudaMemcpyAsync(c->keys + o_dst, src->keys + o_src, sizeof(float) * rows * src->d_model,
                                            cudaMemcpyDeviceToDevice, c->stream));
                    CX_CUDA(cudaMemcpyAsync(c->values + o_dst, src->values + o_src,
                                            sizeof(float) * rows * src->d_model, cudaMemcpyDeviceToDevice, c->stream));
                }
            CX_CUDA(cudaStreamSynchronize(c->stream));
        } catch (...) {
            cx_kvcache_destroy(c);
            throw;
        }
        c->positions = src->positions;
        c->origins = src->origins;
        c->last_context_position = src->last_context_position;
        c->context_count = src->context_count;
        c->entry_open = src->entry_open;
        c->layers_written = src->layers_written;
        *out = c;
    });
}

extern "C" cx_status cx_kvcache_destroy(cx_kvcache* c) {
    return guard(__func__, [&] {
        if (!c) return;
        cudaStreamSynchronize(c->stream);
        if (c->keys) cudaFree(c->keys);
        if (c->values) cudaFree(c->values);
        if (c->ev) cudaEventDestroy(c->ev);
        cudaStreamDestroy(c->stream);
        delete c;
    });
}

extern "C" int64_t cx_kvcache_size(const cx_kvcache* c) { return c ? (int64_t)c->positions.size() : 0; }
extern "C" int64_t cx_kvcache_context_count(const cx_kvcache* c) { return c ? c->context_count : 0; }
extern "C" int64_t cx_kvcache_last_context_position(const cx_kvcache* c) { return c ? c->last_context_position : -1; }
extern "C" int cx_kvcache_entry_open(const cx_kvcache* c) { return c && c->entry_open ? 1 : 0; }
extern "C" int64_t cx_kvcache_capacity(const cx_kvcache* c) { return c ? c->capacity : 0; }
extern "C" float* cx_kvcache_keys_dev(cx_kvcache* c) { return c ? c->keys : nullptr; }
extern "C" float* cx_kvcache_values_dev(cx_kvcache* c) { return c ? c->values : nullptr; }
extern "C" const int64_t* cx_kvcache_positions_host(const cx_kvcache* c) { return c ? c->positions.data() : nullptr; }
extern "C" const uint8_t* cx_kvcache_origins_host(const cx_kvcache* c) { return c ? c->origins.data() : nullptr; }

extern "C" cx_status cx_kvcache_begin_entry(cx_kvcache* c, int64_t position, cx_origin origin) {
    return guard(__func__, [&] {
        if (!c) fail(CX_INVALID_ARGUMENT, "null cache");
        kv_begin(c, position, origin);
    });
}

extern "C" cx_status cx_kvcache_write_layer(cx_kvcache* c, int layer, const float* key, const float* value,
                                            int64_t width) {
    return guard(__func__, [&] {
        if (!c) fail(CX_INVALID_ARGUMENT, "null cache");
        // model.cpp:144-147
        if (!c->entry_open) fail(CX_SEQUENCING_ERROR, "no open cache entry");
        if (layer != c->layers_written) fail(CX_SEQUENCING_ERROR, "layers must be written in order");
        if (width != c->d_model || !key || !value) fail(CX_PRECONDITION_ERROR, "write_layer: width mismatch");
        const int64_t row = (int64_t)c->positions.size() - 1;
        const size_t off = ((size_t)layer * c->capacity + row) * c->d_model;
        h2d(c->keys + off, key, sizeof(float) * c->d_model, c->stream);
        h2d(c->values + off, value, sizeof(float) * c->d_model, c->stream);
        CX_CUDA(cudaStreamSynchronize(c->stream));  // caller's spans may die after return
        ++c->layers_written;
    });
}

extern "C" cx_status cx_kvcache_end_entry(cx_kvcache* c) {
    return guard(__func__, [&] {
        if (!c) fail(CX_INVALID_ARGUMENT, "null cache");
        // model.cpp:155-157
        if (!c->entry_open) fail(CX_SEQUENCING_ERROR, "no open cache entry");
        if (c->layers_written != c->n_layers) fail(CX_SEQUENCING_ERROR, "entry incomplete: not all layers written");
        c->entry_open = false;
    });
}

extern "C" cx_status cx_kvcache_append_entry(cx_kvcache* c, int64_t position, cx_origin origin, const float* keys,
                                             const float* values) {
    return guard(__func__, [&] {
        if (!c || !keys || !values) fail(CX_INVALID_ARGUMENT, "null pointer");
        kv_begin(c, position, origin);  // model.cpp:161-173: begin, write every layer, end
        const int64_t row = (int64_t)c->positions.size() - 1;
        for (int l = 0; l < c->n_layers; ++l) {
            const size_t off = ((size_t)l * c->capacity + row) * c->d_model;
            h2d(c->keys + off, keys + (size_t)l * c->d_model, sizeof(float) * c->d_model, c->stream);
            h2d(c->values + off, values + (size_t)l * c->d_model, sizeof(float) * c->d_model, c->stream);
        }
        CX_CUDA(cudaStreamSynchronize(c->stream));
        c->layers_written = c->n_layers;
        c->entry_open = false;
    });
}

extern "C" cx_status cx_kvcache_append_context_dev(cx_kvcache* c, const float* keys, const float* values,
                                                    int64_t base_position, int64_t count, void* stream) {
    return guard(__func__, [&] {
        if (!c) fail(CX_INVALID_ARGUMENT, "null cache");
        if (count < 0) fail(CX_INVALID_ARGUMENT, "negative count");
        if (count == 0) return;
        if (!keys || !values) fail(CX_INVALID_ARGUMENT, "null block");
        // the checks begin_entry would make for each entry in turn (model.cpp:124-140)
        cx_status err = CX_OK;
        std::string msg;
        int64_t n_ok = 0;
        if (c->entry_open) {
            err = CX_SEQUENCING_ERROR;
            msg = "cache entry already open";
        } else {
            int64_t last = c->last_context_position;
            for (; n_ok < count; ++n_ok) {
                const int64_t p = base_position + n_ok;
                if (p < 0 || p >= c->max_positions) {
                    err = CX_CAPACITY_ERROR;
                    msg = "position " + std::to_string(p) + " outside max_positions " + std::to_string(c->max_positions);
                    break;
                }
                if (p <= last) {
                    err = CX_PRECONDITION_ERROR;
                    msg = "context positions must be strictly increasing";
                    break;
                }
                last = p;
            }
        }
        if (n_ok > 0) {
            cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
            const int64_t row0 = (int64_t)c->positions.size();
            kv_grow(c, row0 + n_ok);
            kv_before(c, s);
            if (n_ok == count) {  // the whole block: one launch for all layers
                kv_append_rows(c->keys, c->values, c->capacity, c->n_layers, c->d_model, keys, values, n_ok, row0, s);
            } else {
                for (int l = 0; l < c->n_layers; ++l)
                    kv_append_rows(c->keys + (size_t)l * c->capacity * c->d_model,
                                   c->values + (size_t)l * c->capacity * c->d_model, c->capacity, 1, c->d_model,
                                   keys + (size_t)l * count * c->d_model, values + (size_t)l * count * c->d_model,
                                   n_ok, row0, s);
            }
            kv_after(c, s);
            for (int64_t t = 0; t < n_ok; ++t) {
                c->positions.push_back(base_position + t);
                c->origins.push_back((uint8_t)CX_ORIGIN_CONTEXT);
            }
            c->last_context_position = base_position + n_ok - 1;
            c->context_count += n_ok;
        }
        if (err != CX_OK) fail(err, msg);
    });
}

extern "C" cx_status cx_kvcache_read(const cx_kvcache* c, int layer, int64_t first, int64_t n, float* keys_out,
                                     float* values_out) {
    return guard(__func__, [&] {
        if (!c) fail(CX_INVALID_ARGUMENT, "null cache");
        if (layer < 0 || layer >= c->n_layers || first < 0 || n < 0 || first + n > (int64_t)c->positions.size())
            fail(CX_PRECONDITION_ERROR, "kvcache_read: range outside the cache");
        const size_t off = ((size_t)layer * c->capacity + first) * c->d_model;
        if (keys_out) d2h(keys_out, c->keys + off, sizeof(float) * n * c->d_model, c->stream);
        if (values_out) d2h(values_out, c->values + off, sizeof(float) * n * c->d_model, c->stream);
        CX_CUDA(cudaStreamSynchronize(c->stream));
    });
}

// ---- inject (injector.cpp:70-94) ------------------------------------------
namespace {

// Validates like inject() and begin_entry() per token; returns how many tokens
// the reference would append before throwing (err set to the error to throw).
int64_t inject_validate(cx_kvcache* c, int64_t base, int64_t T, int n_layers, int d_model, cx_status* err,
                        std::string* msg) {
    *err = CX_OK;
    if (T < 1) { *err = CX_PRECONDITION_ERROR; *msg = "inject: empty block"; return 0; }
    if (c->entry_open) { *err = CX_SEQUENCING_ERROR; *msg = "inject: river cache has a step in flight"; return 0; }
    if (n_layers != c->n_layers || d_model != c->d_model) {
        *err = CX_PRECONDITION_ERROR;
        *msg = "inject: block shape mismatch";
        return 0;
    }
    for (int64_t t = 0; t < T; ++t) {
        const int64_t p = base + t;
        if (p < 0 || p >= c->max_positions) {
            *err = CX_CAPACITY_ERROR;
            *msg = "position " + std::to_string(p) + " outside max_positions " + std::to_string(c->max_positions);
            return t;
        }
    }
    return T;
}

void inject_apply(cx_kvcache* c, const float* dk, const float* dv, int64_t block_T, int64_t n_ok, int64_t base,
                  cudaStream_t s) {
    const int64_t row0 = (int64_t)c->positions.size();
    kv_grow(c, row0 + n_ok);
    kv_before(c, s);
    // copy tokens [0, n_ok) of every layer: block layout [layer][block_T][d_model]
    if (n_ok == block_T) {
        kv_append_rows(c->keys, c->values, c->capacity, c->n_layers, c->d_model, dk, dv, n_ok, row0, s);
    } else {
        for (int l = 0; l < c->n_layers; ++l)
            kv_append_rows(c->keys + (size_t)l * c->capacity * c->d_model,
                           c->values + (size_t)l * c->capacity * c->d_model, c->capacity, 1, c->d_model,
                           dk + (size_t)l * block_T * c->d_model, dv + (size_t)l * block_T * c->d_model, n_ok, row0, s);
    }
    kv_after(c, s);
    for (int64_t t = 0; t < n_ok; ++t) {
        c->positions.push_back(base + t);
        c->origins.push_back((uint8_t)CX_ORIGIN_INJECTED);
    }
}

}  // namespace

extern "C" cx_status cx_inject_host(cx_kvcache* c, const float* keys, const float* values, int64_t base_position,
                                    int64_t token_count, int n_layers, int d_model, int64_t thought_id,
                                    int64_t stream_position, cx_injection_record* rec) {
    return guard(__func__, [&] {
        if (!c) fail(CX_INVALID_ARGUMENT, "null cache");
        cx_status err;
        std::string msg;
        const int64_t n_ok = inject_validate(c, base_position, token_count, n_layers, d_model, &err, &msg);
        if (n_ok > 0) {
            if (!keys || !values) fail(CX_INVALID_ARGUMENT, "null block");
            cx_ctx* x = default_ctx();
            std::lock_guard<std::mutex> lk(x->mu);
            const size_t n = (size_t)n_layers * token_count * d_model;
            x->arena.reserve(2 * sizeof(float) * n + 1024);
            x->arena.reset();
            float* dk = x->arena.take<float>(n);
            float* dv = x->arena.take<float>(n);
            h2d(dk, keys, sizeof(float) * n, c->stream);
            h2d(dv, values, sizeof(float) * n, c->stream);
            inject_apply(c, dk, dv, token_count, n_ok, base_position, c->stream);
            CX_CUDA(cudaStreamSynchronize(c->stream));
        }
        if (err != CX_OK) fail(err, msg);
        if (rec) {
            rec->thought_id = thought_id;
            rec->token_count = token_count;
            rec->virtual_position_base = base_position;
            rec->applied_at_stream_position = stream_position;
        }
    });
}

extern "C" cx_status cx_inject_dev(cx_kvcache* c, const float* keys, const float* values, int64_t base_position,
                                   int64_t token_count, int n_layers, int d_model, int64_t thought_id,
                                   int64_t stream_position, cx_injection_record* rec, void* stream) {
    return guard(__func__, [&] {
        if (!c) fail(CX_INVALID_ARGUMENT, "null cache");
        cx_status err;
        std::string msg;
        const int64_t n_ok = inject_validate(c, base_position, token_count, n_layers, d_model, &err, &msg);
        if (n_ok > 0) {
            if (!keys || !values) fail(CX_INVALID_ARGUMENT, "null block");
            cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
            inject_apply(c, keys, values, token_count, n_ok, base_position, s);
        }
        if (err != CX_OK) fail(err, msg);
        if (rec) {
            rec->thought_id = thought_id;
            rec->token_count = token_count;
            rec->virtual_position_base = base_position;
            rec->applied_at_stream_position = stream_position;
        }
    });
}

// ============================================================================
// cache-level select_landmarks (synapse.cpp:286-320) + snapshots + buffer
// ============================================================================
struct cx_snapshot {
    std::atomic<int> refs{1};
    uint64_t version = 0;
    int64_t source_length = 0;
    int k_configured = 0;
    int n_layers = 0;
    int d_model = 0;
    int64_t count = 0;
    std::vector<int64_t> positions;
    std::vector<double> scores;
    float* keys = nullptr;  // device [n_layers][count][d_model]
    float* values = nullptr;
    ~cx_snapshot() {
        if (keys) cudaFree(keys);
        if (values) cudaFree(values);
    }
};

extern "C" cx_status cx_select_landmarks(const cx_kvcache* kc, const float* query, int64_t query_len, int k,
                                         double lambda, cx_snapshot** out) {
    return guard(__func__, [&] {
        if (k < 1) fail(CX_CONFIG_ERROR, "select_landmarks: k must be >= 1");  // synapse.cpp:288
        if (!kc || !out) fail(CX_INVALID_ARGUMENT, "null cache/out");
        auto snap = std::make_unique<cx_snapshot>();
        const int layer = kc->n_layers - 1;  // :290
        // A1 context_key_cloud (synapse.cpp:48-61): rows with origin == context
        std::vector<int64_t> entry_index;
        entry_index.reserve(kc->positions.size());
        for (size_t i = 0; i < kc->positions.size(); ++i)
            if (kc->origins[i] == (uint8_t)CX_ORIGIN_CONTEXT) entry_index.push_back((int64_t)i);
        const int64_t count = (int64_t)entry_index.size();
        snap->source_length = count;
        snap->k_configured = k;
        snap->n_layers = kc->n_layers;
        snap->d_model = kc->d_model;
        if (count == 0) {  // :298
            *out = snap.release();
            return;
        }
        // attention_scores_points checks (synapse.cpp:67-70)
        if (query_len != kc->d_model) fail(CX_PRECONDITION_ERROR, "attention_scores: query width mismatch");
        if (!query) fail(CX_INVALID_ARGUMENT, "null query");
        cx_ctx* c = default_ctx();
        std::lock_guard<std::mutex> lk(c->mu);
        const int dm = kc->d_model;
        const int take = (int)std::min<int64_t>(k, count);
        const bool dense = (count == (int64_t)kc->positions.size());
        GroupView g{};
        g.G = 1;
        g.L = count;
        g.dim = dm;
        g.gstride = count * dm;
        g.rstride = dm;
        g.P = kc->n_heads;
        g.d_k = kc->d_k;
        g.col_step = kc->d_k;
        ArenaPlan pl;
        pl.take<float>(dense ? 1 : (size_t)count * dm);
        pl.take<int64_t>((size_t)count);
        pl.take<float>((size_t)dm);
        pl.take<double>((size_t)count);
        pl.take<int64_t>((size_t)take);
        pl.take<double>((size_t)take);
        pl.take<int64_t>((size_t)take);
        plan_attention(pl, g);
        plan_select(pl, g, k);
        c->arena.reserve(pl.used);
        c->arena.reset();
        float* cloud = c->arena.take<float>(dense ? 1 : (size_t)count * dm);
        int64_t* d_entries = c->arena.take<int64_t>((size_t)count);
        float* dq = c->arena.take<float>((size_t)dm);
        double* attn = c->arena.take<double>((size_t)count);
        int64_t* rows = c->arena.take<int64_t>((size_t)take);
        double* scores = c->arena.take<double>((size_t)take);
        int64_t* entries_sel = c->arena.take<int64_t>((size_t)take);
        cudaStream_t s = c->stream;
        // order after the cache's pending device work
        CX_CUDA(cudaStreamSynchronize(kc->stream));
        const float* final_keys = kc->keys + (size_t)layer * kc->capacity * dm;
        if (dense) {
            g.X = final_keys;
        } else {
            h2d(d_entries, entry_index.data(), sizeof(int64_t) * count, s);
            GroupView src = g;
            src.X = final_keys;
            src.gstride = kc->capacity * dm;
            gather_rows(src, final_keys, d_entries, (int)count, cloud, s);  // compaction
            g.X = cloud;
        }
        h2d(dq, query, sizeof(float) * dm, s);
        g.Q = dq;
        CX_CUDA(cudaMemsetAsync(c->d_flag, 0, sizeof(int), s));
        const size_t mark = c->arena.used;
        attention_grouped(c, g, attn, s);
        c->arena.used = mark;
        select_grouped(c, g, attn, k, lambda, 0u, rows, scores, s);
        std::vector<int64_t> h_rows((size_t)take);
        snap->scores.resize((size_t)take);
        d2h(h_rows.data(), rows, sizeof(int64_t) * take, s);
        d2h(snap->scores.data(), scores, sizeof(double) * take, s);
        check_flag_and_sync(c);
        // gather the winners' K/V for EVERY layer (synapse.cpp:303-318)
        std::vector<int64_t> h_entries((size_t)take);
        snap->positions.resize((size_t)take);
        for (int s2 = 0; s2 < take; ++s2) {
            h_entries[s2] = entry_index[(size_t)h_rows[s2]];
            snap->positions[s2] = kc->positions[(size_t)h_entries[s2]];
        }
        snap->count = take;
        CX_CUDA(cudaMalloc(&snap->keys, sizeof(float) * (size_t)kc->n_layers * take * dm));
        CX_CUDA(cudaMalloc(&snap->values, sizeof(float) * (size_t)kc->n_layers * take * dm));
        h2d(entries_sel, h_entries.data(), sizeof(int64_t) * take, s);
        GroupView lg{};
        lg.G = kc->n_layers;
        lg.L = kc->capacity;
        lg.dim = dm;
        lg.gstride = kc->capacity * dm;
        lg.rstride = dm;
        // gather_rows indexes rows[g*take + s]; all layers share the same entry list,
        // so gather layer by layer.
        for (int l = 0; l < kc->n_layers; ++l) {
            GroupView one = lg;
            one.G = 1;
            gather_rows(one, kc->keys + (size_t)l * kc->capacity * dm, entries_sel, take,
                        snap->keys + (size_t)l * take * dm, s);
            gather_rows(one, kc->values + (size_t)l * kc->capacity * dm, entries_sel, take,
                        snap->values + (size_t)l * take * dm, s);
        }
        CX_CUDA(cudaStreamSynchronize(s));
        *out = snap.release();
    });
}

extern "C" cx_status cx_snapshot_create(int64_t source_length, int k_configured, int n_layers, int d_model,
                                        int64_t count, const int64_t* positions, const double* scores,
                                        const float* keys, const float* values, cx_snapshot** out) {
    return guard(__func__, [&] {
        if (!out || count < 0 || n_layers < 0 || d_model < 0) fail(CX_INVALID_ARGUMENT, "bad snapshot arguments");
        if (count > 0 && (!positions || !scores || n_layers < 1 || d_model < 1))
            fail(CX_INVALID_ARGUMENT, "snapshot arrays missing");
        auto snap = std::make_unique<cx_snapshot>();
        snap->source_length = source_length;
        snap->k_configured = k_configured;
        snap->n_layers = n_layers;
        snap->d_model = d_model;
        snap->count = count;
        if (count > 0) {
            snap->positions.assign(positions, positions + count);
            snap->scores.assign(scores, scores + count);
            const size_t n = (size_t)n_layers * count * d_model;
            CX_CUDA(cudaMalloc(&snap->keys, sizeof(float) * n));
            CX_CUDA(cudaMalloc(&snap->values, sizeof(float) * n));
            const size_t row = sizeof(float) * d_model;
            for (int l = 0; l < n_layers; ++l) {  // host [entry][layer][d] -> device [layer][entry][d]
                if (keys)
                    CX_CUDA(cudaMemcpy2D(snap->keys + (size_t)l * count * d_model, row, keys + (size_t)l * d_model,
                                         row * n_layers, row, (size_t)count, cudaMemcpyHostToDevice));
                else
                    CX_CUDA(cudaMemset(snap->keys + (size_t)l * count * d_model, 0, row * count));
                if (values)
                    CX_CUDA(cudaMemcpy2D(snap->values + (size_t)l * count * d_model, row, values + (size_t)l * d_model,
                                         row * n_layers, row, (size_t)count, cudaMemcpyHostToDevice));
                else
                    CX_CUDA(cudaMemset(snap->values + (size_t)l * count * d_model, 0, row * count));
            }
        }
        *out = snap.release();
    });
}

extern "C" cx_status cx_snapshot_release(const cx_snapshot* s) {
    return guard(__func__, [&] {
        if (!s) return;
        auto* m = const_cast<cx_snapshot*>(s);
        if (m->refs.fetch_sub(1) == 1) delete m;
    });
}
extern "C" cx_status cx_snapshot_destroy(cx_snapshot* s) { return cx_snapshot_release(s); }
extern "C" uint64_t cx_snapshot_version(const cx_snapshot* s) { return s ? s->version : 0; }
extern "C" int64_t cx_snapshot_source_length(const cx_snapshot* s) { return s ? s->source_length : 0; }
extern "C" int cx_snapshot_k_configured(const cx_snapshot* s) { return s ? s->k_configured : 0; }
extern "C" int cx_snapshot_n_layers(const cx_snapshot* s) { return s ? s->n_layers : 0; }
extern "C" int cx_snapshot_d_model(const cx_snapshot* s) { return s ? s->d_model : 0; }
extern "C" int64_t cx_snapshot_count(const cx_snapshot* s) { return s ? s->count : 0; }
extern "C" const float* cx_snapshot_keys_dev(const cx_snapshot* s) { return s ? s->keys : nullptr; }
extern "C" const float* cx_snapshot_values_dev(const cx_snapshot* s) { return s ? s->values : nullptr; }

extern "C" cx_status cx_snapshot_read(const cx_snapshot* s, int64_t* positions, double* scores, float* keys,
                                      float* values) {
    return guard(__func__, [&] {
        if (!s) fail(CX_INVALID_ARGUMENT, "null snapshot");
        if (positions) std::copy(s->positions.begin(), s->positions.end(), positions);
        if (scores) std::copy(s->scores.begin(), s->scores.end(), scores);
        if ((keys || values) && s->count > 0) {
            // device [layer][entry][d] -> host [entry][layer][d] (LandmarkEntry layout, synapse.hpp:30-35)
            const size_t row = sizeof(float) * s->d_model;
            for (int l = 0; l < s->n_layers; ++l) {
                if (keys)
                    CX_CUDA(cudaMemcpy2D(keys + (size_t)l * s->d_model, row * s->n_layers,
                                         s->keys + (size_t)l * s->count * s->d_model, row, row, (size_t)s->count,
                                         cudaMemcpyDeviceToHost));
                if (values)
                    CX_CUDA(cudaMemcpy2D(values + (size_t)l * s->d_model, row * s->n_layers,
                                         s->values + (size_t)l * s->count * s->d_model, row, row, (size_t)s->count,
                                         cudaMemcpyDeviceToHost));
            }
        }
    });
}

// ---- SynapseBuffer (synapse.cpp:337-362) --------------------------------------
struct cx_synapse_buffer {
    std::mutex mu;
    std::condition_variable cv;
    cx_snapshot* latest = nullptr;
    uint64_t version = 0;
    bool shutdown = false;
};

extern "C" cx_status cx_synapse_buffer_create(cx_synapse_buffer** out) {
    return guard(__func__, [&] {
        if (!out) fail(CX_INVALID_ARGUMENT, "null out");
        *out = new cx_synapse_buffer();
    });
}

extern "C" cx_status cx_synapse_buffer_destroy(cx_synapse_buffer* b) {
    return guard(__func__, [&] {
        if (!b) return;
        if (b->latest) cx_snapshot_release(b->latest);
        delete b;
    });
}

extern "C" cx_status cx_synapse_buffer_push(cx_synapse_buffer* b, cx_snapshot* snap, uint64_t* version) {
    return guard(__func__, [&] {
        if (!b || !snap) fail(CX_INVALID_ARGUMENT, "null buffer/snapshot");
        cx_snapshot* old = nullptr;
        {
            std::lock_guard<std::mutex> lk(b->mu);
            snap->version = ++b->version;
            old = b->latest;
            b->latest = snap;
            if (version) *version = b->version;
            b->cv.notify_all();
        }
        if (old) cx_snapshot_release(old);
    });
}

extern "C" cx_status cx_synapse_buffer_read_latest(cx_synapse_buffer* b, const cx_snapshot** out) {
    return guard(__func__, [&] {
        if (!b || !out) fail(CX_INVALID_ARGUMENT, "null buffer/out");
        std::lock_guard<std::mutex> lk(b->mu);
        if (b->latest) b->latest->refs.fetch_add(1);
        *out = b->latest;
    });
}

extern "C" cx_status cx_synapse_buffer_wait_nonempty(cx_synapse_buffer* b, int64_t timeout_ms, const cx_snapshot** out) {
    return guard(__func__, [&] {
        if (!b || !out) fail(CX_INVALID_ARGUMENT, "null buffer/out");
        std::unique_lock<std::mutex> lk(b->mu);
        b->cv.wait_for(lk, std::chrono::milliseconds(timeout_ms), [&] { return b->latest != nullptr || b->shutdown; });
        if (b->latest) b->latest->refs.fetch_add(1);
        *out = b->latest;
    });
}

extern "C" cx_status cx_synapse_buffer_shutdown(cx_synapse_buffer* b) {
    return guard(__func__, [&] {
        if (!b) fail(CX_INVALID_ARGUMENT, "null buffer");
        std::lock_guard<std::mutex> lk(b->mu);
        b->shutdown = true;
        b->cv.notify_all();
    });
}

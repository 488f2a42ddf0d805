// forward.cu -- the toy transformer's incremental decode step on the device,
// batched across agents: forward_step (model.cpp:175-235)
// for B agents at once, each on its own device KvCache, plus the kernels:: host
// primitives it is built from (matvec, rmsnorm, add_inplace, relu_inplace,
// apply_rope; kernels.cpp:12-62).
//
// Numerics follow the reference: every projection accumulates in fp64 and
// rounds to fp32 once (kernels.cpp:12-26), RMSNorm in fp64 (:28-38), RoPE in
// fp64 (:49-62), attention in fp64 (:103-142), residual adds and ReLU in fp32.
// Sums run as warp trees instead of one sequential chain, so results agree with
// the reference to ~1e-15 relative per op (its own tests allow 1e-6).
//
// Batching: the agents' activations form a matrix, so each projection is one
// launch for all agents (a warp per (agent, output row); the weight rows are read
// once per launch and shared through L1/L2).  Attention splits every (agent, head)
// over 128-entry chunks (partial max / sum / P.V in fp64, then a combine), so a
// river with an 8192-row cache spreads over many CTAs.
#include <cmath>
#include <memory>
#include <vector>

#include "cx_internal.cuh"


namespace cx {
namespace {

constexpr int FW_CHUNK = 128;  // attention entries per CTA

// per agent: its cache arrays and the row the new entry goes to
struct FwAgent {
    float* keys;    // [n_layers][cap][d_model]
    float* values;
    int64_t cap;
    int64_t row;    // entries before this step (the new one is row `row`)
    int64_t position;
    int token;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void fw_embed(const FwAgent* ag, int B, const float* emb, int d, float* x) {
    const int b = blockIdx.x;
    if (b >= B) return;
    for (int i = threadIdx.x; i < d; i += blockDim.x) x[(size_t)b * d + i] = emb[(size_t)ag[b].token * d + i];
}

// out[b] = x[b] * (1 / sqrt(mean(x^2) + eps)) * gain, fp64 (kernels.cpp:28-38); one warp per agent
__global__ void fw_rmsnorm(const float* x, const float* gain, int d, int B, float* out, double eps) {
    const int b = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x & 31;
    if (b >= B) return;
    const float* xb = x + (size_t)b * d;
    double ssq = 0.0;
    for (int i = lane; i < d; i += 32) ssq += (double)xb[i] * (double)xb[i];
    ssq = warp_sum(ssq);
    const double inv = 1.0 / sqrt(ssq / (double)d + eps);
    for (int i = lane; i < d; i += 32) out[(size_t)b * d + i] = (float)((double)xb[i] * inv * (double)gain[i]);
}

// Y[b][r] (op) = sum_c W[r][c] x[b][c] in fp64, rounded once (kernels.cpp:12-26); a warp per
// (b, r).  mode 0: store; 1: store relu; 2: Y += result (the residual add, fp32 like
// kernels.cpp:40-43).  nmat matrices at W + m * mat_stride, outputs at Y + m * y_stride.
__global__ void fw_matvec(const float* W, size_t mat_stride, int nmat, int n_out, int n_in, const float* X, int B,
                          float* Y, size_t y_stride, int mode) {
    const int wpb = blockDim.x / 32;
    const long long item = (long long)blockIdx.x * wpb + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (item >= (long long)nmat * n_out * B) return;
    const int b = (int)(item % B);
    const long long mr = item / B;
    const int r = (int)(mr % n_out), m = (int)(mr / n_out);
    const float* row = W + m * mat_stride + (size_t)r * n_in;
    const float* xb = X + (size_t)b * n_in;
    double acc = 0.0;
    for (int c = lane; c < n_in; c += 32) acc += (double)row[c] * (double)xb[c];
    acc = warp_sum(acc);
    if (lane == 0) {
        float* y = Y + m * y_stride + (size_t)b * n_out + r;
        const float v = (float)acc;
        if (mode == 0) *y = v;
        else if (mode == 1) *y = fmaxf(v, 0.0f);
        else *y = *y + v;
    }
}

// RoPE on q and k (each head's pairs (2j, 2j+1), kernels.cpp:49-62), then the new entry's
// K / V rows into the agent's cache at layer l (model.cpp:142-152 write_layer)
__global__ void fw_rope_append(FwAgent* ag, int B, int l, int n_heads, int d_k, double base, float* q, const float* k,
                               const float* v, float* final_q) {
    const int b = blockIdx.x;
    if (b >= B) return;
    const int d = n_heads * d_k;
    const FwAgent a = ag[b];
    float* kdst = a.keys + ((size_t)l * a.cap + a.row) * d;
    float* vdst = a.values + ((size_t)l * a.cap + a.row) * d;
    for (int e = threadIdx.x; e < d / 2; e += blockDim.x) {
        const int h = e / (d_k / 2), j = e % (d_k / 2);
        const int i0 = h * d_k + 2 * j;
        const double freq = pow(base, -2.0 * j / (double)d_k);
        const double ang = (double)a.position * freq;
        const double c = cos(ang), s = sin(ang);
        const size_t o = (size_t)b * d + i0;
        const double q0 = q[o], q1 = q[o + 1], k0 = k[o], k1 = k[o + 1];
        const float rq0 = (float)(c * q0 - s * q1), rq1 = (float)(s * q0 + c * q1);
        q[o] = rq0;
        q[o + 1] = rq1;
        kdst[i0] = (float)(c * k0 - s * k1);
        kdst[i0 + 1] = (float)(s * k0 + c * k1);
        if (final_q) {
            final_q[o] = rq0;
            final_q[o + 1] = rq1;
        }
    }
    for (int i = threadIdx.x; i < d; i += blockDim.x) vdst[i] = v[(size_t)b * d + i];
}

// attention partials: block (chunk, head, agent) over entries [chunk*128, +128) of rows
// [0, row + 1): m = max score, l = sum exp(s - m), acc = sum exp(s - m) v  (fp64)
__global__ void fw_attend_partial(const FwAgent* ag, int l, int n_heads, int d_k, const float* q, double* part,
                                  int n_chunks) {
    const int ch = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const FwAgent a = ag[b];
    const int64_t n = a.row + 1;
    const int64_t e0 = (int64_t)ch * FW_CHUNK;
    const int d = n_heads * d_k;
    double* out = part + (((size_t)b * n_heads + h) * n_chunks + ch) * (2 + d_k);
    if (e0 >= n) {
        if (threadIdx.x == 0) {
            out[0] = -INFINITY;
            out[1] = 0.0;
        }
        for (int c = threadIdx.x; c < d_k; c += blockDim.x) out[2 + c] = 0.0;
        return;
    }
    __shared__ double w[FW_CHUNK];
    __shared__ double red[FW_CHUNK / 32];
    __shared__ double qs[64];
    const float* kb = a.keys + (size_t)l * a.cap * d + (size_t)h * d_k;
    const float* vb = a.values + (size_t)l * a.cap * d + (size_t)h * d_k;
    for (int c = threadIdx.x; c < d_k; c += blockDim.x) qs[c] = (double)q[(size_t)b * d + h * d_k + c];
    __syncthreads();
    const int t = threadIdx.x;
    const int64_t e = e0 + t;
    const double inv = 1.0 / sqrt((double)d_k);
    double s = -INFINITY;
    if (e < n) {
        const float* kr = kb + (size_t)e * d;
        double dot = 0.0;
        for (int c = 0; c < d_k; ++c) dot += qs[c] * (double)kr[c];
        s = dot * inv;
    }
    double mx = s;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((t & 31) == 0) red[t >> 5] = mx;
    __syncthreads();
    mx = red[0];
    for (int i = 1; i < FW_CHUNK / 32; ++i) mx = fmax(mx, red[i]);
    const double p = e < n ? exp(s - mx) : 0.0;
    w[t] = p;
    __syncthreads();
    double sum = warp_sum(p);
    __syncthreads();
    if ((t & 31) == 0) red[t >> 5] = sum;
    __syncthreads();
    if (t == 0) {
        double acc = 0.0;
        for (int i = 0; i < FW_CHUNK / 32; ++i) acc += red[i];
        out[0] = mx;
        out[1] = acc;
    }
    const int64_t ne = min((int64_t)FW_CHUNK, n - e0);
    for (int c = t; c < d_k; c += blockDim.x) {
        double acc = 0.0;
        for (int64_t j = 0; j < ne; ++j) acc += w[j] * (double)vb[(size_t)(e0 + j) * d + c];
        out[2 + c] = acc;
    }
}

// out[b][h*d_k + c] = (sum_ch acc e^{m_ch - M}) / (sum_ch l e^{m_ch - M}), rounded to fp32
__global__ void fw_attend_combine(int B, int n_heads, int d_k, const double* part, int n_chunks, float* att) {
    const int b = blockIdx.x, h = blockIdx.y;
    if (b >= B) return;
    const double* pp = part + ((size_t)b * n_heads + h) * n_chunks * (2 + d_k);
    double M = -INFINITY;
    for (int ch = 0; ch < n_chunks; ++ch) M = fmax(M, pp[(size_t)ch * (2 + d_k)]);
    double L = 0.0;
    for (int ch = 0; ch < n_chunks; ++ch) {
        const double m = pp[(size_t)ch * (2 + d_k)];
        if (m > -INFINITY) L += pp[(size_t)ch * (2 + d_k) + 1] * exp(m - M);
    }
    for (int c = threadIdx.x; c < d_k; c += blockDim.x) {
        double acc = 0.0;
        for (int ch = 0; ch < n_chunks; ++ch) {
            const double m = pp[(size_t)ch * (2 + d_k)];
            if (m > -INFINITY) acc += pp[(size_t)ch * (2 + d_k) + 2 + c] * exp(m - M);
        }
        att[(size_t)b * n_heads * d_k + h * d_k + c] = (float)(acc / L);
    }
}

__global__ void fw_elementwise(float* x, const float* y, int64_t n, int op) {  // 0: x += y, 1: relu
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = op == 0 ? x[i] + y[i] : fmaxf(x[i], 0.0f);
}

__global__ void fw_rope_vec(float* v, int n, int64_t position, double base) {  // kernels.cpp:49-62
    for (int j = threadIdx.x; 2 * j < n; j += blockDim.x) {
        const double freq = pow(base, -2.0 * j / (double)n);
        const double ang = (double)position * freq;
        const double c = cos(ang), s = sin(ang);
        const double x0 = v[2 * j], x1 = v[2 * j + 1];
        v[2 * j] = (float)(c * x0 - s * x1);
        v[2 * j + 1] = (float)(s * x0 + c * x1);
    }
}

void matvec_launch(const float* W, size_t mat_stride, int nmat, int n_out, int n_in, const float* X, int B, float* Y,
                   size_t y_stride, int mode, cudaStream_t s) {
    const long long items = (long long)nmat * n_out * B;
    const int wpb = 8;
    fw_matvec<<<(unsigned)((items + wpb - 1) / wpb), 32 * wpb, 0, s>>>(W, mat_stride, nmat, n_out, n_in, X, B, Y,
                                                                        y_stride, mode);
    check_launch("fw_matvec");
}

}  // namespace
}  // namespace cx

using namespace cx;

extern "C" size_t cx_weights_flat_floats(int n_layers, int d_model, int vocab_size) {
    const size_t d = (size_t)d_model, dff = 4 * d;
    return 2 * (size_t)vocab_size * d + d + (size_t)n_layers * (2 * d + 4 * d * d + 2 * dff * d);
}

extern "C" cx_status cx_weights_create(int n_layers, int n_heads, int d_model, int d_k, int vocab_size,
                                       int64_t max_positions, double rope_base, const float* flat, cx_weights** out) {
    return guard([&] {
        if (!flat || !out) fail(CX_INVALID_ARGUMENT, "null flat/out");
        if (n_layers < 1 || n_heads < 1 || d_k < 1 || n_heads * d_k != d_model || d_k % 2 != 0 || vocab_size < 1 ||
            d_k > 64)
            fail(CX_CONFIG_ERROR, "weights: inconsistent dimensions (d_model = n_heads * d_k, even d_k <= 64)");
        auto w = std::make_unique<cx_weights>();
        w->n_layers = n_layers;
        w->n_heads = n_heads;
        w->d_model = d_model;
        w->d_k = d_k;
        w->vocab = vocab_size;
        w->max_positions = max_positions;
        w->rope_base = rope_base;
        const size_t d = (size_t)d_model, dff = 4 * d;
        w->per_layer = 2 * d + 4 * d * d + 2 * dff * d;
        w->emb = 0;
        w->layers = (size_t)vocab_size * d;
        w->final_norm = w->layers + (size_t)n_layers * w->per_layer;
        w->unemb = w->final_norm + d;
        const size_t n = cx_weights_flat_floats(n_layers, d_model, vocab_size);
        CX_CUDA(cudaMalloc(&w->buf, n * sizeof(float)));
        CX_CUDA(cudaMemcpy(w->buf, flat, n * sizeof(float), cudaMemcpyHostToDevice));
        *out = w.release();
    });
}

extern "C" cx_status cx_weights_destroy(cx_weights* w) {
    return guard([&] {
        if (!w) return;
        if (w->buf) cudaFree(w->buf);
        delete w;
    });
}

// forward_step (model.cpp:175-235) for n_agents agents, agent i on caches[i].
extern "C" cx_status cx_forward_step_dev(cx_ctx* c, const cx_weights* w, int n_agents, cx_kvcache* const* caches,
                                         const int* tokens, const int64_t* positions, float* logits, float* hidden,
                                         float* final_query, void* stream) {
    return guard([&] {
        if (!c || !w) fail(CX_INVALID_ARGUMENT, "null ctx/weights");
        if (n_agents < 0) fail(CX_INVALID_ARGUMENT, "negative agent count");
        if (n_agents == 0) return;
        if (!caches || !tokens || !positions) fail(CX_INVALID_ARGUMENT, "null caches/tokens/positions");
        const int B = n_agents, d = w->d_model, dff = 4 * d, L = w->n_layers;
        // the reference's checks, in its order, for every agent before any work (model.cpp:177-183,
        // then begin_entry :124-140)
        for (int b = 0; b < B; ++b) {
            cx_kvcache* kc = caches[b];
            if (!kc) fail(CX_INVALID_ARGUMENT, "null cache");
            if (kc->n_layers != L || kc->d_model != d || kc->n_heads != w->n_heads)
                fail(CX_PRECONDITION_ERROR, "forward_step: cache shape does not match the weights");
            if (tokens[b] < 0 || tokens[b] >= w->vocab) fail(CX_PRECONDITION_ERROR, "token id outside vocabulary");
            if (kc->entry_open) fail(CX_SEQUENCING_ERROR, "forward_step with an open cache entry");
            if (positions[b] >= w->max_positions) fail(CX_CAPACITY_ERROR, "position beyond max_positions");
            if (positions[b] < 0 || positions[b] >= kc->max_positions)
                fail(CX_CAPACITY_ERROR, "position " + std::to_string(positions[b]) + " outside max_positions " +
                                            std::to_string(kc->max_positions));
            if (positions[b] <= kc->last_context_position)
                fail(CX_PRECONDITION_ERROR, "context positions must be strictly increasing");
            for (int b2 = 0; b2 < b; ++b2)
                if (caches[b2] == kc) fail(CX_INVALID_ARGUMENT, "forward_step: a cache appears twice in the batch");
        }
        cudaStream_t s = (cudaStream_t)stream;
        std::vector<FwAgent> ag((size_t)B);
        int64_t max_rows = 1;
        for (int b = 0; b < B; ++b) {
            cx_kvcache* kc = caches[b];
            const int64_t row = (int64_t)kc->positions.size();
            kv_grow(kc, row + 1);
            kv_before(kc, s);
            ag[(size_t)b] = FwAgent{kc->keys, kc->values, kc->capacity, row, positions[b], tokens[b]};
            max_rows = std::max(max_rows, row + 1);
        }
        const int n_chunks = (int)((max_rows + FW_CHUNK - 1) / FW_CHUNK);
        ArenaPlan pl;
        pl.take<FwAgent>((size_t)B);
        pl.take<float>((size_t)B * d);          // x
        pl.take<float>((size_t)B * d);          // normed
        pl.take<float>((size_t)3 * B * d);      // q, k, v
        pl.take<float>((size_t)B * d);          // att
        pl.take<float>((size_t)B * dff);        // ff
        pl.take<double>((size_t)B * w->n_heads * n_chunks * (2 + w->d_k));
        c->arena.reserve(pl.used);
        c->arena.reset();
        FwAgent* dag = c->arena.take<FwAgent>((size_t)B);
        float* x = c->arena.take<float>((size_t)B * d);
        float* nrm = c->arena.take<float>((size_t)B * d);
        float* qkv = c->arena.take<float>((size_t)3 * B * d);
        float* att = c->arena.take<float>((size_t)B * d);
        float* ff = c->arena.take<float>((size_t)B * dff);
        double* part = c->arena.take<double>((size_t)B * w->n_heads * n_chunks * (2 + w->d_k));
        CX_CUDA(cudaMemcpyAsync(dag, ag.data(), sizeof(FwAgent) * B, cudaMemcpyHostToDevice, s));
        const float* W = w->buf;
        fw_embed<<<B, 128, 0, s>>>(dag, B, W + w->emb, d, x);
        check_launch("fw_embed");
        const unsigned nb_warps = (unsigned)((B + 7) / 8);
        for (int l = 0; l < L; ++l) {
            fw_rmsnorm<<<nb_warps, 256, 0, s>>>(x, W + w->attn_norm(l), d, B, nrm, 1e-5);
            check_launch("fw_rmsnorm");
            // q, k, v: three matrices in one launch (wq, wk, wv are consecutive)
            matvec_launch(W + w->wq(l), (size_t)d * d, 3, d, d, nrm, B, qkv, (size_t)B * d, 0, s);
            fw_rope_append<<<B, 128, 0, s>>>(dag, B, l, w->n_heads, w->d_k, w->rope_base, qkv, qkv + (size_t)B * d,
                                             qkv + (size_t)2 * B * d, l == L - 1 ? final_query : nullptr);
            check_launch("fw_rope_append");
            fw_attend_partial<<<dim3((unsigned)n_chunks, (unsigned)w->n_heads, (unsigned)B), FW_CHUNK, 0, s>>>(
                dag, l, w->n_heads, w->d_k, qkv, part, n_chunks);
            check_launch("fw_attend_partial");
            fw_attend_combine<<<dim3((unsigned)B, (unsigned)w->n_heads), 64, 0, s>>>(B, w->n_heads, w->d_k, part,
                                                                                    n_chunks, att);
            check_launch("fw_attend_combine");
            matvec_launch(W + w->wo(l), 0, 1, d, d, att, B, x, 0, 2, s);                 // x += Wo att
            fw_rmsnorm<<<nb_warps, 256, 0, s>>>(x, W + w->mlp_norm(l), d, B, nrm, 1e-5);
            check_launch("fw_rmsnorm");
            matvec_launch(W + w->w_in(l), 0, 1, dff, d, nrm, B, ff, 0, 1, s);            // relu(W_in n)
            matvec_launch(W + w->w_out(l), 0, 1, d, dff, ff, B, x, 0, 2, s);             // x += W_out ff
        }
        float* hid = hidden ? hidden : nrm;
        fw_rmsnorm<<<nb_warps, 256, 0, s>>>(x, W + w->final_norm, d, B, hid, 1e-5);
        check_launch("fw_rmsnorm");
        if (logits) matvec_launch(W + w->unemb, 0, 1, w->vocab, d, hid, B, logits, 0, 0, s);
        // the entry is complete at every layer (end_entry)
        for (int b = 0; b < B; ++b) {
            cx_kvcache* kc = caches[b];
            kv_after(kc, s);
            kc->positions.push_back(positions[b]);
            kc->origins.push_back((uint8_t)CX_ORIGIN_CONTEXT);
            kc->last_context_position = positions[b];
            kc->context_count += 1;
        }
    });
}

extern "C" cx_status cx_device_alloc(size_t bytes, void** out) {
    return guard([&] {
        if (!out) fail(CX_INVALID_ARGUMENT, "null out");
        *out = nullptr;
        if (bytes) CX_CUDA(cudaMalloc(out, bytes));
    });
}

extern "C" cx_status cx_device_free(void* p) {
    return guard([&] {
        if (p) CX_CUDA(cudaFree(p));
    });
}

extern "C" cx_status cx_device_read(void* host, const void* dev, size_t bytes, void* stream) {
    return guard([&] {
        if (!bytes) return;
        if (!host || !dev) fail(CX_INVALID_ARGUMENT, "null pointer");
        CX_CUDA(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
        CX_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    });
}

// ---- kernels:: host primitives (kernels.cpp:12-62) on the device ---------------
namespace {
template <class F>
void on_default(F&& f) {
    cx_ctx* c = default_ctx();
    std::lock_guard<std::mutex> lk(c->mu);
    f(c);
    CX_CUDA(cudaStreamSynchronize(c->stream));
}
}  // namespace

extern "C" cx_status cx_matvec(const float* w, int n_out, int n_in, const float* x, float* y) {
    return guard([&] {
        if (n_out < 0 || n_in < 0) fail(CX_PRECONDITION_ERROR, "matvec: bad shape");
        if (n_out == 0) return;
        if (!w || !x || !y) fail(CX_INVALID_ARGUMENT, "null pointer");
        on_default([&](cx_ctx* c) {
            ArenaPlan pl;
            pl.take<float>((size_t)n_out * n_in);
            pl.take<float>((size_t)n_in);
            pl.take<float>((size_t)n_out);
            c->arena.reserve(pl.used);
            c->arena.reset();
            float* dw = c->arena.take<float>((size_t)n_out * n_in);
            float* dx = c->arena.take<float>((size_t)n_in);
            float* dy = c->arena.take<float>((size_t)n_out);
            CX_CUDA(cudaMemcpyAsync(dw, w, sizeof(float) * n_out * n_in, cudaMemcpyHostToDevice, c->stream));
            CX_CUDA(cudaMemcpyAsync(dx, x, sizeof(float) * n_in, cudaMemcpyHostToDevice, c->stream));
            matvec_launch(dw, 0, 1, n_out, n_in, dx, 1, dy, 0, 0, c->stream);
            CX_CUDA(cudaMemcpyAsync(y, dy, sizeof(float) * n_out, cudaMemcpyDeviceToHost, c->stream));
        });
    });
}

extern "C" cx_status cx_rmsnorm(const float* x, const float* gain, int64_t n, double eps, float* out) {
    return guard([&] {
        if (n < 1) fail(CX_PRECONDITION_ERROR, "rmsnorm: empty input");
        if (!x || !gain || !out) fail(CX_INVALID_ARGUMENT, "null pointer");
        on_default([&](cx_ctx* c) {
            ArenaPlan pl;
            pl.take<float>((size_t)n);
            pl.take<float>((size_t)n);
            pl.take<float>((size_t)n);
            c->arena.reserve(pl.used);
            c->arena.reset();
            float* dx = c->arena.take<float>((size_t)n);
            float* dg = c->arena.take<float>((size_t)n);
            float* dout = c->arena.take<float>((size_t)n);
            CX_CUDA(cudaMemcpyAsync(dx, x, sizeof(float) * n, cudaMemcpyHostToDevice, c->stream));
            CX_CUDA(cudaMemcpyAsync(dg, gain, sizeof(float) * n, cudaMemcpyHostToDevice, c->stream));
            fw_rmsnorm<<<1, 32, 0, c->stream>>>(dx, dg, (int)n, 1, dout, eps);
            check_launch("fw_rmsnorm");
            CX_CUDA(cudaMemcpyAsync(out, dout, sizeof(float) * n, cudaMemcpyDeviceToHost, c->stream));
        });
    });
}

extern "C" cx_status cx_elementwise(float* x, const float* y, int64_t n, int op) {
    return guard([&] {
        if (n < 0 || (op != 0 && op != 1)) fail(CX_INVALID_ARGUMENT, "elementwise: bad arguments");
        if (n == 0) return;
        if (!x || (op == 0 && !y)) fail(CX_INVALID_ARGUMENT, "null pointer");
        on_default([&](cx_ctx* c) {
            ArenaPlan pl;
            pl.take<float>((size_t)n);
            pl.take<float>((size_t)n);
            c->arena.reserve(pl.used);
            c->arena.reset();
            float* dx = c->arena.take<float>((size_t)n);
            float* dy = c->arena.take<float>((size_t)n);
            CX_CUDA(cudaMemcpyAsync(dx, x, sizeof(float) * n, cudaMemcpyHostToDevice, c->stream));
            if (op == 0) CX_CUDA(cudaMemcpyAsync(dy, y, sizeof(float) * n, cudaMemcpyHostToDevice, c->stream));
            fw_elementwise<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, c->stream>>>(dx, dy, n, op);
            check_launch("fw_elementwise");
            CX_CUDA(cudaMemcpyAsync(x, dx, sizeof(float) * n, cudaMemcpyDeviceToHost, c->stream));
        });
    });
}

extern "C" cx_status cx_apply_rope(float* v, int64_t n, int64_t position, double rope_base) {
    return guard([&] {
        if (n < 0 || n % 2 != 0) fail(CX_PRECONDITION_ERROR, "apply_rope: odd length");
        if (n == 0) return;
        if (!v) fail(CX_INVALID_ARGUMENT, "null pointer");
        on_default([&](cx_ctx* c) {
            c->arena.reserve(sizeof(float) * n + 256);
            c->arena.reset();
            float* dv = c->arena.take<float>((size_t)n);
            CX_CUDA(cudaMemcpyAsync(dv, v, sizeof(float) * n, cudaMemcpyHostToDevice, c->stream));
            fw_rope_vec<<<1, 128, 0, c->stream>>>(dv, (int)n, position, rope_base);
            check_launch("fw_rope_vec");
            CX_CUDA(cudaMemcpyAsync(v, dv, sizeof(float) * n, cudaMemcpyDeviceToHost, c->stream));
        });
    });
}

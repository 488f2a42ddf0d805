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
#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstring>
#include <memory>
#include <vector>

#include "cx_internal.cuh"


namespace cx {
namespace {

constexpr int FW_CHUNK = 128;      // attention entries per CTA
#ifndef CX_FW_MAX_B
#define CX_FW_MAX_B 32
#endif
constexpr int FW_MAX_B = CX_FW_MAX_B;  // agents per launch (kernel-parameter batch; larger batches are split)
constexpr int FW_MAX_CHUNKS = 1024;  // attention chunks per (agent, head): 131072 rows

// per agent: its cache arrays and the row the new entry goes to
struct FwAgent {
    float* keys;    // [n_layers][cap][d_model]
    float* values;
    int64_t cap;
    int64_t row;    // entries before this step (the new one is row `row`)
    int64_t position;
    int token;
};
// the batch is copied to device memory once per step from a pinned staging slot (a pageable
// cudaMemcpyAsync would synchronise the stream), so the kernels' parameters do not change from
// token to token and the step replays as one CUDA graph
struct FwBatch {
    int B;
    FwAgent a[FW_MAX_B];
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Programmatic dependent launch inside forward_step: every launch after the first one may
// start while its predecessor drains; it waits for the predecessor's results here (a no-op
// for a normally launched grid) and lets its own successor launch right away.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__global__ void fw_embed(const FwBatch* __restrict__ Pd, const float* emb, int d, float* x) {
    const FwBatch& P = *Pd;
    const int b = blockIdx.x;
    if (b >= P.B) return;
    for (int i = threadIdx.x; i < d; i += blockDim.x) x[(size_t)b * d + i] = emb[(size_t)P.a[b].token * d + i];
}

// 1 / sqrt(mean(x^2) + eps) of one agent's row, by a full warp (kernels.cpp:28-38)
__device__ __forceinline__ double warp_rms_inv(const float* xb, int d, double eps) {
    double ssq = 0.0;
#pragma unroll 4
    for (int i = threadIdx.x & 31; i < d; i += 32) ssq += (double)xb[i] * (double)xb[i];
    ssq = warp_sum(ssq);
    return 1.0 / sqrt(ssq / (double)d + eps);
}

// out[b] = x[b] * (1 / sqrt(mean(x^2) + eps)) * gain, fp64 (kernels.cpp:28-38); one warp per agent
__global__ void fw_rmsnorm(const float* x, const float* gain, int d, int B, float* out, double eps) {
    pdl_enter();
    const int b = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x & 31;
    if (b >= B) return;
    const float* xb = x + (size_t)b * d;
    const double inv = warp_rms_inv(xb, d, eps);
    for (int i = lane; i < d; i += 32) out[(size_t)b * d + i] = (float)((double)xb[i] * inv * (double)gain[i]);
}

// Y[b][r] (op) = sum_c W[r][c] x[b][c] in fp64, rounded once (kernels.cpp:12-26); a warp per
// (b, r).  mode 0: store; 1: store relu; 2: Y += result (the residual add, fp32 like
// kernels.cpp:40-43).  gain != NULL: x is rmsnorm(x) * gain first (fused; the normed value is
// rounded to fp32 exactly as the separate rmsnorm's output).
__global__ void fw_matvec(const float* W, int n_out, int n_in, const float* X, int B, float* Y, int mode,
                          const float* gain, double eps) {
    pdl_enter();
    const int wpb = blockDim.x / 32;
    const long long item = (long long)blockIdx.x * wpb + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (item >= (long long)n_out * B) return;
    const int b = (int)(item % B), r = (int)(item / B);
    const float* row = W + (size_t)r * n_in;
    const float* xb = X + (size_t)b * n_in;
    double acc = 0.0;
    if (gain) {
        const double inv = warp_rms_inv(xb, n_in, eps);
#pragma unroll 4
        for (int c = lane; c < n_in; c += 32)
            acc += (double)row[c] * (double)(float)((double)xb[c] * inv * (double)gain[c]);
    } else {
#pragma unroll 4
        for (int c = lane; c < n_in; c += 32) acc += (double)row[c] * (double)xb[c];
    }
    acc = warp_sum(acc);
    if (lane == 0) {
        float* y = Y + (size_t)b * n_out + r;
        const float v = (float)acc;
        if (mode == 0) *y = v;
        else if (mode == 1) *y = fmaxf(v, 0.0f);
        else *y = *y + v;
    }
}

// q, k, v = W{q,k,v} rmsnorm(x) for one rotation pair (2e, 2e+1) per warp, then RoPE on q and
// k (kernels.cpp:49-62) and the new entry's K / V into the agent's cache at layer l
// (model.cpp:142-152 write_layer); q (rotated) -> qbuf, and final_q at the last layer.
__global__ void fw_qkv_rope(const FwBatch* __restrict__ Pd, int l, const float* Wq, int n_heads, int d_k,
                            double base, const float* x, const float* gain, double eps, float* qbuf, float* final_q) {
    pdl_enter();
    const FwBatch& P = *Pd;
    const int d = n_heads * d_k;
    const int wpb = blockDim.x / 32, lane = threadIdx.x & 31;
    const long long item = (long long)blockIdx.x * wpb + threadIdx.x / 32;
    if (item >= (long long)(d / 2) * P.B) return;
    const int b = (int)(item % P.B), e = (int)(item / P.B);
    const int i0 = 2 * e;
    const float* xb = x + (size_t)b * d;
    const double inv = warp_rms_inv(xb, d, eps);
    const size_t dd = (size_t)d * d;
    double acc[6] = {0, 0, 0, 0, 0, 0};
    // unrolled: the 6 weight rows' loads of several column steps are in flight together
    // (a rolled loop waited one memory round trip per step); the per-lane order is unchanged
#pragma unroll 4
    for (int c = lane; c < d; c += 32) {
        const double xn = (double)(float)((double)xb[c] * inv * (double)gain[c]);
#pragma unroll
        for (int m = 0; m < 3; ++m) {
            acc[2 * m] += (double)Wq[m * dd + (size_t)i0 * d + c] * xn;
            acc[2 * m + 1] += (double)Wq[m * dd + (size_t)(i0 + 1) * d + c] * xn;
        }
    }
#pragma unroll
    for (int m = 0; m < 6; ++m) acc[m] = warp_sum(acc[m]);
    if (lane == 0) {
        const FwAgent& a = P.a[b];
        const int j = e % (d_k / 2);
        const double freq = pow(base, -2.0 * j / (double)d_k);
        const double ang = (double)a.position * freq;
        const double cs = cos(ang), sn = sin(ang);
        const double q0 = (float)acc[0], q1 = (float)acc[1], k0 = (float)acc[2], k1 = (float)acc[3];
        const float rq0 = (float)(cs * q0 - sn * q1), rq1 = (float)(sn * q0 + cs * q1);
        const size_t o = (size_t)b * d + i0;
        qbuf[o] = rq0;
        qbuf[o + 1] = rq1;
        if (final_q) {
            final_q[o] = rq0;
            final_q[o + 1] = rq1;
        }
        float* kdst = a.keys + ((size_t)l * a.cap + a.row) * d;
        float* vdst = a.values + ((size_t)l * a.cap + a.row) * d;
        kdst[i0] = (float)(cs * k0 - sn * k1);
        kdst[i0 + 1] = (float)(sn * k0 + cs * k1);
        vdst[i0] = (float)acc[4];
        vdst[i0 + 1] = (float)acc[5];
    }
}

// rows [e0, e0 + ne) x columns [0, d_k) of a head's K or V -> tile (coalesced; float4 when aligned)
__device__ __forceinline__ void stage_tile(float (*tile)[65], const float* src, int64_t e0, int ne, int d, int d_k) {
    if ((d_k & 3) == 0) {
        const int q4 = d_k / 4;
        for (int i = threadIdx.x; i < ne * q4; i += blockDim.x) {
            const int r = i / q4, c = (i % q4) * 4;
            const float4 v = __ldg(reinterpret_cast<const float4*>(src + (size_t)(e0 + r) * d + c));
            tile[r][c] = v.x;
            tile[r][c + 1] = v.y;
            tile[r][c + 2] = v.z;
            tile[r][c + 3] = v.w;
        }
    } else {
        for (int i = threadIdx.x; i < ne * d_k; i += blockDim.x) {
            const int r = i / d_k, c = i % d_k;
            tile[r][c] = __ldg(src + (size_t)(e0 + r) * d + c);
        }
    }
}

// attention (kernels.cpp:103-142) of one (chunk of 128 entries, head, agent) per CTA over rows
// [0, row + 1): K / V tiles staged through shared memory with coalesced loads; the chunk's
// partial (max m, sum l of e^{s-m}, sum e^{s-m} v, all fp64) goes to `part`, and the last CTA
// of the (agent, head) to finish combines every chunk (no second launch).
__global__ void __launch_bounds__(256) fw_attend(const FwBatch* __restrict__ Pd, int l, int n_heads, int d_k,
                                                 const float* q, double* part, unsigned* counters, int n_chunks,
                                                 float* att, const char* pf, size_t pf_bytes) {
    // the weights the next launches read (this layer's Wo / W_in / W_out, the next layer's
    // Wq / Wk / Wv: contiguous) -> L2 while the cache rows stream: the matvecs that follow then
    // start from L2 hits instead of HBM round trips.  Read-only data, so no ordering with the
    // predecessor is needed.
    if (threadIdx.x == 0 && pf_bytes) {
        const size_t ncta = (size_t)gridDim.x * gridDim.y * gridDim.z;
        const size_t cid = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        const size_t share = ((pf_bytes + ncta - 1) / ncta + 255) & ~(size_t)255;
        for (size_t o = cid * share; o < min(pf_bytes, (cid + 1) * share); o += 16384) {
            const uint32_t n = (uint32_t)min((size_t)16384, min(pf_bytes, (cid + 1) * share) - o);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf + o), "r"(n) : "memory");
        }
    }
    pdl_enter();
    const FwBatch& P = *Pd;
    const int ch = blockIdx.x, h = blockIdx.y, b = blockIdx.z, t = threadIdx.x;
    const FwAgent& a = P.a[b];
    const int64_t n = a.row + 1;
    const int my_chunks = (int)((n + FW_CHUNK - 1) / FW_CHUNK);
    if (ch >= my_chunks) return;
    const int d = n_heads * d_k;
    const int64_t e0 = (int64_t)ch * FW_CHUNK;
    const int ne = (int)min((int64_t)FW_CHUNK, n - e0);
    __shared__ float tile[FW_CHUNK][65];
    __shared__ double qs[64];
    __shared__ double w[FW_CHUNK];
    __shared__ double red[8];
    __shared__ double pacc[4][64];
    __shared__ double sc[FW_MAX_CHUNKS];
    __shared__ int last;
    const float* kb = a.keys + (size_t)l * a.cap * d + (size_t)h * d_k;
    const float* vb = a.values + (size_t)l * a.cap * d + (size_t)h * d_k;
    if (t < d_k) qs[t] = (double)q[(size_t)b * d + h * d_k + t];
    // full chunks at d_k = 64: every K and V load of the chunk is issued up front (8 + 8 float4
    // per thread); V waits in registers until the K tile has been consumed (a load -> store
    // loop per tile was one DRAM round trip per iteration)
    const bool fast = ne == FW_CHUNK && d_k == 64 && blockDim.x == 256;
    constexpr int FV = FW_CHUNK * 16 / 256;
    float4 vreg[FV];
    if (fast) {
        float4 kreg[FV];
#pragma unroll
        for (int i = 0; i < FV; ++i) {
            const int idx = t + 256 * i, r = idx >> 4, c = (idx & 15) * 4;
            kreg[i] = __ldg(reinterpret_cast<const float4*>(kb + (size_t)(e0 + r) * d + c));
            vreg[i] = __ldg(reinterpret_cast<const float4*>(vb + (size_t)(e0 + r) * d + c));
        }
#pragma unroll
        for (int i = 0; i < FV; ++i) {
            const int idx = t + 256 * i, r = idx >> 4, c = (idx & 15) * 4;
            tile[r][c] = kreg[i].x;
            tile[r][c + 1] = kreg[i].y;
            tile[r][c + 2] = kreg[i].z;
            tile[r][c + 3] = kreg[i].w;
        }
    } else {
        stage_tile(tile, kb, e0, ne, d, d_k);
    }
    __syncthreads();
    const double inv = 1.0 / sqrt((double)d_k);
    double s = -INFINITY;
    if (t < ne) {
        double dot = 0.0;  // the reference's order: c = 0 .. d_k - 1
        for (int c = 0; c < d_k; ++c) dot += qs[c] * (double)tile[t][c];
        s = dot * inv;
    }
    double mx = s;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((t & 31) == 0) red[t >> 5] = mx;
    __syncthreads();
    mx = red[0];
    for (int i = 1; i < FW_CHUNK / 32; ++i) mx = fmax(mx, red[i]);
    const double p = t < ne ? exp(s - mx) : 0.0;
    if (t < FW_CHUNK) w[t] = p;
    __syncthreads();  // every thread has read red[] and the K tile
    const double ps = warp_sum(p);
    if ((t & 31) == 0) red[t >> 5] = ps;
    if (fast) {
#pragma unroll
        for (int i = 0; i < FV; ++i) {
            const int idx = t + 256 * i, r = idx >> 4, c = (idx & 15) * 4;
            tile[r][c] = vreg[i].x;
            tile[r][c + 1] = vreg[i].y;
            tile[r][c + 2] = vreg[i].z;
            tile[r][c + 3] = vreg[i].w;
        }
    } else {
        stage_tile(tile, vb, e0, ne, d, d_k);
    }
    __syncthreads();
    double* out = part + (((size_t)b * n_heads + h) * n_chunks + ch) * (2 + d_k);
    {
        const int c = t % 64, qtr = t / 64;  // 4 row quarters x 64 columns
        if (c < d_k) {
            double acc = 0.0;
            const int r1 = min(ne, (qtr + 1) * (FW_CHUNK / 4));
            for (int r = qtr * (FW_CHUNK / 4); r < r1; ++r) acc += w[r] * (double)tile[r][c];
            pacc[qtr][c] = acc;
        }
    }
    __syncthreads();
    if (t < d_k) out[2 + t] = ((pacc[0][t] + pacc[1][t]) + pacc[2][t]) + pacc[3][t];
    if (t == 0) {
        double acc = 0.0;
        for (int i = 0; i < FW_CHUNK / 32; ++i) acc += red[i];
        out[0] = mx;
        out[1] = acc;
    }
    __threadfence();
    __syncthreads();
    if (t == 0) last = atomicAdd(&counters[b * n_heads + h], 1u) == (unsigned)(my_chunks - 1);
    __syncthreads();
    if (!last) return;
    // the combine: out = (sum_ch acc e^{m_ch - M}) / (sum_ch l e^{m_ch - M}), rounded to fp32
    __threadfence();
    const double* pp = part + ((size_t)b * n_heads + h) * n_chunks * (2 + d_k);
    double M = -INFINITY;
    for (int i = t; i < my_chunks; i += blockDim.x) M = fmax(M, __ldcg(pp + (size_t)i * (2 + d_k)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmax(M, __shfl_xor_sync(0xffffffffu, M, o));
    __syncthreads();
    if ((t & 31) == 0) red[t >> 5] = M;
    __syncthreads();
    M = red[0];
    for (int i = 1; i < 8; ++i) M = fmax(M, red[i]);
    double Ls = 0.0;
    for (int i = t; i < my_chunks; i += blockDim.x) {
        const double f = exp(__ldcg(pp + (size_t)i * (2 + d_k)) - M);
        sc[i] = f;
        Ls += __ldcg(pp + (size_t)i * (2 + d_k) + 1) * f;
    }
    Ls = warp_sum(Ls);
    __syncthreads();
    if ((t & 31) == 0) red[t >> 5] = Ls;
    __syncthreads();
    Ls = 0.0;
    for (int i = 0; i < 8; ++i) Ls += red[i];
    {
        const int c = t % 64, qtr = t / 64;
        if (c < d_k) {
            // the chunks' partial P.V in order, 8 L2 loads in flight per batch
            double acc = 0.0;
            for (int i0 = qtr; i0 < my_chunks; i0 += 32) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int i = i0 + 4 * u;
                    v[u] = i < my_chunks ? __ldcg(pp + (size_t)i * (2 + d_k) + 2 + c) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (i0 + 4 * u < my_chunks) acc += v[u] * sc[i0 + 4 * u];
            }
            pacc[qtr][c] = acc;
        }
    }
    __syncthreads();
    if (t < d_k)
        att[(size_t)b * d + h * d_k + t] = (float)((((pacc[0][t] + pacc[1][t]) + pacc[2][t]) + pacc[3][t]) / Ls);
    if (t == 0) counters[b * n_heads + h] = 0u;  // ready for the next launch
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

// a launch that may overlap its stream predecessor's tail (the kernel calls pdl_enter first)
template <class... KArgs, class... Args>
void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, bool pdl, Args&&... args) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = grid;
    lc.blockDim = block;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = pdl ? 1 : 0;
    CX_CUDA(cudaLaunchKernelEx(&lc, k, std::forward<Args>(args)...));
    count_launch();
}

void matvec_launch(const float* W, int n_out, int n_in, const float* X, int B, float* Y, int mode, cudaStream_t s,
                   const float* gain = nullptr, double eps = 1e-5, bool pdl = false) {
    const long long items = (long long)n_out * B;
    const int wpb = 8;
    if (pdl) {
        launch_pdl(fw_matvec, dim3((unsigned)((items + wpb - 1) / wpb)), dim3(32 * wpb), s, true, W, n_out, n_in, X, B,
                   Y, mode, gain, eps);
        return;
    }
    fw_matvec<<<(unsigned)((items + wpb - 1) / wpb), 32 * wpb, 0, s>>>(W, n_out, n_in, X, B, Y, mode, gain, eps);
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
    return guard(__func__, [&] {
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
    return guard(__func__, [&] {
        if (!w) return;
        if (w->buf) cudaFree(w->buf);
        delete w;
    });
}

namespace cx {
namespace {
// one launch sequence for nb <= FW_MAX_B agents (checks already done)
void forward_batch(cx_ctx* c, const cx_weights* w, int nb, cx_kvcache* const* caches, const int* tokens,
                   const int64_t* positions, float* logits, float* hidden, float* final_query, cudaStream_t s) {
    const int d = w->d_model, dff = 4 * d, L = w->n_layers;
    FwBatch P{};
    P.B = nb;
    int64_t max_rows = 1;
    for (int b = 0; b < nb; ++b) {
        cx_kvcache* kc = caches[b];
        const int64_t row = (int64_t)kc->positions.size();
        kv_grow(kc, row + 1);
        kv_before(kc, s);
        P.a[b] = FwAgent{kc->keys, kc->values, kc->capacity, row, positions[b], tokens[b]};
        max_rows = std::max(max_rows, row + 1);
    }
    const int n_chunks = (int)((max_rows + FW_CHUNK - 1) / FW_CHUNK);
    if (n_chunks > FW_MAX_CHUNKS) fail(CX_CAPACITY_ERROR, "forward_step: cache beyond 131072 entries");
    const int n_cnt = nb * w->n_heads;
    if (c->fw_counters_n < n_cnt) {  // zeroed once; every attention launch leaves them zero
        if (c->fw_counters) CX_CUDA(cudaFree(c->fw_counters));
        c->fw_counters = nullptr;
        c->fw_counters_n = 0;
        CX_CUDA(cudaMalloc(&c->fw_counters, sizeof(unsigned) * FW_MAX_B * 64));
        CX_CUDA(cudaMemset(c->fw_counters, 0, sizeof(unsigned) * FW_MAX_B * 64));
        c->fw_counters_n = FW_MAX_B * 64;
        if (n_cnt > c->fw_counters_n) fail(CX_CONFIG_ERROR, "forward_step: more than 64 heads");
    }
    ArenaPlan pl;
    pl.take<float>((size_t)nb * d);          // x
    pl.take<float>((size_t)nb * d);          // q (rotated)
    pl.take<float>((size_t)nb * d);          // att
    pl.take<float>((size_t)nb * d);          // hidden scratch
    pl.take<float>((size_t)nb * dff);        // ff
    pl.take<double>((size_t)nb * w->n_heads * n_chunks * (2 + w->d_k));
    c->arena.reserve(pl.used);
    c->arena.reset();
    float* x = c->arena.take<float>((size_t)nb * d);
    float* qb = c->arena.take<float>((size_t)nb * d);
    float* att = c->arena.take<float>((size_t)nb * d);
    float* hs = c->arena.take<float>((size_t)nb * d);
    float* ff = c->arena.take<float>((size_t)nb * dff);
    double* part = c->arena.take<double>((size_t)nb * w->n_heads * n_chunks * (2 + w->d_k));
    const float* W = w->buf;
    // the batch -> device memory (a pinned staging slot whose previous copy has long completed)
    if (!c->fw_dev) {
        CX_CUDA(cudaMalloc(&c->fw_dev, sizeof(FwBatch)));
        CX_CUDA(cudaMallocHost(&c->fw_host, sizeof(FwBatch) * cx_ctx::kFwRing));
        for (cudaEvent_t& e : c->fw_ev) CX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    {
        const int slot = c->fw_slot;
        c->fw_slot = (slot + 1) % cx_ctx::kFwRing;
        CX_CUDA(cudaEventSynchronize(c->fw_ev[slot]));
        FwBatch* hp = static_cast<FwBatch*>(c->fw_host) + slot;
        const size_t bytes = offsetof(FwBatch, a) + sizeof(FwAgent) * (size_t)nb;
        std::memcpy(hp, &P, bytes);
        CX_CUDA(cudaMemcpyAsync(c->fw_dev, hp, bytes, cudaMemcpyHostToDevice, s));
        CX_CUDA(cudaEventRecord(c->fw_ev[slot], s));
    }
    const FwBatch* Pd = static_cast<const FwBatch*>(c->fw_dev);
    float* hid = hidden ? hidden : hs;
    auto issue = [&]() {
        fw_embed<<<nb, 128, 0, s>>>(Pd, W + w->emb, d, x);
        check_launch("fw_embed");
        const long long pairs = (long long)(d / 2) * nb;
        for (int l = 0; l < L; ++l) {
            // rmsnorm + q/k/v + RoPE + the cache append, one launch
            // every launch after fw_embed is a programmatic dependent of the previous one
            launch_pdl(fw_qkv_rope, dim3((unsigned)((pairs + 7) / 8)), dim3(256), s, true, Pd, l, W + w->wq(l),
                       w->n_heads, w->d_k, w->rope_base, (const float*)x, W + w->attn_norm(l), 1e-5, qb,
                       l == L - 1 ? final_query : nullptr);
            // L2 prefetch of [Wo(l), Wv(l + 1) end): this layer's output / MLP weights and the next
            // layer's q / k / v weights (the last layer: up to the end of its block)
            const size_t pf0 = w->wo(l), pf1 = l + 1 < L ? w->wo(l + 1) : w->attn_norm(l) + w->per_layer;
            launch_pdl(fw_attend, dim3((unsigned)n_chunks, (unsigned)w->n_heads, (unsigned)nb), dim3(256), s, true, Pd,
                       l, w->n_heads, w->d_k, (const float*)qb, part, c->fw_counters, n_chunks, att,
                       reinterpret_cast<const char*>(W + pf0),
                       (reinterpret_cast<uintptr_t>(W + pf0) & 15) ? 0 : ((pf1 - pf0) * sizeof(float) & ~(size_t)15));
            matvec_launch(W + w->wo(l), d, d, att, nb, x, 2, s, nullptr, 1e-5, true);                // x += Wo att
            matvec_launch(W + w->w_in(l), dff, d, x, nb, ff, 1, s, W + w->mlp_norm(l), 1e-5, true);  // relu(W_in rmsnorm(x))
            matvec_launch(W + w->w_out(l), d, dff, ff, nb, x, 2, s, nullptr, 1e-5, true);            // x += W_out ff
        }
        launch_pdl(fw_rmsnorm, dim3((unsigned)((nb + 7) / 8)), dim3(256), s, true, (const float*)x, W + w->final_norm,
                   d, nb, hid, 1e-5);
        if (logits) matvec_launch(W + w->unemb, w->vocab, d, hid, nb, logits, 0, s, nullptr, 1e-5, true);
    };
    // replay the captured sequence (a named stream that is not already being captured)
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    const bool named = s != nullptr && s != cudaStreamLegacy && s != cudaStreamPerThread;
    if (named) CX_CUDA(cudaStreamIsCapturing(s, &cs));
    if (!named || cs != cudaStreamCaptureStatusNone) {
        issue();
    } else {
        // everything the captured launches bake in: the weights' device buffer and shape (a
        // destroyed cx_weights' address may come back with other contents), scratch and outputs
        const uintptr_t shape = (uintptr_t)L | (uintptr_t)d << 8 | (uintptr_t)w->vocab << 24 | (uintptr_t)w->n_heads << 48;
        const void* key[10] = {w, w->buf, reinterpret_cast<const void*>(shape), x, part, logits, hidden,
                               final_query, c->fw_counters, c->fw_dev};
        cx_ctx::FwGraph* hit = nullptr;
        for (auto& fg : c->fw_graphs)
            if (fg.nb == nb && fg.n_chunks == n_chunks && std::equal(key, key + 10, fg.key)) hit = &fg;
        if (!hit) {
            // the launches issue() makes (counted per replay, not at capture)
            const uint64_t n = 2 + 5 * (uint64_t)L + (logits ? 1 : 0);
            CX_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            cudaGraph_t graph = nullptr;
            try {
                issue();
            } catch (...) {
                cudaStreamEndCapture(s, &graph);
                if (graph) cudaGraphDestroy(graph);
                throw;
            }
            CX_CUDA(cudaStreamEndCapture(s, &graph));
            count_launch(0 - n);  // captured, not launched: counted at each replay
            cudaGraphExec_t exec = nullptr;
            const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
            cudaGraphDestroy(graph);
            if (ie != cudaSuccess) fail(CX_DEVICE_ERROR, std::string("forward_step graph: ") + cudaGetErrorString(ie));
            if (c->fw_graphs.size() >= 16) {  // oldest out
                cudaGraphExecDestroy(c->fw_graphs.front().exec);
                c->fw_graphs.erase(c->fw_graphs.begin());
            }
            cx_ctx::FwGraph fg{};
            std::copy(key, key + 10, fg.key);
            fg.nb = nb;
            fg.n_chunks = n_chunks;
            fg.exec = exec;
            fg.launches = n;
            c->fw_graphs.push_back(fg);
            hit = &c->fw_graphs.back();
        }
        CX_CUDA(cudaGraphLaunch(hit->exec, s));
        count_launch(hit->launches);
    }
    // the entry is complete at every layer (end_entry)
    for (int b = 0; b < nb; ++b) {
        cx_kvcache* kc = caches[b];
        kv_after(kc, s);
        kc->positions.push_back(positions[b]);
        kc->origins.push_back((uint8_t)CX_ORIGIN_CONTEXT);
        kc->last_context_position = positions[b];
        kc->context_count += 1;
    }
}
}  // namespace
}  // namespace cx

// forward_step (model.cpp:175-235) for n_agents agents, agent i on caches[i].
extern "C" cx_status cx_forward_step_dev(cx_ctx* c, const cx_weights* w, int n_agents, cx_kvcache* const* caches,
                                         const int* tokens, const int64_t* positions, float* logits, float* hidden,
                                         float* final_query, void* stream) {
    return guard(__func__, [&] {
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
        for (int b0 = 0; b0 < B; b0 += FW_MAX_B) {
            const int nb = std::min(FW_MAX_B, B - b0);
            forward_batch(c, w, nb, caches + b0, tokens + b0, positions + b0,
                          logits ? logits + (size_t)b0 * w->vocab : nullptr, hidden ? hidden + (size_t)b0 * d : nullptr,
                          final_query ? final_query + (size_t)b0 * d : nullptr, s);
        }
        (void)dff;
    });
}

extern "C" cx_status cx_device_alloc(size_t bytes, void** out) {
    return guard(__func__, [&] {
        if (!out) fail(CX_INVALID_ARGUMENT, "null out");
        *out = nullptr;
        if (bytes) CX_CUDA(cudaMalloc(out, bytes));
    });
}

extern "C" cx_status cx_device_free(void* p) {
    return guard(__func__, [&] {
        if (p) CX_CUDA(cudaFree(p));
    });
}

extern "C" cx_status cx_device_read(void* host, const void* dev, size_t bytes, void* stream) {
    return guard(__func__, [&] {
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
    return guard(__func__, [&] {
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
            matvec_launch(dw, n_out, n_in, dx, 1, dy, 0, c->stream);
            CX_CUDA(cudaMemcpyAsync(y, dy, sizeof(float) * n_out, cudaMemcpyDeviceToHost, c->stream));
        });
    });
}

extern "C" cx_status cx_rmsnorm(const float* x, const float* gain, int64_t n, double eps, float* out) {
    return guard(__func__, [&] {
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
    return guard(__func__, [&] {
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
    return guard(__func__, [&] {
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

// attend_kernels.cu -- decode attention against the shared synapse (SURVEY.md
// §8(a) A9) and the KV append used by Referential Injection (A10/A11).
//
// attend_fp64: the reference-shaped kernels::attend (kernels.cpp:103-142) for
//   the drop-in call, fp64 scores/softmax/accumulation (reference tolerance
//   1e-6, test_kernels.cpp:159-160).
// decode_step: one decode step of N agents.  For every (agent, layer, q-head)
//   the agent's cache is [k synapse rows of its KV head || private tail rows],
//   exactly what run_agent builds by copying the snapshot (scheduler.cpp:
//   245-262) -- here the synapse is shared, not copied.  The new token's K/V
//   is appended to the private tail first (fused), then attended, fp32
//   accumulate (north_star tolerance 1e-3 relative).
#include <climits>

#include "cx_internal.cuh"

namespace cx {

namespace {

template <class T, class Op>
__device__ __forceinline__ T warp_all(T v, Op op) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ---- attend_fp64: one block per head ---------------------------------------
__global__ void attend_fp64_kernel(const float* __restrict__ q, const float* __restrict__ keys,
                                   const float* __restrict__ values, int64_t n, int H, int dk,
                                   double inv_sqrt_dk, double* __restrict__ w, float* __restrict__ out) {
    __shared__ double red[32];
    const int h = blockIdx.x;
    const int dm = H * dk;
    double* wh = w + (int64_t)h * n;
    const float* qh = q + (int64_t)h * dk;
    double m = -INFINITY;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
        const float* kj = keys + j * dm + (int64_t)h * dk;
        double dot = 0.0;
        for (int c = 0; c < dk; ++c) dot = __dadd_rn(dot, __dmul_rn((double)qh[c], (double)kj[c]));
        const double s = __dmul_rn(dot, inv_sqrt_dk);
        wh[j] = s;
        m = (m < s) ? s : m;
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    m = warp_all(m, [](double a, double b) { return (a < b) ? b : a; });
    if (lane == 0) red[wid] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double mm = red[0];
        for (int i = 1; i < nw; ++i) mm = (mm < red[i]) ? red[i] : mm;
        red[0] = mm;
    }
    __syncthreads();
    m = red[0];
    __syncthreads();
    double acc = 0.0;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
        const double e = exp(__dsub_rn(wh[j], m));
        wh[j] = e;
        acc = __dadd_rn(acc, e);
    }
    acc = warp_all(acc, [](double a, double b) { return __dadd_rn(a, b); });
    if (lane == 0) red[wid] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < nw; ++i) s = __dadd_rn(s, red[i]);
        red[0] = s;
    }
    __syncthreads();
    const double sum = red[0];
    for (int c = threadIdx.x; c < dk; c += blockDim.x) {
        double a = 0.0;
        for (int64_t j = 0; j < n; ++j)  // reference order over entries
            a = __dadd_rn(a, __dmul_rn(wh[j], (double)values[j * dm + (int64_t)h * dk + c]));
        out[(int64_t)h * dk + c] = (float)__ddiv_rn(a, sum);
    }
}

// ---- batched decode step (fp32) ----------------------------------------------
// grid.x = n_layers * n_kv; grid.y = agent chunks.  blockDim = apb * qpg warps:
// warp (a_slot, hh) handles q-head g*qpg+hh of the a_slot-th agent of the batch.
// Shared memory: synapse K,V of this (layer, kv head) [k][d_k+1] (padded, so
// lane-per-row dot products and lane-per-column mixes are conflict-free),
// per-agent-slot tail K,V [t_cap+1][d_k+1], per-warp q and probabilities.
struct DecodeSmem {
    size_t ks, vs, tk, tv, qv, pw, total;
};

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline DecodeSmem decode_layout(int k_syn, int t_rows, int dk, int apb, int warps,
                                                    int n_max) {
    DecodeSmem L;
    const size_t pitch = (size_t)dk + 1;
    size_t o = 0;
    L.ks = o; o = al16(o + sizeof(float) * (size_t)k_syn * pitch);
    L.vs = o; o = al16(o + sizeof(float) * (size_t)k_syn * pitch);
    L.tk = o; o = al16(o + sizeof(float) * (size_t)apb * t_rows * pitch);
    L.tv = o; o = al16(o + sizeof(float) * (size_t)apb * t_rows * pitch);
    L.qv = o; o = al16(o + sizeof(float) * (size_t)warps * dk);
    L.pw = o; o = al16(o + sizeof(float) * (size_t)warps * n_max);
    L.total = o;
    return L;
}

__global__ void __launch_bounds__(256) decode_step_kernel(cx_decode_batch b, int apb, int agents_per_cta,
                                                         float inv_sqrt_dk, int* flag) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int tlen_s[8];  // rows each agent of the batch attends (apb <= 8)
    const int qpg = b.n_q / b.n_kv;
    const int lh = blockIdx.x;
    const int l = lh / b.n_kv, g = lh % b.n_kv;
    const int dk = b.d_k, pitch = dk + 1;
    const int t_rows = b.t_cap + 1;
    const int warps = apb * qpg;
    const int n_max = b.k_syn + t_rows;
    const DecodeSmem lay = decode_layout(b.k_syn, t_rows, dk, apb, warps, n_max);
    float* Ks = reinterpret_cast<float*>(smem + lay.ks);
    float* Vs = reinterpret_cast<float*>(smem + lay.vs);
    float* Tk = reinterpret_cast<float*>(smem + lay.tk);
    float* Tv = reinterpret_cast<float*>(smem + lay.tv);
    float* Qv = reinterpret_cast<float*>(smem + lay.qv);
    float* Pw = reinterpret_cast<float*>(smem + lay.pw);
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int a_slot = warp / qpg, hh = warp % qpg;

    // synapse rows of this (layer, kv head): loaded once, reused by every agent
    const float* sk = b.syn_keys + (size_t)lh * b.k_syn * dk;
    const float* sv = b.syn_values + (size_t)lh * b.k_syn * dk;
    for (int e = tid; e < b.k_syn * dk; e += nt) {
        const int j = e / dk, c = e % dk;
        Ks[j * pitch + c] = __ldg(sk + e);
        Vs[j * pitch + c] = __ldg(sv + e);
    }

    const int a_begin = blockIdx.y * agents_per_cta;
    const int a_end = min(b.n_agents, a_begin + agents_per_cta);
    for (int a0 = a_begin; a0 < a_end; a0 += apb) {
        __syncthreads();  // previous batch done with tails / synapse staged
        // stage private tails (+ append the new row) for the apb agents of this batch
        for (int s = 0; s < apb; ++s) {
            const int a = a0 + s;
            if (a >= a_end) break;
            int len = __ldg(b.tail_len + a);  // validated like decode_tc (FLAG_TAIL_RANGE)
            const bool len_ok = len >= 0 && len <= b.t_cap - (b.new_keys ? 1 : 0);
            if (!len_ok) {
                if (tid == 0) atomicOr(flag, FLAG_TAIL_RANGE);
                len = len < 0 ? 0 : b.t_cap - (b.new_keys ? 1 : 0);
            }
            if (tid == 0) tlen_s[s] = len_ok ? len + (b.new_keys ? 1 : 0) : len;  // rows attended
            const size_t toff = ((((size_t)a * b.n_layers + l) * b.n_kv + g) * b.t_cap) * dk;
            float* tk = Tk + (size_t)s * t_rows * pitch;
            float* tv = Tv + (size_t)s * t_rows * pitch;
            for (int e = tid; e < len * dk; e += nt) {
                const int j = e / dk, c = e % dk;
                tk[j * pitch + c] = __ldg(b.tail_keys + toff + e);
                tv[j * pitch + c] = __ldg(b.tail_values + toff + e);
            }
            if (b.new_keys && len_ok) {
                const size_t noff = (((size_t)a * b.n_layers + l) * b.n_kv + g) * dk;
                for (int c = tid; c < dk; c += nt) {
                    const float nk = __ldg(b.new_keys + noff + c), nv = __ldg(b.new_values + noff + c);
                    tk[len * pitch + c] = nk;
                    tv[len * pitch + c] = nv;
                    b.tail_keys[toff + (size_t)len * dk + c] = nk;  // append into the private cache
                    b.tail_values[toff + (size_t)len * dk + c] = nv;
                }
            }
        }
        __syncthreads();
        const int a = a0 + a_slot;
        if (a < a_end) {
            const int h = g * qpg + hh;
            const int tn = tlen_s[a_slot];
            const int n = b.k_syn + tn;
            const size_t qoff = (((size_t)a * b.n_layers + l) * b.n_q + h) * dk;
            float* qv = Qv + (size_t)warp * dk;
            float* pw = Pw + (size_t)warp * n_max;
            for (int c = lane; c < dk; c += 32) qv[c] = __ldg(b.q + qoff + c);
            __syncwarp();
            const float* tk = Tk + (size_t)a_slot * t_rows * pitch;
            const float* tv = Tv + (size_t)a_slot * t_rows * pitch;
            float m = -INFINITY;
            for (int j = lane; j < n; j += 32) {
                const float* kr = (j < b.k_syn) ? Ks + j * pitch : tk + (j - b.k_syn) * pitch;
                float d0 = 0.f, d1 = 0.f;
                int c = 0;
                for (; c + 2 <= dk; c += 2) {
                    d0 = fmaf(qv[c], kr[c], d0);
                    d1 = fmaf(qv[c + 1], kr[c + 1], d1);
                }
                if (c < dk) d0 = fmaf(qv[c], kr[c], d0);
                const float s = (d0 + d1) * inv_sqrt_dk;
                pw[j] = s;
                m = fmaxf(m, s);
            }
            m = warp_all(m, [](float x, float y) { return fmaxf(x, y); });
            float sum = 0.f;
            for (int j = lane; j < n; j += 32) {
                const float e = __expf(pw[j] - m);
                pw[j] = e;
                sum += e;
            }
            sum = warp_all(sum, [](float x, float y) { return x + y; });
            __syncwarp();
            const float inv = 1.0f / sum;
            for (int c = lane; c < dk; c += 32) {
                float acc0 = 0.f, acc1 = 0.f;
                int j = 0;
                for (; j + 2 <= b.k_syn; j += 2) {
                    acc0 = fmaf(pw[j], Vs[j * pitch + c], acc0);
                    acc1 = fmaf(pw[j + 1], Vs[(j + 1) * pitch + c], acc1);
                }
                for (; j < b.k_syn; ++j) acc0 = fmaf(pw[j], Vs[j * pitch + c], acc0);
                for (int t = 0; t < tn; ++t) acc1 = fmaf(pw[b.k_syn + t], tv[t * pitch + c], acc1);
                b.out[qoff + c] = (acc0 + acc1) * inv;
            }
        }
    }
}

// ---- decode v2: warp per agent, register-tiled (d_k = 64, <= 8 q-heads / KV head) ----
// CTA = one (layer, KV head) and a contiguous agent range; the synapse K (rows
// padded to 68 floats: conflict-free per-lane row reads) and V are staged once
// and reused by every agent of the range.  Each warp owns one agent at a time:
//   scores  lane j holds keys j, j+32, ... for all q-heads of the group
//           (QPG x 6 accumulators; q broadcast from shared memory, K rows as float4);
//           private rows are read straight from global memory (lane per row);
//   softmax per q-head with warp shuffles, unnormalised weights to shared memory;
//   mix     lane owns output dims (2 lane, 2 lane + 1): synapse V from shared
//           memory, private V rows coalesced from global memory.
// The new token's K/V is appended to the private rows first (fused).
constexpr int DV2_DK = 64;
constexpr int DV2_MAXQ = 8;
constexpr int DV2_KPL = 6;       // synapse keys per lane (k_syn <= 192)
constexpr int DV2_KPITCH = 68;
constexpr int DV2_WARPS = 16;

struct DecodeV2Smem {
    size_t ks, vs, qs, ps, total;
    int pstride;
};

__host__ __device__ inline DecodeV2Smem decode_v2_layout(int k_syn, int t_cap) {
    DecodeV2Smem L;
    L.pstride = ((k_syn + t_cap + 3) / 4) * 4;
    size_t o = 0;
    L.ks = o; o = al16(o + sizeof(float) * (size_t)k_syn * DV2_KPITCH);
    L.vs = o; o = al16(o + sizeof(float) * (size_t)k_syn * DV2_DK);
    L.qs = o; o = al16(o + sizeof(float) * (size_t)DV2_WARPS * DV2_MAXQ * DV2_DK);
    L.ps = o; o = al16(o + sizeof(float) * (size_t)DV2_WARPS * DV2_MAXQ * L.pstride);
    L.total = o;
    return L;
}

template <int QPG>
__global__ void __launch_bounds__(DV2_WARPS * 32, 1) decode_v2_kernel(cx_decode_batch b, int agents_per_cta,
                                                                    float scale, int* flag) {
    extern __shared__ __align__(16) unsigned char smem[];
    const DecodeV2Smem lay = decode_v2_layout(b.k_syn, b.t_cap);
    float* Ks = reinterpret_cast<float*>(smem + lay.ks);
    float* Vs = reinterpret_cast<float*>(smem + lay.vs);
    const int lh = blockIdx.x;
    const int l = lh / b.n_kv, g = lh % b.n_kv;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ks = b.k_syn;
    float* Qw = reinterpret_cast<float*>(smem + lay.qs) + warp * DV2_MAXQ * DV2_DK;
    float* Pw = reinterpret_cast<float*>(smem + lay.ps) + warp * DV2_MAXQ * lay.pstride;

    // stage the synapse rows of this (layer, KV head)
    const float4* sk4 = reinterpret_cast<const float4*>(b.syn_keys + (size_t)lh * ks * DV2_DK);
    const float4* sv4 = reinterpret_cast<const float4*>(b.syn_values + (size_t)lh * ks * DV2_DK);
    for (int e = tid; e < ks * (DV2_DK / 4); e += blockDim.x) {
        const int j = e / (DV2_DK / 4), c4 = e % (DV2_DK / 4);
        reinterpret_cast<float4*>(Ks + j * DV2_KPITCH)[c4] = __ldg(sk4 + e);
        reinterpret_cast<float4*>(Vs)[e] = __ldg(sv4 + e);
    }
    __syncthreads();

    const int a_begin = blockIdx.y * agents_per_cta;
    const int a_end = min(b.n_agents, a_begin + agents_per_cta);
    const bool app_all = b.new_keys != nullptr;
    for (int a = a_begin + warp; a < a_end; a += DV2_WARPS) {
        int len = __ldg(b.tail_len + a);  // validated like decode_tc (FLAG_TAIL_RANGE)
        const bool len_ok = len >= 0 && len <= b.t_cap - (app_all ? 1 : 0);
        if (!len_ok) {
            if (lane == 0) atomicOr(flag, FLAG_TAIL_RANGE);
            len = len < 0 ? 0 : b.t_cap - (app_all ? 1 : 0);
        }
        const bool app = app_all && len_ok;
        const int nt = len + (app ? 1 : 0);
        const size_t toff = ((((size_t)a * b.n_layers + l) * b.n_kv + g) * b.t_cap) * DV2_DK;
        const size_t noff = (((size_t)a * b.n_layers + l) * b.n_kv + g) * DV2_DK;
        const size_t qoff = (((size_t)a * b.n_layers + l) * b.n_q + (size_t)g * QPG) * DV2_DK;
        const float* tk = b.tail_keys + toff;
        const float* tv = b.tail_values + toff;
        // q-heads of this group -> shared (coalesced), append the new row (fused)
        for (int e = lane; e < QPG * DV2_DK / 4; e += 32)
            reinterpret_cast<float4*>(Qw)[e] = __ldg(reinterpret_cast<const float4*>(b.q + qoff) + e);
        if (app && lane < 16) {
            reinterpret_cast<float4*>(b.tail_keys + toff + (size_t)len * DV2_DK)[lane] =
                __ldg(reinterpret_cast<const float4*>(b.new_keys + noff) + lane);
            reinterpret_cast<float4*>(b.tail_values + toff + (size_t)len * DV2_DK)[lane] =
                __ldg(reinterpret_cast<const float4*>(b.new_values + noff) + lane);
        }
        __syncwarp();
        // ---- scores: synapse keys lane + 32 i, private row lane (+32) ----
        float acc[DV2_KPL][QPG];
        float acct[2][QPG];
#pragma unroll
        for (int i = 0; i < DV2_KPL; ++i)
#pragma unroll
            for (int h = 0; h < QPG; ++h) acc[i][h] = 0.f;
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int h = 0; h < QPG; ++h) acct[i][h] = 0.f;
        const float* trow0 = (app && lane == len) ? b.new_keys + noff : tk + (size_t)lane * DV2_DK;
        const float* trow1 = (app && lane + 32 == len) ? b.new_keys + noff : tk + (size_t)(lane + 32) * DV2_DK;
#pragma unroll 2
        for (int c4 = 0; c4 < DV2_DK / 4; ++c4) {
            float4 qv[QPG];
#pragma unroll
            for (int h = 0; h < QPG; ++h) qv[h] = reinterpret_cast<const float4*>(Qw + h * DV2_DK)[c4];
#pragma unroll
            for (int i = 0; i < DV2_KPL; ++i) {
                const int j = lane + 32 * i;
                if (j < ks) {
                    const float4 kv = reinterpret_cast<const float4*>(Ks + j * DV2_KPITCH)[c4];
#pragma unroll
                    for (int h = 0; h < QPG; ++h) {
                        acc[i][h] = fmaf(qv[h].x, kv.x, acc[i][h]);
                        acc[i][h] = fmaf(qv[h].y, kv.y, acc[i][h]);
                        acc[i][h] = fmaf(qv[h].z, kv.z, acc[i][h]);
                        acc[i][h] = fmaf(qv[h].w, kv.w, acc[i][h]);
                    }
                }
            }
            if (lane < nt) {
                const float4 kv = __ldg(reinterpret_cast<const float4*>(trow0) + c4);
#pragma unroll
                for (int h = 0; h < QPG; ++h) {
                    acct[0][h] = fmaf(qv[h].x, kv.x, acct[0][h]);
                    acct[0][h] = fmaf(qv[h].y, kv.y, acct[0][h]);
                    acct[0][h] = fmaf(qv[h].z, kv.z, acct[0][h]);
                    acct[0][h] = fmaf(qv[h].w, kv.w, acct[0][h]);
                }
            }
            if (lane + 32 < nt) {
                const float4 kv = __ldg(reinterpret_cast<const float4*>(trow1) + c4);
#pragma unroll
                for (int h = 0; h < QPG; ++h) {
                    acct[1][h] = fmaf(qv[h].x, kv.x, acct[1][h]);
                    acct[1][h] = fmaf(qv[h].y, kv.y, acct[1][h]);
                    acct[1][h] = fmaf(qv[h].z, kv.z, acct[1][h]);
                    acct[1][h] = fmaf(qv[h].w, kv.w, acct[1][h]);
                }
            }
        }
        // ---- softmax per q-head (max, exp, sum over k_syn + nt keys) ----
        float inv[QPG];
#pragma unroll
        for (int h = 0; h < QPG; ++h) {
            float m = -INFINITY;
#pragma unroll
            for (int i = 0; i < DV2_KPL; ++i)
                if (lane + 32 * i < ks) m = fmaxf(m, acc[i][h] * scale);
            if (lane < nt) m = fmaxf(m, acct[0][h] * scale);
            if (lane + 32 < nt) m = fmaxf(m, acct[1][h] * scale);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            float s = 0.f;
            float* ph = Pw + h * lay.pstride;
#pragma unroll
            for (int i = 0; i < DV2_KPL; ++i) {
                const int j = lane + 32 * i;
                if (j < ks) {
                    const float e = __expf(acc[i][h] * scale - m);
                    ph[j] = e;
                    s += e;
                }
            }
            if (lane < nt) {
                const float e = __expf(acct[0][h] * scale - m);
                ph[ks + lane] = e;
                s += e;
            }
            if (lane + 32 < nt) {
                const float e = __expf(acct[1][h] * scale - m);
                ph[ks + lane + 32] = e;
                s += e;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            inv[h] = 1.0f / s;
        }
        __syncwarp();
        // ---- mix: lane owns dims 2 lane, 2 lane + 1 ----
        float2 o[QPG];
#pragma unroll
        for (int h = 0; h < QPG; ++h) o[h] = make_float2(0.f, 0.f);
        int j = 0;
        for (; j + 4 <= ks; j += 4) {
            float4 p4[QPG];
#pragma unroll
            for (int h = 0; h < QPG; ++h) p4[h] = reinterpret_cast<const float4*>(Pw + h * lay.pstride + j)[0];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float2 v = reinterpret_cast<const float2*>(Vs + (j + u) * DV2_DK)[lane];
#pragma unroll
                for (int h = 0; h < QPG; ++h) {
                    const float pw = u == 0 ? p4[h].x : u == 1 ? p4[h].y : u == 2 ? p4[h].z : p4[h].w;
                    o[h].x = fmaf(pw, v.x, o[h].x);
                    o[h].y = fmaf(pw, v.y, o[h].y);
                }
            }
        }
        for (; j < ks; ++j) {
            const float2 v = reinterpret_cast<const float2*>(Vs + j * DV2_DK)[lane];
#pragma unroll
            for (int h = 0; h < QPG; ++h) {
                const float pw = Pw[h * lay.pstride + j];
                o[h].x = fmaf(pw, v.x, o[h].x);
                o[h].y = fmaf(pw, v.y, o[h].y);
            }
        }
        for (int t = 0; t < nt; ++t) {
            const float* vrow = (app && t == len) ? b.new_values + noff : tv + (size_t)t * DV2_DK;
            const float2 v = __ldg(reinterpret_cast<const float2*>(vrow) + lane);
#pragma unroll
            for (int h = 0; h < QPG; ++h) {
                const float pw = Pw[h * lay.pstride + ks + t];
                o[h].x = fmaf(pw, v.x, o[h].x);
                o[h].y = fmaf(pw, v.y, o[h].y);
            }
        }
#pragma unroll
        for (int h = 0; h < QPG; ++h)
            reinterpret_cast<float2*>(b.out + qoff + (size_t)h * DV2_DK)[lane] = make_float2(o[h].x * inv[h], o[h].y * inv[h]);
        __syncwarp();  // Qw / Pw reuse by the next agent of this warp
    }
}

// ---- KV append: [n_layers][T][d_model] block into [n_layers][cap][d_model] --
// ---- gate (gate.cpp:27-61): cosine of the main model's hidden state and a side
// agent's thought, one thread per pair; the three fp64 sums run sequentially in the
// reference's order with explicit roundings (no FMA contraction), so scores are bitwise.
__global__ void gate_kernel(const float* __restrict__ h, int64_t hs, const float* __restrict__ t, int64_t ts,
                            int64_t n, int dim, double theta, double* __restrict__ score,
                            uint8_t* __restrict__ accepted, uint8_t* __restrict__ degenerate) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* a = h + i * hs;
    const float* c = t + i * ts;
    double dot = 0.0, na = 0.0, nb = 0.0;
    for (int k = 0; k < dim; ++k) {
        const double x = (double)__ldg(a + k), y = (double)__ldg(c + k);
        dot = __dadd_rn(dot, __dmul_rn(x, y));
        na = __dadd_rn(na, __dmul_rn(x, x));
        nb = __dadd_rn(nb, __dmul_rn(y, y));
    }
    const bool deg = na == 0.0 || nb == 0.0;  // degenerate_input_error: decide() rejects
    double s = __longlong_as_double(0x7ff8000000000000LL);  // quiet NaN
    if (!deg) {
        s = __ddiv_rn(dot, __dmul_rn(__dsqrt_rn(na), __dsqrt_rn(nb)));
        s = s < -1.0 ? -1.0 : (1.0 < s ? 1.0 : s);  // std::clamp(s, -1, 1)
    }
    score[i] = s;
    if (accepted) accepted[i] = (!deg && s >= theta) ? 1 : 0;
    if (degenerate) degenerate[i] = deg ? 1 : 0;
}

__global__ void kv_append_kernel(float* __restrict__ ck, float* __restrict__ cv, int64_t cap, int dm,
                                 const float* __restrict__ bk, const float* __restrict__ bv, int64_t T,
                                 int64_t dst_row) {
    const int64_t t = blockIdx.x;
    const int l = blockIdx.y;
    const float* sk = bk + ((int64_t)l * T + t) * dm;
    const float* sv = bv + ((int64_t)l * T + t) * dm;
    float* dk = ck + ((int64_t)l * cap + dst_row + t) * dm;
    float* dv = cv + ((int64_t)l * cap + dst_row + t) * dm;
    if ((dm & 3) == 0 && ((reinterpret_cast<uintptr_t>(sk) | reinterpret_cast<uintptr_t>(sv) |
                           reinterpret_cast<uintptr_t>(dk) | reinterpret_cast<uintptr_t>(dv)) & 15) == 0) {
        for (int c = threadIdx.x; c < dm / 4; c += blockDim.x) {
            reinterpret_cast<float4*>(dk)[c] = __ldg(reinterpret_cast<const float4*>(sk) + c);
            reinterpret_cast<float4*>(dv)[c] = __ldg(reinterpret_cast<const float4*>(sv) + c);
        }
    } else {
        for (int c = threadIdx.x; c < dm; c += blockDim.x) {
            dk[c] = __ldg(sk + c);
            dv[c] = __ldg(sv + c);
        }
    }
}

}  // namespace

// kernels::softmax (kernels.cpp:66-81): max-subtracted exp in fp64, the sum taken
// SEQUENTIALLY in index order (the reference's order) by one thread, then the
// divisions.  A non-finite input sets FLAG_NONFINITE (the reference throws
// precondition_error before any output).  One CTA: a host-API call on a vector.
__global__ void __launch_bounds__(1024) softmax_fp64_kernel(const double* __restrict__ s, int64_t n,
                                                            double* __restrict__ out, int* flag) {
    __shared__ double red[32];
    __shared__ double sum_s;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    double mx = -INFINITY;
    bool bad = false;
    for (int64_t i = tid; i < n; i += blockDim.x) {
        const double v = s[i];
        bad |= !isfinite(v);
        mx = (mx < v) ? v : mx;  // std::max
    }
    if (__syncthreads_or(bad)) {
        if (tid == 0) atomicOr(flag, FLAG_NONFINITE);
        return;
    }
    for (int o = 16; o; o >>= 1) {
        const double t = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = (mx < t) ? t : mx;
    }
    if (lane == 0) red[wid] = mx;
    __syncthreads();
    if (wid == 0) {
        double v = lane < (int)(blockDim.x >> 5) ? red[lane] : -INFINITY;
        for (int o = 16; o; o >>= 1) {
            const double t = __shfl_xor_sync(0xffffffffu, v, o);
            v = (v < t) ? t : v;
        }
        if (lane == 0) red[0] = v;
    }
    __syncthreads();
    mx = red[0];
    for (int64_t i = tid; i < n; i += blockDim.x) out[i] = exp(__dsub_rn(s[i], mx));
    __syncthreads();
    if (tid == 0) {
        double acc = 0.0;
        for (int64_t i = 0; i < n; ++i) acc = __dadd_rn(acc, out[i]);
        sum_s = acc;
    }
    __syncthreads();
    const double sum = sum_s;
    for (int64_t i = tid; i < n; i += blockDim.x) out[i] = __ddiv_rn(out[i], sum);
}

// kernels::argmax (kernels.cpp:94-101): best = 0, then i wins iff v[i] > v[best]:
// the lowest index of the maximum; a NaN never wins, except v[0] (nothing beats it)
__global__ void __launch_bounds__(1024) argmax_f32_kernel(const float* __restrict__ v, int64_t n, int* out) {
    __shared__ float bv[32];
    __shared__ int bi[32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    float best = NAN;
    int idx = INT_MAX;
    for (int64_t i = tid; i < n; i += blockDim.x) {
        const float x = v[i];
        if (isnan(x)) continue;
        if (idx == INT_MAX || x > best) { best = x; idx = (int)i; }  // i ascending per thread: first max kept
    }
    for (int o = 16; o; o >>= 1) {
        const float ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (oi != INT_MAX && (idx == INT_MAX || ob > best || (ob == best && oi < idx))) { best = ob; idx = oi; }
    }
    if (lane == 0) { bv[wid] = best; bi[wid] = idx; }
    __syncthreads();
    if (wid == 0) {
        best = lane < (int)(blockDim.x >> 5) ? bv[lane] : NAN;
        idx = lane < (int)(blockDim.x >> 5) ? bi[lane] : INT_MAX;
        for (int o = 16; o; o >>= 1) {
            const float ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
            if (oi != INT_MAX && (idx == INT_MAX || ob > best || (ob == best && oi < idx))) { best = ob; idx = oi; }
        }
        if (lane == 0) *out = (isnan(v[0]) || idx == INT_MAX) ? 0 : idx;
    }
}

void softmax_fp64(const double* s, int64_t n, double* out, int* flag, cudaStream_t st) {
    softmax_fp64_kernel<<<1, 1024, 0, st>>>(s, n, out, flag);
    check_launch("softmax_fp64_kernel");
}

void argmax_f32(const float* v, int64_t n, int* out, cudaStream_t st) {
    argmax_f32_kernel<<<1, 1024, 0, st>>>(v, n, out);
    check_launch("argmax_f32_kernel");
}

void attend_fp64_ws(const float* q, const float* k, const float* v, int64_t n, int H, int dk, double* w,
                    float* out, cudaStream_t s) {
    attend_fp64_kernel<<<H, 256, 0, s>>>(q, k, v, n, H, dk, 1.0 / std::sqrt((double)dk), w, out);
    check_launch("attend_fp64_kernel");
}

template <int QPG>
static bool launch_decode_v2(cx_ctx* ctx, const cx_decode_batch& b, cudaStream_t s) {
    const DecodeV2Smem lay = decode_v2_layout(b.k_syn, b.t_cap);
    static int max_optin = -1;
    if (max_optin < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    }
    if (lay.total > (size_t)max_optin) return false;
    const int n_lh = b.n_layers * b.n_kv;
    const int sms = ctx->num_sms > 0 ? ctx->num_sms : 148;
    int chunks = std::max(1, sms / n_lh);  // ~one CTA per SM; each stages its synapse once
    chunks = std::min(chunks, (b.n_agents + DV2_WARPS - 1) / DV2_WARPS);
    chunks = std::max(chunks, 1);
    const int per = (b.n_agents + chunks - 1) / chunks;
    kernel_smem(decode_v2_kernel<QPG>, lay.total);
    decode_v2_kernel<QPG><<<dim3((unsigned)n_lh, (unsigned)chunks), DV2_WARPS * 32, lay.total, s>>>(
        b, per, (float)(1.0 / std::sqrt((double)b.d_k)), ctx->d_flag);
    check_launch("decode_v2_kernel");
    return true;
}

void decode_step(cx_ctx* ctx, const cx_decode_batch& b, cudaStream_t s) {
    const int qpg = b.n_q / b.n_kv;
    // CX_OPT_DECODE_IMPL pins an implementation (tests; a pinned kernel that does not
    // apply to the shape is an error, not a silent fallback).  Default: the tcgen05
    // kernel (decode_tc.cu), then v2 (CUDA cores), then the generic v1.
    const int pin = ctx->opt.decode_impl;
    const bool allow_tc = pin == CX_DECODE_AUTO || pin == CX_DECODE_TC;
    const bool allow_v2 = pin == CX_DECODE_AUTO || pin == CX_DECODE_V2;
    if (allow_tc && decode_tc_launch(ctx, b, s)) return;
    if (pin == CX_DECODE_TC) fail(CX_PRECONDITION_ERROR, "decode_step: the pinned tcgen05 kernel does not apply to this shape");
    auto al = [](const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; };
    const bool v2_aligned = al(b.syn_keys, 16) && al(b.syn_values, 16) && al(b.q, 16) && al(b.tail_keys, 16) &&
                            al(b.tail_values, 16) && al(b.new_keys, 16) && al(b.new_values, 16) && al(b.out, 8);
    if (allow_v2 && v2_aligned && b.d_k == DV2_DK && b.k_syn <= 32 * DV2_KPL && b.t_cap <= 64) {
        bool done = false;
        switch (qpg) {
            case 1: done = launch_decode_v2<1>(ctx, b, s); break;
            case 2: done = launch_decode_v2<2>(ctx, b, s); break;
            case 4: done = launch_decode_v2<4>(ctx, b, s); break;
            case 7: done = launch_decode_v2<7>(ctx, b, s); break;
            case 8: done = launch_decode_v2<8>(ctx, b, s); break;
            default: break;
        }
        if (done) return;
    }
    if (pin == CX_DECODE_V2) fail(CX_PRECONDITION_ERROR, "decode_step: the pinned v2 kernel does not apply to this shape");
    int apb = std::max(1, 8 / qpg);
    const int warps = apb * qpg;
    const int t_rows = b.t_cap + 1;
    const DecodeSmem lay = decode_layout(b.k_syn, t_rows, b.d_k, apb, warps, b.k_syn + t_rows);
    static int max_optin = -1;
    if (max_optin < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    }
    if (lay.total > (size_t)max_optin) fail(CX_DEVICE_ERROR, "decode_step: synapse tile exceeds shared memory");
    const int n_lh = b.n_layers * b.n_kv;
    const int sms = ctx->num_sms > 0 ? ctx->num_sms : 148;
    // aim for ~2 CTAs per SM over the whole grid; each CTA reuses its staged synapse
    int chunks = std::max(1, (2 * sms + n_lh - 1) / n_lh);
    chunks = std::min(chunks, (b.n_agents + apb - 1) / apb);
    int per = (b.n_agents + chunks - 1) / chunks;
    per = ((per + apb - 1) / apb) * apb;
    chunks = (b.n_agents + per - 1) / per;
    kernel_smem(decode_step_kernel, lay.total);
    decode_step_kernel<<<dim3((unsigned)n_lh, (unsigned)chunks), warps * 32, lay.total, s>>>(
        b, apb, per, (float)(1.0 / std::sqrt((double)b.d_k)), ctx->d_flag);
    check_launch("decode_step_kernel");
}

void kv_append_rows(float* ck, float* cv, int64_t cap, int n_layers, int dm, const float* bk, const float* bv,
                    int64_t T, int64_t dst_row, cudaStream_t s) {
    if (T <= 0) return;
    kv_append_kernel<<<dim3((unsigned)T, (unsigned)n_layers), 128, 0, s>>>(ck, cv, cap, dm, bk, bv, T, dst_row);
    check_launch("kv_append_kernel");
}

void gate_decide(const float* h, int64_t hs, const float* t, int64_t ts, int64_t n, int dim, double theta,
                 double* score, uint8_t* accepted, uint8_t* degenerate, cudaStream_t s) {
    if (n <= 0) return;
    gate_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(h, hs, t, ts, n, dim, theta, score, accepted, degenerate);
    check_launch("gate_kernel");
}

}  // namespace cx

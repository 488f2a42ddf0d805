// decode_tc.cu -- batched decode attention with the shared-synapse part on the
// 5th-generation tensor cores (tcgen05 + TMEM), SURVEY.md §8(a) A9.
//
// For one (layer, KV head) the synapse part of every agent's attention is a
// GEMM across agents: S = Q K_syn^T with M = agents x q-heads, N = k_syn,
// K = d_k = 64, then O_syn = P V_syn.  A CTA owns one (layer, KV head) and
// loops over tiles of 128 query rows (18 agents x 7 q-heads):
//   1. Q tile -> shared memory as a bf16 hi/lo pair (x = hi + lo exactly to
//      2^-17), K_syn / V_syn^T staged once per CTA the same way;
//   2. one thread issues S = Qhi Khi + Qhi Klo + Qlo Khi (tcgen05.mma kind::f16,
//      fp32 accumulate in TMEM) while all warps compute the private-row scores
//      on CUDA cores (warp per agent, lane per private row);
//   3. thread-per-row softmax over [synapse || private] (tcgen05.ld of the S
//      row, max/exp/sum in fp32), unnormalised P_syn written back as bf16 hi/lo;
//   4. one thread issues O = P V_syn (3 MMAs per k-step) while the warps mix the
//      private rows (lane per output dim) into shared memory;
//   5. thread-per-row epilogue: (O_syn + O_priv) / sum -> global.
// The new token's K/V is appended to the private rows first (fused).
// Accuracy: every product is formed to ~2^-16 relative, accumulated in fp32,
// i.e. the north_star's "fp32 accumulate, 1e-3 relative" contract.
#include <cuda_bf16.h>

#include "cx_internal.cuh"

namespace cx {

namespace {

constexpr int TD = 64;         // d_k
constexpr int TM = 128;        // MMA M (query rows per tile)
constexpr int TNS_MAX = 176;   // padded synapse keys (multiple of 16)
constexpr int TTAIL = 64;      // max private rows
constexpr int TTHREADS = 256;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major SWIZZLE_NONE core-matrix layout (8 rows x 16 B core matrices; row
// groups 128 B apart (SBO); 8-element K chunks (R/8)*128 B apart (LBO)).
__host__ __device__ __forceinline__ uint32_t cm_off(int r, int k, int R) {
    return (uint32_t)((((k >> 3) * (R >> 3) + (r >> 3)) << 7) + ((r & 7) << 4) + ((k & 7) << 1));
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    return d;                // SWIZZLE_NONE, base offset 0
}

__host__ __device__ __forceinline__ uint32_t idesc_bf16_f32(int m, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t dtmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(dtmem),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(mbar))
                 : "memory");
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t* m, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok)
                     : "r"(su32(m)), "r"(parity)
                     : "memory");
    } while (!ok);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* out) {
    uint32_t v[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 16; ++j) out[j] = __uint_as_float(v[j]);
}

// split x into bf16 hi + lo (x - hi - lo ~ 2^-17 |x|)
__device__ __forceinline__ void split_bf16(float x, __nv_bfloat16& hi, __nv_bfloat16& lo) {
    hi = __float2bfloat16_rn(x);
    lo = __float2bfloat16_rn(x - __bfloat162float(hi));
}

constexpr int TPCH = 96;       // synapse keys per P.V chunk (P buffer = 128 x 96 bf16 hi/lo)

struct TcLayout {
    size_t kh, kl, vh, vl, qh, ql, ph, pl, st, rs, mbar, tbase, total;
    int ns;       // padded synapse keys
    int sstride;  // private-score row stride
};

__host__ __device__ inline TcLayout tc_layout(int k_syn, int t_cap) {
    TcLayout L;
    L.ns = ((k_syn + 15) / 16) * 16;
    L.sstride = t_cap + 1;
    const size_t kv = (size_t)L.ns * TD * 2;       // one bf16 operand
    const size_t q = (size_t)TM * TD * 2;
    const size_t pp = (size_t)TM * TPCH * 2;
    size_t o = 0;
    L.kh = o; o += kv;
    L.kl = o; o += kv;
    L.vh = o; o += kv;
    L.vl = o; o += kv;
    L.qh = o; o += q;   // Q hi/lo; reused as the private-row output [TM][TD] fp32 in step 4
    L.ql = o; o += q;
    L.ph = o; o += pp;
    L.pl = o; o += pp;
    L.st = o; o += sizeof(float) * (size_t)TM * L.sstride;  // private scores / weights
    L.rs = o; o += sizeof(float) * TM;                       // row sums
    L.mbar = o; o += 16;
    L.tbase = o; o += 16;
    L.total = (o + 127) & ~(size_t)127;
    return L;
}

template <int QPG>
__global__ void __launch_bounds__(TTHREADS, 1) decode_tc_kernel(cx_decode_batch b, float scale) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const TcLayout lay = tc_layout(b.k_syn, b.t_cap);
    const int NS = lay.ns;
    __nv_bfloat16* Kh = reinterpret_cast<__nv_bfloat16*>(smem + lay.kh);
    __nv_bfloat16* Kl = reinterpret_cast<__nv_bfloat16*>(smem + lay.kl);
    __nv_bfloat16* Vh = reinterpret_cast<__nv_bfloat16*>(smem + lay.vh);
    __nv_bfloat16* Vl = reinterpret_cast<__nv_bfloat16*>(smem + lay.vl);
    __nv_bfloat16* Qh = reinterpret_cast<__nv_bfloat16*>(smem + lay.qh);
    __nv_bfloat16* Ql = reinterpret_cast<__nv_bfloat16*>(smem + lay.ql);
    float* Ot = reinterpret_cast<float*>(smem + lay.qh);  // aliases Q after the score MMAs
    __nv_bfloat16* Ph = reinterpret_cast<__nv_bfloat16*>(smem + lay.ph);
    __nv_bfloat16* Pl = reinterpret_cast<__nv_bfloat16*>(smem + lay.pl);
    float* St = reinterpret_cast<float*>(smem + lay.st);   // [TM][TTAIL + 1]
    float* Rs = reinterpret_cast<float*>(smem + lay.rs);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + lay.mbar);
    uint32_t* tbase_s = reinterpret_cast<uint32_t*>(smem + lay.tbase);

    const int lh = blockIdx.x;
    const int l = lh / b.n_kv, g = lh % b.n_kv;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ks = b.k_syn;
    constexpr int AT = TM / QPG;  // agents per tile
    const bool app = b.new_keys != nullptr;

    // ---- one-time: TMEM (S: NS cols, O: 64 cols), mbarriers, K_syn / V_syn^T ----
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tbase_s)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    const float* sk = b.syn_keys + (size_t)lh * ks * TD;
    const float* sv = b.syn_values + (size_t)lh * ks * TD;
    for (int e = tid; e < NS * TD; e += blockDim.x) {
        const int j = e / TD, c = e % TD;
        const float kv = j < ks ? __ldg(sk + (size_t)j * TD + c) : 0.f;
        const float vv = j < ks ? __ldg(sv + (size_t)j * TD + c) : 0.f;
        __nv_bfloat16 h, lo;
        split_bf16(kv, h, lo);
        Kh[cm_off(j, c, NS) >> 1] = h;   // B of S = Q K^T: N = keys, K = dims
        Kl[cm_off(j, c, NS) >> 1] = lo;
        split_bf16(vv, h, lo);
        Vh[cm_off(c, j, TD) >> 1] = h;   // B of O = P V: N = dims, K = keys (V^T)
        Vl[cm_off(c, j, TD) >> 1] = lo;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tS = *tbase_s, tO = tS + (uint32_t)NS;
    const uint32_t idS = idesc_bf16_f32(TM, NS), idO = idesc_bf16_f32(TM, TD);
    uint32_t ph0 = 0, ph1 = 0;

    const int n_tiles = (b.n_agents + AT - 1) / AT;
    for (int tile = blockIdx.y; tile < n_tiles; tile += gridDim.y) {
        const int a0 = tile * AT;
        const int na = min(AT, b.n_agents - a0);
        const int rows = na * QPG;
        // ---- 1. Q tile -> bf16 hi/lo (rows >= `rows` zero) ----
        for (int e = tid; e < TM * TD; e += blockDim.x) {
            const int r = e / TD, c = e % TD;
            float x = 0.f;
            if (r < rows) {
                const int a = a0 + r / QPG, hh = r % QPG;
                x = __ldg(b.q + (((size_t)a * b.n_layers + l) * b.n_q + (size_t)g * QPG + hh) * TD + c);
            }
            __nv_bfloat16 h, lo;
            split_bf16(x, h, lo);
            Qh[cm_off(r, c, TM) >> 1] = h;
            Ql[cm_off(r, c, TM) >> 1] = lo;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        // ---- 2. S = Q K^T on the tensor cores (3 MMAs per 16-wide k-step) ----
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t qlbo = (TM / 8) * 128, klbo = (uint32_t)(NS / 8) * 128;
            for (int kk = 0; kk < TD / 16; ++kk) {
                const uint32_t qo = kk * 2 * qlbo, ko = kk * 2 * klbo;
                const uint64_t qh = sdesc(su32(Qh) + qo, qlbo, 128), ql = sdesc(su32(Ql) + qo, qlbo, 128);
                const uint64_t kh = sdesc(su32(Kh) + ko, klbo, 128), kl = sdesc(su32(Kl) + ko, klbo, 128);
                mma_bf16(tS, ql, kh, idS, kk > 0 ? 1u : 0u);
                mma_bf16(tS, qh, kl, idS, 1u);
                mma_bf16(tS, qh, kh, idS, 1u);
            }
            mma_commit(&mbar[0]);
        }
        // private-row scores on CUDA cores while the MMAs run: warp per agent,
        // lane t (and t + 32) per private row, all q-heads of the group
        for (int ai = warp; ai < na; ai += TTHREADS / 32) {
            const int a = a0 + ai;
            const int len = min(b.tail_len[a], b.t_cap - (app ? 1 : 0));
            const int nt = len + (app ? 1 : 0);
            const size_t toff = ((((size_t)a * b.n_layers + l) * b.n_kv + g) * b.t_cap) * TD;
            const size_t noff = (((size_t)a * b.n_layers + l) * b.n_kv + g) * TD;
            if (app && lane < 16) {  // append the new row (fused)
                reinterpret_cast<float4*>(b.tail_keys + toff + (size_t)len * TD)[lane] =
                    __ldg(reinterpret_cast<const float4*>(b.new_keys + noff) + lane);
                reinterpret_cast<float4*>(b.tail_values + toff + (size_t)len * TD)[lane] =
                    __ldg(reinterpret_cast<const float4*>(b.new_values + noff) + lane);
            }
            float acc[2][QPG];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int h = 0; h < QPG; ++h) acc[i][h] = 0.f;
            const float* r0p = (app && lane == len) ? b.new_keys + noff : b.tail_keys + toff + (size_t)lane * TD;
            const float* r1p = (app && lane + 32 == len) ? b.new_keys + noff : b.tail_keys + toff + (size_t)(lane + 32) * TD;
#pragma unroll 2
            for (int c8 = 0; c8 < TD / 8; ++c8) {
                float4 k0a = make_float4(0.f, 0.f, 0.f, 0.f), k0b = k0a, k1a = k0a, k1b = k0a;
                if (lane < nt) {
                    k0a = __ldg(reinterpret_cast<const float4*>(r0p) + 2 * c8);
                    k0b = __ldg(reinterpret_cast<const float4*>(r0p) + 2 * c8 + 1);
                }
                if (lane + 32 < nt) {
                    k1a = __ldg(reinterpret_cast<const float4*>(r1p) + 2 * c8);
                    k1b = __ldg(reinterpret_cast<const float4*>(r1p) + 2 * c8 + 1);
                }
                const float k0[8] = {k0a.x, k0a.y, k0a.z, k0a.w, k0b.x, k0b.y, k0b.z, k0b.w};
                const float k1[8] = {k1a.x, k1a.y, k1a.z, k1a.w, k1b.x, k1b.y, k1b.z, k1b.w};
#pragma unroll
                for (int h = 0; h < QPG; ++h) {
                    const int r = ai * QPG + h;  // q = hi + lo, read back from the A operand
                    const uint4 hv = *reinterpret_cast<const uint4*>(reinterpret_cast<const unsigned char*>(Qh) + cm_off(r, 8 * c8, TM));
                    const uint4 lv = *reinterpret_cast<const uint4*>(reinterpret_cast<const unsigned char*>(Ql) + cm_off(r, 8 * c8, TM));
                    const __nv_bfloat16* hb = reinterpret_cast<const __nv_bfloat16*>(&hv);
                    const __nv_bfloat16* lb = reinterpret_cast<const __nv_bfloat16*>(&lv);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const float qv = __bfloat162float(hb[u]) + __bfloat162float(lb[u]);
                        acc[0][h] = fmaf(qv, k0[u], acc[0][h]);
                        acc[1][h] = fmaf(qv, k1[u], acc[1][h]);
                    }
                }
            }
#pragma unroll
            for (int h = 0; h < QPG; ++h) {
                float* srow = St + (ai * QPG + h) * lay.sstride;
                if (lane < nt) srow[lane] = acc[0][h] * scale;
                if (lane + 32 < nt) srow[lane + 32] = acc[1][h] * scale;
            }
        }
        mbar_wait_parity(&mbar[0], ph0);
        ph0 ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        __syncthreads();  // private scores in St; S in TMEM; Q (shared) is dead -> Ot may reuse it

        // ---- 3. softmax per row (warps 0-3 own TMEM lanes 0-127 = rows) ----
        const int sst = lay.sstride;
        const uint32_t trow = tS + ((uint32_t)((warp & 3) * 32) << 16);
        const int r_own = (warp & 3) * 32 + lane;
        float m_row = -INFINITY, sum_row = 0.f;
        if (warp < 4) {
            const bool live = r_own < rows;
            int nt = 0;
            if (live) {
                const int a = a0 + r_own / QPG;
                nt = min(b.tail_len[a], b.t_cap - (app ? 1 : 0)) + (app ? 1 : 0);
            }
            for (int c0 = 0; c0 < NS; c0 += 16) {
                float v[16];
                tmem_ld16(trow + (uint32_t)c0, v);
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (c0 + j < ks) m_row = fmaxf(m_row, v[j] * scale);
            }
            float* srow = St + r_own * sst;
            for (int t = 0; t < nt; ++t) m_row = fmaxf(m_row, srow[t]);
            for (int t = 0; t < nt; ++t) {  // private weights (unnormalised)
                const float p = __expf(srow[t] - m_row);
                srow[t] = p;
                sum_row += p;
            }
        }
        // ---- 4. O_syn = P V_syn on the tensor cores in 96-key chunks; the
        //         private rows are mixed on CUDA cores during the first chunk ----
        for (int k0 = 0; k0 < NS; k0 += TPCH) {
            const int kn = min(TPCH, NS - k0);
            if (warp < 4) {
                const bool live = r_own < rows;
                for (int c0 = 0; c0 < kn; c0 += 16) {
                    float v[16];
                    tmem_ld16(trow + (uint32_t)(k0 + c0), v);
#pragma unroll
                    for (int j8 = 0; j8 < 2; ++j8) {  // 8 keys = one 16-byte core-matrix row chunk
                        __align__(16) __nv_bfloat16 hv[8], lv[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int j = k0 + c0 + j8 * 8 + u;
                            const float p = (live && j < ks) ? __expf(v[j8 * 8 + u] * scale - m_row) : 0.f;
                            sum_row += p;
                            split_bf16(p, hv[u], lv[u]);
                        }
                        const uint32_t off = cm_off(r_own, c0 + j8 * 8, TM);
                        *reinterpret_cast<uint4*>(reinterpret_cast<unsigned char*>(Ph) + off) = *reinterpret_cast<uint4*>(hv);
                        *reinterpret_cast<uint4*>(reinterpret_cast<unsigned char*>(Pl) + off) = *reinterpret_cast<uint4*>(lv);
                    }
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncthreads();
            if (tid == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t plbo = (TM / 8) * 128, vlbo = (TD / 8) * 128;
                for (int kk = 0; kk < kn / 16; ++kk) {
                    const uint32_t po = kk * 2 * plbo, vo = ((k0 >> 3) + kk * 2) * vlbo;
                    const uint64_t ph = sdesc(su32(Ph) + po, plbo, 128), pl = sdesc(su32(Pl) + po, plbo, 128);
                    const uint64_t vh = sdesc(su32(Vh) + vo, vlbo, 128), vl = sdesc(su32(Vl) + vo, vlbo, 128);
                    mma_bf16(tO, pl, vh, idO, (k0 > 0 || kk > 0) ? 1u : 0u);
                    mma_bf16(tO, ph, vl, idO, 1u);
                    mma_bf16(tO, ph, vh, idO, 1u);
                }
                mma_commit(&mbar[1]);
            }
            if (k0 == 0) {
                for (int ai = warp; ai < na; ai += TTHREADS / 32) {  // lane owns dims 2 lane, 2 lane + 1
            const int a = a0 + ai;
            const int len = min(b.tail_len[a], b.t_cap - (app ? 1 : 0));
            const int nt = len + (app ? 1 : 0);
            const size_t toff = ((((size_t)a * b.n_layers + l) * b.n_kv + g) * b.t_cap) * TD;
            const size_t noff = (((size_t)a * b.n_layers + l) * b.n_kv + g) * TD;
            float2 o[QPG];
#pragma unroll
            for (int h = 0; h < QPG; ++h) o[h] = make_float2(0.f, 0.f);
#pragma unroll 4
            for (int t = 0; t < nt; ++t) {
                const float* vrow = (app && t == len) ? b.new_values + noff : b.tail_values + toff + (size_t)t * TD;
                const float2 v = __ldg(reinterpret_cast<const float2*>(vrow) + lane);
#pragma unroll
                for (int h = 0; h < QPG; ++h) {
                    const float p = St[(ai * QPG + h) * sst + t];
                    o[h].x = fmaf(p, v.x, o[h].x);
                    o[h].y = fmaf(p, v.y, o[h].y);
                }
            }
#pragma unroll
            for (int h = 0; h < QPG; ++h) reinterpret_cast<float2*>(Ot + (ai * QPG + h) * TD)[lane] = o[h];
                }
            }
            mbar_wait_parity(&mbar[1], ph1);  // P chunk consumed (and O complete after the last)
            ph1 ^= 1u;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            __syncthreads();
        }
        // ---- 5. epilogue: (O_syn + O_priv) / sum ----
        if (warp < 4) {
            const int r = r_own;
            const uint32_t trow_o = tO + ((uint32_t)(warp * 32) << 16);
            float v[TD];
#pragma unroll
            for (int c0 = 0; c0 < TD; c0 += 16) tmem_ld16(trow_o + (uint32_t)c0, v + c0);
            if (r < rows) {
                const int a = a0 + r / QPG, hh = r % QPG;
                const float inv = 1.0f / sum_row;
                float* out = b.out + (((size_t)a * b.n_layers + l) * b.n_q + (size_t)g * QPG + hh) * TD;
                const float* ot = Ot + r * TD;
#pragma unroll
                for (int c4 = 0; c4 < TD / 4; ++c4) {
                    const float4 p = reinterpret_cast<const float4*>(ot)[c4];
                    reinterpret_cast<float4*>(out)[c4] =
                        make_float4((v[4 * c4] + p.x) * inv, (v[4 * c4 + 1] + p.y) * inv, (v[4 * c4 + 2] + p.z) * inv,
                                    (v[4 * c4 + 3] + p.w) * inv);
                }
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();  // Ot / St / TMEM reuse by the next tile
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tbase_s), "r"(256));
}

}  // namespace

bool decode_tc_launch(cx_ctx* ctx, const cx_decode_batch& b, cudaStream_t s) {
    const int qpg = b.n_q / b.n_kv;
    if (b.d_k != TD || b.k_syn < 1 || b.k_syn > TNS_MAX || b.t_cap > TTAIL) return false;
    const TcLayout lay = tc_layout(b.k_syn, b.t_cap);
    static int max_optin = -1;
    if (max_optin < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    }
    if (lay.total > (size_t)max_optin) return false;
    void (*kern)(cx_decode_batch, float) = nullptr;
    switch (qpg) {
        case 1: kern = decode_tc_kernel<1>; break;
        case 2: kern = decode_tc_kernel<2>; break;
        case 4: kern = decode_tc_kernel<4>; break;
        case 7: kern = decode_tc_kernel<7>; break;
        case 8: kern = decode_tc_kernel<8>; break;
        default: return false;
    }
    const int n_lh = b.n_layers * b.n_kv;
    const int at = TM / qpg;
    const int n_tiles = (b.n_agents + at - 1) / at;
    const int sms = ctx->num_sms > 0 ? ctx->num_sms : 148;
    const int per_lh = std::max(1, std::min(n_tiles, (sms + n_lh - 1) / n_lh));
    CX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lay.total));
    kern<<<dim3((unsigned)n_lh, (unsigned)per_lh), TTHREADS, lay.total, s>>>(b, (float)(1.0 / std::sqrt((double)b.d_k)));
    check_launch("decode_tc_kernel");
    return true;
}

}  // namespace cx

// decode_tc.cu -- batched decode attention with the shared-synapse part on the
// 5th-generation tensor cores (tcgen05 + TMEM), SURVEY.md §8(a) A9.
//
// For one (layer, KV head) the synapse part of every agent's attention is a
// GEMM across agents: S = Q K_syn^T with M = agents x q-heads, N = k_syn,
// K = d_k = 64, then O_syn = P V_syn.  The private rows (each agent's own
// recent K/V, the dominant HBM stream) are per-agent and have no reuse.  A CTA
// owns one (layer, KV head), stages K_syn / V_syn^T once, and loops over tiles
// of 128 query rows (e.g. 18 agents x 7 q-heads) with two warp roles that run
// concurrently and meet once per tile:
//   synapse warps 0-3 (thread per TMEM lane = query row; they alone stage
//   K_syn / V_syn^T, the private warps start streaming at kernel start):
//     1. Q tile -> shared memory as a bf16 hi/lo pair (x = hi + lo to 2^-17);
//     2. one thread issues S = Qlo Khi + Qhi Klo + Qhi Khi (tcgen05.mma
//        kind::f16, fp32 accumulate in TMEM);
//     3. row softmax over the synapse keys (m_s, l_s); the unnormalised P goes
//        to TMEM as packed bf16x2 hi / lo (tcgen05.st) and is the A operand of
//        O_syn = P V_syn: per k-step one N = 128 TS-MMA P_hi [V_hi | V_lo] and one
//        N = 64 P_lo V_hi (V_hi / V_lo stacked as one 128-row B operand);
//     4. tile i+1's Q and S are issued while tile i's P.V runs (pipelined);
//     5. epilogue: merge with the private partial (flash-style rescale).
//   private warps 4-15 (warp per agent, agents dealt round-robin over the CTA's
//   whole agent sequence): append the new token's K/V (fused, used from
//   registers), stream the stored private rows in 16-row batches (8 lanes per
//   row: q fits in registers, one warp load reads 4 rows x 128 B; the next
//   batch is prefetched into L1), form scores (packed FMAs + reduce-scatter),
//   softmax (m_p, l_p) and O_priv on CUDA cores, publish to shared memory
//   (gated by an epilogue counter; two parity-split mbarriers hand tiles over).
// The merge (m = max(m_s, m_p); O = (O_s e^{m_s-m} + O_p e^{m_p-m}) /
// (l_s e^{m_s-m} + l_p e^{m_p-m})) is the one-pass softmax of the reference's
// kernels::attend (kernels.cpp:103-142) over [synapse rows || private rows].
// Accuracy: every synapse product is formed to ~2^-16 relative and all sums
// accumulate in fp32: the north_star's "fp32 accumulate, 1e-3 relative".
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>

#include "cx_internal.cuh"

namespace cx {

namespace {

constexpr int TD = 64;          // d_k
constexpr int TM = 128;         // MMA M (query rows per tile)
constexpr int TNS_MAX = 176;    // padded synapse keys (multiple of 16)
constexpr int TTAIL = 64;       // max private rows
constexpr int SWARPS = 4;       // synapse warps (TMEM lanes 0-127)
constexpr int PWARPS = 12;      // private-row warps (13+ warps allocate registers like 16)
constexpr int TTHREADS = 32 * (SWARPS + PWARPS);
constexpr int OPS = TD + 4;     // O_priv row stride (floats; conflict-free float4 rows)
constexpr int SST = TTAIL + 4;
// O_priv buffers: 2 lets the private warps publish a tile before the previous tile's
// epilogue; 1 saves 35 KB of shared memory, i.e. leaves L1 room for the private stream
#ifndef CX_TC_OP_BUFS
#define CX_TC_OP_BUFS 1
#endif
constexpr int OP_BUFS = CX_TC_OP_BUFS;  // O_priv buffers (2: private warps may run a whole tile ahead)


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

// A operand from tensor memory (packed bf16x2, row = lane), B from shared memory
__device__ __forceinline__ void mma_bf16_ts(uint32_t dtmem, uint32_t atmem, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }" ::"r"(dtmem),
        "r"(atmem), "l"(bd), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
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
    __syncwarp();
}

// Named barrier among the synapse warps.  Named barriers count whole warps
// (.aligned): reconverge first -- lanes leave the mbarrier spin loops at different
// iterations.  (Cross-role hand-offs use mbarriers, not bar.arrive.)
__device__ __forceinline__ void bar_sync(int id, int n) {
    __syncwarp();
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// packed fp32x2 FMA (sm_100): two independent fp32 FMAs per instruction
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(d)
        : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)),
          "l"(*reinterpret_cast<uint64_t*>(&c)));
    return *reinterpret_cast<float2*>(&d);
}

// bulk prefetch of a contiguous block into L2 (no registers, no shared memory)
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// packed fp32x2 add (sm_100)
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;"
        : "=l"(d)
        : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)));
    return *reinterpret_cast<float2*>(&d);
}

// one 32-byte sector per lane (256-bit load, sm_100), no L1 allocation
__device__ __forceinline__ void ld_v8_na(const float* p, float (&x)[8]) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]), "=f"(x[5]), "=f"(x[6]), "=f"(x[7])
                 : "l"(p));
}

// long waits (a role waiting for the other): back off instead of spinning on issue slots
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* m, uint32_t parity) {
    uint32_t ok = 0;
    for (;;) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok)
                     : "r"(su32(m)), "r"(parity)
                     : "memory");
        if (ok) break;
        __nanosleep(128);
    }
    __syncwarp();
}

// private warps: wait until at least `n` tile epilogues have completed
__device__ __forceinline__ void wait_epilogues(volatile int* epi_done, int n) {
    if (n > 0)
        while (*epi_done < n) __nanosleep(64);
    __threadfence_block();
    __syncwarp();
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

// two 16-column loads under ONE wait (the O halves of the epilogue): out = a + b
__device__ __forceinline__ void tmem_ld16x2_sum(uint32_t ta, uint32_t tb, float* out) {
    uint32_t a[16], b[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), "=r"(a[7]), "=r"(a[8]),
          "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]), "=r"(a[13]), "=r"(a[14]), "=r"(a[15])
        : "r"(ta));
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3]), "=r"(b[4]), "=r"(b[5]), "=r"(b[6]), "=r"(b[7]), "=r"(b[8]),
          "=r"(b[9]), "=r"(b[10]), "=r"(b[11]), "=r"(b[12]), "=r"(b[13]), "=r"(b[14]), "=r"(b[15])
        : "r"(tb));
    // the wait takes every destination register as an operand: no use can move above it
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7]),
                   "+r"(a[8]), "+r"(a[9]), "+r"(a[10]), "+r"(a[11]), "+r"(a[12]), "+r"(a[13]), "+r"(a[14]), "+r"(a[15]),
                   "+r"(b[0]), "+r"(b[1]), "+r"(b[2]), "+r"(b[3]), "+r"(b[4]), "+r"(b[5]), "+r"(b[6]), "+r"(b[7]),
                   "+r"(b[8]), "+r"(b[9]), "+r"(b[10]), "+r"(b[11]), "+r"(b[12]), "+r"(b[13]), "+r"(b[14]), "+r"(b[15])
                 :
                 : "memory");
#pragma unroll
    for (int j = 0; j < 16; ++j) out[j] = __uint_as_float(a[j]) + __uint_as_float(b[j]);
}

// 8 floats -> one 16-byte core-matrix row chunk of hi and of lo (packed bf16x2 conversions)
__device__ __forceinline__ void split8_store(const float* x, unsigned char* hi_base, unsigned char* lo_base, uint32_t off) {
    uint32_t hv[4], lv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const __nv_bfloat162 h2 = __floats2bfloat162_rn(x[2 * u], x[2 * u + 1]);
        const float2 hf = __bfloat1622float2(h2);
        const __nv_bfloat162 l2 = __floats2bfloat162_rn(x[2 * u] - hf.x, x[2 * u + 1] - hf.y);
        hv[u] = *reinterpret_cast<const uint32_t*>(&h2);
        lv[u] = *reinterpret_cast<const uint32_t*>(&l2);
    }
    *reinterpret_cast<uint4*>(hi_base + off) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
    *reinterpret_cast<uint4*>(lo_base + off) = make_uint4(lv[0], lv[1], lv[2], lv[3]);
}

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}


struct TcLayout {
    size_t kh, kl, vh, vl, qo, op, sw, mp, lp, mbar, tbase, total;
    int ns;  // padded synapse keys
};

__host__ __device__ inline TcLayout tc_layout(int k_syn, int qpg) {
    TcLayout L;
    L.ns = ((k_syn + 15) / 16) * 16;
    const size_t kv = (size_t)L.ns * TD * 2;  // one bf16 operand
    const size_t q2 = (size_t)2 * TM * TD * 2, op = sizeof(float) * (size_t)TM * OPS;
    const size_t pw = sizeof(float) * (size_t)PWARPS * qpg * SST;
    size_t o = 0;
    L.kh = o; o += kv;
    L.kl = o; o += kv;
    L.vh = o; o += 2 * kv;             // V^T hi (rows 0-63) | lo (rows 64-127): one N = 128 operand
    L.qo = o; o += q2;                 // Q hi | lo (A operand of the score MMAs)
    L.op = o; o += OP_BUFS * op;       // O_priv [OP_BUFS][TM][OPS]
    L.sw = o; o += pw;                 // per private warp: scores / weights [qpg][SST]
    L.mp = o; o += sizeof(float) * 2 * TM;  // private (m, l) per row, double-buffered by tile parity
    L.lp = o; o += sizeof(float) * 2 * TM;
    L.mbar = o; o += 32;
    L.tbase = o; o += 16;              // TMEM base address, then the epilogue counter
    L.total = (o + 127) & ~(size_t)127;
    return L;
}

#ifdef CX_EXPERIMENTS
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// build-time debugging only (CX_NVCC_EXTRA=-DCX_EXPERIMENTS): trc (CX_TC_TRACE=1) = phase
// timestamps of CTA (0, 0); skip (CX_TC_SKIP=1|2) = skip one role's math (timing only:
// the outputs are NOT valid then).  The release library compiles both out.
#define TC_TRACE(slot)                                                                  \
    do {                                                                                \
        if (trc && blockIdx.x == 0 && blockIdx.y == 0) trc[(slot)] = gtime();            \
    } while (0)
#define TC_SKIP(bit) (skip & (bit))
#else
#define TC_TRACE(slot) \
    do {               \
    } while (0)
#define TC_SKIP(bit) false
#endif

// ---- private-row helpers (warp per agent) ----
// L1PF: private rows go through L1 (ld.global.nc) and each 16-row batch is
// prefetched into L1 one batch ahead (prefetch.global.L1: no registers, no shared
// memory); otherwise they are streamed with ld.global.cg (L2 only).
constexpr bool L1PF = true;
constexpr int PB = 16;  // private rows per batch (8: 331 us at N=1000 vs 301 us -- more exposed round trips)
template <class T>
__device__ __forceinline__ T ldrow(const T* p) { return L1PF ? __ldg(p) : __ldcg(p); }
// the 32 lines of 16 private rows starting at row r0 (row = 256 B), one per lane
template <int NR = 16>  // NR rows = NR * 2 lines; lanes beyond them idle
__device__ __forceinline__ void prefetch_rows16_l1(const float* base, int r0, int nrows, int lane) {
    if (lane >= 2 * NR) return;
    if (L1PF && r0 + (lane >> 1) < nrows)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(base + (size_t)r0 * TD + lane * 32));
}
// q lives in registers: lane rl of a row's 8 lanes holds dims [8 rl, 8 rl + 8) of every
// head (one 256-bit load per row and lane), as qa = [8 rl, 8 rl + 4), qb = [8 rl + 4, 8 rl + 8).
// 256-bit load of a row's 8-dim chunk through L1 (the private rows are prefetched there)
__device__ __forceinline__ void ld_row8(const float* p, float4& a, float4& b) {
    asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                 : "l"(p));
}

// score of one row per 8-lane group (row t of lane group lane / 8, whose lanes hold
// its dims [8 rl, 8 rl + 4) in ka and [8 rl + 4, 8 rl + 8) in kb): packed FMAs, then a
// reduce-scatter so that the 8 lanes end up with one head each; stored when `valid`
template <int QPG>
__device__ __forceinline__ void score_group(const float4& ka, const float4& kb, int t, bool valid,
                                            const float4 (&qa)[QPG], const float4 (&qb)[QPG], float* Sw, int lane,
                                            float scale) {
    constexpr int NV = QPG <= 1 ? 1 : QPG <= 2 ? 2 : QPG <= 4 ? 4 : 8;
    constexpr int RB = 8 / NV;
    int hown = 0;
#pragma unroll
    for (int w = NV / 2, bit = 4; w >= 1; w >>= 1, bit >>= 1)
        if (lane & bit) hown += w;
    float v[NV];
#pragma unroll
    for (int h = 0; h < NV; ++h) {
        v[h] = 0.f;
        if (h < QPG) {
            float2 acc = ffma2(make_float2(qa[h].x, qa[h].y), make_float2(ka.x, ka.y), make_float2(0.f, 0.f));
            acc = ffma2(make_float2(qa[h].z, qa[h].w), make_float2(ka.z, ka.w), acc);
            acc = ffma2(make_float2(qb[h].x, qb[h].y), make_float2(kb.x, kb.y), acc);
            acc = ffma2(make_float2(qb[h].z, qb[h].w), make_float2(kb.z, kb.w), acc);
            v[h] = acc.x + acc.y;
        }
    }
#pragma unroll
    for (int w = NV / 2, bit = 4; w >= 1; w >>= 1, bit >>= 1) {
        const bool up = lane & bit;
#pragma unroll
        for (int i = 0; i < w; ++i) {
            const float send = up ? v[i] : v[i + w];
            const float keep = up ? v[i + w] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
        }
    }
#pragma unroll
    for (int bit = RB / 2; bit >= 1; bit >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], bit);
    if ((lane & (RB - 1)) == 0 && hown < QPG && valid) Sw[hown * SST + t] = v[0] * scale;
}

// scores of rows [r0, r0 + 4 NG): 8 lanes per row, 4 rows per warp load (4 x 128
// contiguous bytes); rows at or beyond nt are masked when PRED.
template <int QPG, int NG, bool PRED>
__device__ __forceinline__ void score_rows(const float* tk, int r0, int nt, const float4 (&qa)[QPG],
                                           const float4 (&qb)[QPG], float* Sw, int lane, float scale) {
    const int rl = lane & 7, rg = lane >> 3;
    float4 ka[NG], kb[NG];
#pragma unroll
    for (int j = 0; j < NG; ++j) {
        const int t = r0 + 4 * j + rg;
        const float4* kp = reinterpret_cast<const float4*>(tk + (size_t)t * TD);
        if (!PRED || t < nt) {
            ld_row8(reinterpret_cast<const float*>(kp + 2 * rl), ka[j], kb[j]);
        } else {
            ka[j] = kb[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
#pragma unroll
    for (int j = 0; j < NG; ++j) {
        const int t = r0 + 4 * j + rg;
        score_group<QPG>(ka[j], kb[j], t, !PRED || t < nt, qa, qb, Sw, lane, scale);
    }
}

// o[h] += sum_{t in [r0, r0 + NR)} w[h][t] v[t][2 lane .. 2 lane + 1]; rows >= nt masked when PRED
template <int QPG, int NR, bool PRED>
__device__ __forceinline__ void mix_rows(const float* tv, int r0, int nt, const float* Sw, float2 (&o)[QPG], int lane) {
    float2 v[NR];
#pragma unroll
    for (int t = 0; t < NR; ++t)
        v[t] = (!PRED || r0 + t < nt) ? ldrow(reinterpret_cast<const float2*>(tv + (size_t)(r0 + t) * TD) + lane)
                                      : make_float2(0.f, 0.f);
#pragma unroll
    for (int t4 = 0; t4 < NR / 4; ++t4)
#pragma unroll
        for (int h = 0; h < QPG; ++h) {
            const float4 p4 = reinterpret_cast<const float4*>(Sw + h * SST + r0)[t4];
            o[h].x = fmaf(p4.x, v[4 * t4].x, o[h].x);
            o[h].y = fmaf(p4.x, v[4 * t4].y, o[h].y);
            o[h].x = fmaf(p4.y, v[4 * t4 + 1].x, o[h].x);
            o[h].y = fmaf(p4.y, v[4 * t4 + 1].y, o[h].y);
            o[h].x = fmaf(p4.z, v[4 * t4 + 2].x, o[h].x);
            o[h].y = fmaf(p4.z, v[4 * t4 + 2].y, o[h].y);
            o[h].x = fmaf(p4.w, v[4 * t4 + 3].x, o[h].x);
            o[h].y = fmaf(p4.w, v[4 * t4 + 3].y, o[h].y);
        }
}

template <int QPG>
__global__ void __launch_bounds__(TTHREADS, 1) decode_tc_kernel(cx_decode_batch b, float scale,
                                                                 int* flag, unsigned long long* trc, int skip) {
    extern __shared__ __align__(1024) unsigned char smem[];
    if (threadIdx.x == 0) TC_TRACE(1001);  // kernel start (debugging only)
#ifdef CX_EXPERIMENTS
    if (trc && threadIdx.x == 0) trc[2048 + 2 * (blockIdx.y * gridDim.x + blockIdx.x)] = gtime();
#endif
    const TcLayout lay = tc_layout(b.k_syn, QPG);
    const int NS = lay.ns;
    unsigned char* Kh = smem + lay.kh;
    unsigned char* Kl = smem + lay.kl;
    unsigned char* Vhl = smem + lay.vh;  // [V_hi^T ; V_lo^T] as 128 N-rows
    unsigned char* Qh = smem + lay.qo;
    unsigned char* Ql = smem + lay.qo + (size_t)TM * TD * 2;
    float* Op = reinterpret_cast<float*>(smem + lay.op);
    float* Mp = reinterpret_cast<float*>(smem + lay.mp);
    float* Lp = reinterpret_cast<float*>(smem + lay.lp);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + lay.mbar);
    uint32_t* tbase_s = reinterpret_cast<uint32_t*>(smem + lay.tbase);
    volatile int* epi_done = reinterpret_cast<volatile int*>(smem + lay.tbase + 8);  // epilogues completed

    const int lh = blockIdx.x;
    const int l = lh / b.n_kv, g = lh % b.n_kv;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // programmatic dependent launch: the next step may start its prologue as soon as SMs free
    // up; this step's own reads / writes of agent data wait for the previous step
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const bool syn_early = (b.flags & CX_DECODE_SYN_UNCHANGED) != 0;
    const int ks = b.k_syn;
    constexpr int AT = TM / QPG;  // agents per tile
    const bool app = b.new_keys != nullptr;

    // ---- one-time: TMEM (S: NS cols, O: 64 cols), mbarriers, K_syn / V_syn^T ----
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tbase_s)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar[1])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&mbar[2])), "r"(PWARPS));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&mbar[3])), "r"(PWARPS));
        asm volatile("fence.mbarrier_init.release.cluster;");
        *epi_done = 0;
    }
    // barriers / TMEM base visible to all; the private warps start streaming right away
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp >= SWARPS || !syn_early) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (warp < SWARPS) {  // K_syn / V_syn^T staging: synapse warps only (the private rows never read them)
        {  // the first Q tile -> L2 during the staging
            const int a0q = (int)blockIdx.y * AT;
            if (tid < min(AT, b.n_agents - a0q))
                l2_prefetch(b.q + (((size_t)(a0q + tid) * b.n_layers + l) * b.n_q + (size_t)g * QPG) * TD,
                            (uint32_t)(QPG * TD * sizeof(float)));
        }
        const float* sk = b.syn_keys + (size_t)lh * ks * TD;
        // items per pass per thread: all NS * 8 = 1408 items (k <= 176) in ONE pass, so the
        // staging costs two loaded-latency round trips (K, then V) instead of nine
        constexpr int ST = SWARPS * 32, IT = (TNS_MAX * 8 + ST - 1) / ST;
        // K: item = (key j, 8-dim chunk c): two float4 loads, one hi and one lo store
        for (int base = 0; base < NS * 8; base += IT * ST) {
            float4 ka[IT], kb[IT];
#pragma unroll
            for (int k = 0; k < IT; ++k) {
                const int it = base + tid + k * ST, j = it >> 3, c = it & 7;
                ka[k] = kb[k] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (j < ks) ld_row8(sk + (size_t)j * TD + 8 * c, ka[k], kb[k]);
            }
#pragma unroll
            for (int k = 0; k < IT; ++k) {
                const int it = base + tid + k * ST, j = it >> 3, c = it & 7;
                if (j < NS) {
                    const float x[8] = {ka[k].x, ka[k].y, ka[k].z, ka[k].w, kb[k].x, kb[k].y, kb[k].z, kb[k].w};
                    split8_store(x, Kh, Kl, cm_off(j, 8 * c, NS));  // B of S = Q K^T: N = keys, K = dims
                }
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        bar_sync(1, SWARPS * 32);
        if (tid == 0) TC_TRACE(1000);
    }
    // TMEM columns: S [0, NS), O [NS, NS + 128) (P_hi V_hi + P_lo V_hi | P_hi V_lo), P hi / lo after
    const uint32_t tS = *tbase_s, tO = tS + (uint32_t)NS, tPh = tS + (uint32_t)max(256, NS + 2 * TD),
                   tPl = tPh + (uint32_t)(NS / 2);
    const int n_tiles = (b.n_agents + AT - 1) / AT;
    uint32_t tpar = 0;  // tile parity: mbar[0] / mbar[2] phases, double-buffered O_priv / (m, l)

    if (warp < SWARPS) {
        // ======================= synapse warps =======================
        const uint32_t idS = idesc_bf16_f32(TM, NS), idO = idesc_bf16_f32(TM, TD), idO2 = idesc_bf16_f32(TM, 2 * TD);
        const uint32_t trow = tS + ((uint32_t)(warp * 32) << 16);
        const uint32_t trow_ph = tPh + ((uint32_t)(warp * 32) << 16), trow_pl = tPl + ((uint32_t)(warp * 32) << 16);
        const int r_own = warp * 32 + lane;
        uint32_t ph1 = 0;
        // Q tile -> bf16 hi/lo; lane -> (row rb + lane%8, chunk cb + lane/8): 4 lanes read
        // 128 contiguous bytes of a row, 8 lanes store 128 contiguous bytes
        auto stage_q = [&](int tile_q) {
            const int a0q = tile_q * AT;
            const int rows_q = min(AT, b.n_agents - a0q) * QPG;
            // one 256-bit load per (row, 8-dim chunk): a lane reads a whole 32-B sector, and
            // no L1 allocation over the private rows' prefetches
            float x[8][8];
#pragma unroll
            for (int it = 0; it < 8; ++it) {
                const int r = warp * 32 + (it >> 1) * 8 + (lane & 7), c = (it & 1) * 4 + (lane >> 3);
                if (r < rows_q) {
                    const int a = a0q + r / QPG, hh = r % QPG;
                    ld_v8_na(b.q + (((size_t)a * b.n_layers + l) * b.n_q + (size_t)g * QPG + hh) * TD + 8 * c, x[it]);
                } else {
#pragma unroll
                    for (int u = 0; u < 8; ++u) x[it][u] = 0.f;
                }
            }
#pragma unroll
            for (int it = 0; it < 8; ++it) {
                const int r = warp * 32 + (it >> 1) * 8 + (lane & 7), c = (it & 1) * 4 + (lane >> 3);
                split8_store(x[it], Qh, Ql, cm_off(r, 8 * c, TM));
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            bar_sync(1, SWARPS * 32);
        };
        // a Q tile's agents -> L2 (one bulk prefetch of QPG contiguous rows per agent), a
        // tile ahead of stage_q: the staging then waits on L2, not on a DRAM round trip
        auto prefetch_q = [&](int tile_q) {
            const int a0q = tile_q * AT;
            if (tile_q < n_tiles && tid < min(AT, b.n_agents - a0q))
                l2_prefetch(b.q + (((size_t)(a0q + tid) * b.n_layers + l) * b.n_q + (size_t)g * QPG) * TD,
                            (uint32_t)(QPG * TD * sizeof(float)));
        };
        // S = Q K^T on the tensor cores (3 MMAs per 16-wide k-step), completion on mbar[0]
        auto issue_s = [&]() {
            if (tid == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t qlbo = (TM / 8) * 128, klbo = (uint32_t)(NS / 8) * 128;
#pragma unroll
                for (int kk = 0; kk < TD / 16; ++kk) {
                    const uint32_t qo = kk * 2 * qlbo, ko = kk * 2 * klbo;
                    const uint64_t qh = sdesc(su32(Qh) + qo, qlbo, 128), ql = sdesc(su32(Ql) + qo, qlbo, 128);
                    const uint64_t kh = sdesc(su32(Kh) + ko, klbo, 128), kl = sdesc(su32(Kl) + ko, klbo, 128);
#ifndef CX_NEGCTL_BF16_S
                    mma_bf16(tS, ql, kh, idS, kk > 0 ? 1u : 0u);
                    mma_bf16(tS, qh, kl, idS, 1u);
                    mma_bf16(tS, qh, kh, idS, 1u);
#else  // negative control (tests/negctl only, never the product): bf16-only scores
                    (void)ql;
                    (void)kl;
                    mma_bf16(tS, qh, kh, idS, kk > 0 ? 1u : 0u);
#endif
                }
                mma_commit(&mbar[0]);
            }
        };
        // V_syn^T is first needed by the first P.V: staged while the first scores run (or, when
        // the synapse is unchanged since the previous step, before that step has finished)
        auto stage_v = [&]() {
            const float* sv = b.syn_values + (size_t)lh * ks * TD;
            constexpr int ST = SWARPS * 32, IT = (TNS_MAX * 8 + ST - 1) / ST;
            // V^T: item = (dim c, 8-key chunk jc): 8 strided scalar loads (coalesced across lanes)
            for (int base = 0; base < TD * (NS / 8); base += IT * ST) {
                float xv[IT][8];
#pragma unroll
                for (int k = 0; k < IT; ++k) {
                    const int it = base + tid + k * ST, c = it & (TD - 1), jc = it >> 6;
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int j = 8 * jc + u;
                        xv[k][u] = (jc < NS / 8 && j < ks) ? __ldg(sv + (size_t)j * TD + c) : 0.f;
                    }
                }
#pragma unroll
                for (int k = 0; k < IT; ++k) {
                    const int it = base + tid + k * ST, c = it & (TD - 1), jc = it >> 6;
                    // B of O = P V (N = dims, K = keys): hi at N-row c, lo at N-row 64 + c (+1024 B)
                    if (jc < NS / 8) split8_store(xv[k], Vhl, Vhl + cm_off(TD, 0, 2 * TD), cm_off(c, 8 * jc, 2 * TD));
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bar_sync(1, SWARPS * 32);
        };
        if (syn_early) {
            stage_v();
            // the synapse is staged: from here on agent data, which the previous step may write
            asm volatile("griddepcontrol.wait;" ::: "memory");
        }
        // the first tile's scores are issued before the loop; tile i+1's while tile i's P.V runs
        if (!TC_SKIP(1) && (int)blockIdx.y < n_tiles) {
            stage_q(blockIdx.y);
            issue_s();
        }
        if (!syn_early) stage_v();
        int ti = 0;
        for (int tile = blockIdx.y; tile < n_tiles; tile += gridDim.y, ++ti) {
            if (tid == 0) TC_TRACE(ti * 16 + 0);
            prefetch_q(tile + (int)gridDim.y);  // staged during this tile's P.V
            const int a0 = tile * AT;
            const int rows = min(AT, b.n_agents - a0) * QPG;
            const int next = tile + (int)gridDim.y;
            if (TC_SKIP(1)) {  // debugging only (CX_TC_SKIP): keep the hand-off protocol, skip the math
                mbar_wait_sleep(&mbar[2 + tpar], (uint32_t)(ti >> 1) & 1u);
                bar_sync(1, SWARPS * 32);
                if (tid == 0) *epi_done = ti + 1;
                tpar ^= 1u;
                continue;
            }
            mbar_wait_parity(&mbar[0], tpar);  // S of this tile (issued one tile ahead)
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (tid == 0) TC_TRACE(ti * 16 + 2);
            // softmax over the synapse keys, thread per row
            const bool live = r_own < rows;
            float mx = -INFINITY, l_s = 0.f;
            float2 lsum2 = make_float2(0.f, 0.f);
            for (int c0 = 0; c0 < NS; c0 += 16) {
                float v[16];
                tmem_ld16(trow + (uint32_t)c0, v);
                if (c0 + 16 <= ks) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) mx = fmaxf(mx, v[j]);
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (c0 + j < ks) mx = fmaxf(mx, v[j]);
                }
            }
            const float m_s = mx * scale;                   // scale > 0
            const float c2 = scale * 1.4426950408889634f;   // e^{(s - mx) scale} = 2^{s c2 - mx c2}
            const float m2 = live ? mx * c2 : INFINITY;     // padding rows: all weights 0
            if (tid == 0) TC_TRACE(ti * 16 + 3);
            // unnormalised P -> TMEM as packed bf16x2 hi / lo (row = lane, 2 keys per column):
            // the A operand of O = P V_syn, so no shared-memory round trip and one MMA pass
            for (int c0 = 0; c0 < NS; c0 += 16) {
                float v[16];
                tmem_ld16(trow + (uint32_t)c0, v);
                float p[16];
#pragma unroll
                for (int u = 0; u < 8; ++u) {  // packed exponent arguments: v c2 - m2
                    const float2 e = ffma2(make_float2(v[2 * u], v[2 * u + 1]), make_float2(c2, c2), make_float2(-m2, -m2));
                    p[2 * u] = ex2(e.x);
                    p[2 * u + 1] = ex2(e.y);
                }
                if (c0 + 16 > ks) {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (c0 + j >= ks) p[j] = 0.f;
                }
                // P = hi + lo: hi = p truncated to bf16 (exact bits), lo = p - hi (exact in fp32)
                // rounded to bf16; |P - p| <= 2^-17 |p|
                uint32_t hv[8], lv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t b0 = __float_as_uint(p[2 * u]), b1 = __float_as_uint(p[2 * u + 1]);
                    hv[u] = __byte_perm(b0, b1, 0x7632);  // the two high halves, packed bf16x2
                    const float2 lo = add2(make_float2(p[2 * u], p[2 * u + 1]),
                                           make_float2(-__uint_as_float(b0 & 0xFFFF0000u), -__uint_as_float(b1 & 0xFFFF0000u)));
                    const __nv_bfloat162 l2 = __floats2bfloat162_rn(lo.x, lo.y);
                    lv[u] = *reinterpret_cast<const uint32_t*>(&l2);
                    lsum2 = add2(lsum2, make_float2(p[2 * u], p[2 * u + 1]));
                }
                tmem_st8(trow_ph + (uint32_t)(c0 / 2), hv);
                tmem_st8(trow_pl + (uint32_t)(c0 / 2), lv);
            }
            l_s = lsum2.x + lsum2.y;
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            bar_sync(1, SWARPS * 32);  // S of this tile fully read; P in TMEM
            if (tid == 0) TC_TRACE(ti * 16 + 1);
            if (tid == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t vlbo = (2 * TD / 8) * 128;  // K-chunk stride of the 128-row V operand
                for (int kk = 0; kk < NS / 16; ++kk) {
                    const uint32_t vo = kk * 2 * vlbo;
                    // one N = 128 MMA: [P_hi V_hi | P_hi V_lo]; one N = 64: += P_lo V_hi
                    const uint64_t vhl = sdesc(su32(Vhl) + vo, vlbo, 128);
                    mma_bf16_ts(tO, tPh + (uint32_t)(kk * 8), vhl, idO2, kk > 0 ? 1u : 0u);
                    mma_bf16_ts(tO, tPl + (uint32_t)(kk * 8), vhl, idO, 1u);
                }
                mma_commit(&mbar[1]);
                TC_TRACE(ti * 16 + 15);
            }
            // next tile: its Q (the score MMAs of this tile are done with the buffer) and S
            // (this tile's S is dead) while this tile's P.V runs
            if (next < n_tiles) {
                stage_q(next);
                issue_s();
            }
            if (tid == 0) TC_TRACE(ti * 16 + 7);
            mbar_wait_parity(&mbar[1], ph1);  // O = P V_syn complete
            ph1 ^= 1u;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            // epilogue: wait for the private partials, merge, store
            if (tid == 0) TC_TRACE(ti * 16 + 4);
            // every private warp has published this tile.  Private warps may run one tile
            // ahead, so even / odd tiles use separate barriers (no parity aliasing)
            mbar_wait_sleep(&mbar[2 + tpar], (uint32_t)(ti >> 1) & 1u);
            if (tid == 0) TC_TRACE(ti * 16 + 5);
            {
                float* Opt = Op + (size_t)(OP_BUFS == 2 ? tpar : 0) * TM * OPS;
                float v[TD];
                const uint32_t trow_o = tO + ((uint32_t)(warp * 32) << 16);
#pragma unroll
                for (int c0 = 0; c0 < TD; c0 += 16)
                    tmem_ld16x2_sum(trow_o + (uint32_t)c0, trow_o + (uint32_t)(TD + c0), v + c0);
                if (live) {  // merged row -> the O_priv row it came from (in place, own row)
                    const float m_p = Mp[tpar * TM + r_own], l_p = Lp[tpar * TM + r_own];
                    const float m = fmaxf(m_s, m_p);
                    const float as = __expf(m_s - m), ap = __expf(m_p - m);
                    const float inv = 1.0f / (l_s * as + l_p * ap);
                    const float cs = as * inv, cp = ap * inv;
                    float4* op = reinterpret_cast<float4*>(Opt + r_own * OPS);
#pragma unroll
                    for (int c4 = 0; c4 < TD / 4; ++c4) {
                        const float4 pp = op[c4];
                        op[c4] = make_float4(v[4 * c4] * cs + pp.x * cp, v[4 * c4 + 1] * cs + pp.y * cp,
                                             v[4 * c4 + 2] * cs + pp.z * cp, v[4 * c4 + 3] * cs + pp.w * cp);
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                bar_sync(1, SWARPS * 32);  // merged rows in shared memory, TMEM O read
                // coalesced store: a warp instruction writes two whole 256-B rows (a thread per
                // row would put 32 rows' 16-B pieces in one instruction: 32 partial lines)
                for (int e = tid; e < rows * (TD / 4); e += SWARPS * 32) {
                    const int r = e / (TD / 4), c4 = e % (TD / 4);
                    const int a = a0 + r / QPG, hh = r % QPG;
                    float* out = b.out + (((size_t)a * b.n_layers + l) * b.n_q + (size_t)g * QPG + hh) * TD;
                    reinterpret_cast<float4*>(out)[c4] = reinterpret_cast<const float4*>(Opt + r * OPS)[c4];
                }
            }
            bar_sync(1, SWARPS * 32);  // this tile's O_priv buffer fully read
            if (tid == 0) {
                __threadfence_block();
                *epi_done = ti + 1;    // private warps may now overwrite this parity's buffers
                TC_TRACE(ti * 16 + 6);
            }
            tpar ^= 1u;
        }
    } else {
        // ======================= private warps =======================
        const int pw = warp - SWARPS;
        float* Sw = reinterpret_cast<float*>(smem + lay.sw) + pw * QPG * SST;
        static_assert(QPG <= 8, "the score reduce-scatter handles up to 8 q-heads per KV head");
        int ti = 0;
        for (int tile = blockIdx.y; tile < n_tiles; tile += gridDim.y, ++ti) {
            const int a0 = tile * AT;
            const int na = min(AT, b.n_agents - a0);
            bool published = false, op_free = false;
            if (pw == 0 && lane == 0) TC_TRACE(ti * 16 + 8);
            // agents are dealt round-robin over the CTA's whole agent sequence, not per
            // tile: with 18 agents per tile and 12 warps no warp takes 2 every tile
            const int first = (pw - (ti * AT) % PWARPS + PWARPS) % PWARPS;
            for (int ai = first; ai < na; ai += PWARPS) {
                if (TC_SKIP(2)) continue;  // debugging only (CX_TC_SKIP)
                const int a = a0 + ai;
                // stored rows, validated (model.cpp:124-140 capacity check): out of range ->
                // FLAG_TAIL_RANGE, the agent's rows clamped and nothing appended
                int len = __ldg(b.tail_len + a);
                const int cap = b.t_cap - (app ? 1 : 0);
                const bool len_ok = len >= 0 && len <= cap;
                if (!len_ok) {
                    if (lane == 0) atomicOr(flag, FLAG_TAIL_RANGE);
                    len = len < 0 ? 0 : cap;
                }
                const bool appa = app && len_ok;  // this agent appends its new token
                const int nt = len + (appa ? 1 : 0);
                const size_t toff = ((((size_t)a * b.n_layers + l) * b.n_kv + g) * b.t_cap) * TD;
                const size_t noff = (((size_t)a * b.n_layers + l) * b.n_kv + g) * TD;
                const float* tk = b.tail_keys + toff;
                const float* tv = b.tail_values + toff;
                const float* qrow = b.q + (((size_t)a * b.n_layers + l) * b.n_q + (size_t)g * QPG) * TD;
                // q, the new token's K/V row (it is row `len`) and the first K batch are all in
                // flight together; the new row is used from registers and appended (fused).
                float4 qa[QPG], qb[QPG];
#pragma unroll
                for (int h = 0; h < QPG; ++h) {
                    ld_row8(qrow + (size_t)h * TD + 8 * (lane & 7), qa[h], qb[h]);
                }
                float4 nka = make_float4(0.f, 0.f, 0.f, 0.f), nkb = nka;
                float2 nvv = make_float2(0.f, 0.f);
                if (appa) {
                    ld_row8(b.new_keys + noff + 8 * (lane & 7), nka, nkb);
                    nvv = __ldg(reinterpret_cast<const float2*>(b.new_values + noff) + lane);
                }  // (appended at the end of the agent: a store here would hold back every load below)
                // ---- scores of the stored rows [0, len): 16-row batches, then 4-row groups ----
                // K batch 1 and V batches 0-1 go to L1 now (the whole 32-row tail is in flight
                // with q and K batch 0); longer tails are prefetched two batches ahead
                int r0 = 0;
                prefetch_rows16_l1<PB>(tk, PB, len, lane);
                prefetch_rows16_l1<PB>(tv, 0, len, lane);
                prefetch_rows16_l1<PB>(tv, PB, len, lane);
                for (; r0 + PB <= len; r0 += PB) {
                    prefetch_rows16_l1<PB>(tk, r0 + 2 * PB, len, lane);
                    score_rows<QPG, PB / 4, false>(tk, r0, len, qa, qb, Sw, lane, scale);
                }
                for (; r0 < len; r0 += 4) score_rows<QPG, 1, true>(tk, r0, len, qa, qb, Sw, lane, scale);
                if (appa) score_group<QPG>(nka, nkb, len, lane < 8, qa, qb, Sw, lane, scale);
                if (pw == 0 && lane == 0) TC_TRACE(ti * 16 + (ai == first ? 9 : 12));
                __syncwarp();
                // this tile's (Mp, Lp, O_priv) buffers were last read by the epilogue two
                // tiles back: wait for it before the first write of the tile
                if (!published) {
                    wait_epilogues(epi_done, ti - 1);
                    published = true;
                }
                // softmax per q-head over the private rows (weights 0 up to TTAIL); the
                // heads' shuffle reductions are interleaved (independent chains)
                {
                    float s0[QPG], s1[QPG], mh[QPG], lh[QPG];
#pragma unroll
                    for (int h = 0; h < QPG; ++h) {
                        s0[h] = lane < nt ? Sw[h * SST + lane] : -INFINITY;
                        s1[h] = lane + 32 < nt ? Sw[h * SST + lane + 32] : -INFINITY;
                        mh[h] = fmaxf(s0[h], s1[h]);
                    }
#pragma unroll
                    for (int o = 16; o; o >>= 1)
#pragma unroll
                        for (int h = 0; h < QPG; ++h) mh[h] = fmaxf(mh[h], __shfl_xor_sync(0xffffffffu, mh[h], o));
#pragma unroll
                    for (int h = 0; h < QPG; ++h) {
                        const float p0 = lane < nt ? __expf(s0[h] - mh[h]) : 0.f;
                        const float p1 = lane + 32 < nt ? __expf(s1[h] - mh[h]) : 0.f;
                        Sw[h * SST + lane] = p0;
                        Sw[h * SST + lane + 32] = p1;
                        lh[h] = p0 + p1;
                    }
#pragma unroll
                    for (int o = 16; o; o >>= 1)
#pragma unroll
                        for (int h = 0; h < QPG; ++h) lh[h] += __shfl_xor_sync(0xffffffffu, lh[h], o);
                    if (lane == 0)  // this buffer's previous tile was merged two tiles ago
#pragma unroll
                        for (int h = 0; h < QPG; ++h) {
                            Mp[tpar * TM + ai * QPG + h] = mh[h];
                            Lp[tpar * TM + ai * QPG + h] = lh[h];
                        }
                }
                __syncwarp();
                // ---- O_priv = P V_priv (lane: dims 2 lane, 2 lane + 1) ----
                float2 o[QPG];
#pragma unroll
                for (int h = 0; h < QPG; ++h) o[h] = make_float2(0.f, 0.f);
                r0 = 0;
                {  // the next agent's q and first K batch land in L1 during this mix
                    int na_t = ai + PWARPS, nt_tile = tile;
                    if (na_t >= na) {
                        na_t = (pw - ((ti + 1) * AT) % PWARPS + PWARPS) % PWARPS;
                        nt_tile = tile + (int)gridDim.y;
                    }
                    const int an = nt_tile * AT + na_t;
                    if (nt_tile < n_tiles && an < b.n_agents && na_t < AT) {
                        const size_t off = ((((size_t)an * b.n_layers + l) * b.n_kv + g) * b.t_cap) * TD;
                        prefetch_rows16_l1<PB>(b.tail_keys + off, 0, b.t_cap, lane);
                        const float* qn = b.q + (((size_t)an * b.n_layers + l) * b.n_q + (size_t)g * QPG) * TD;
                        if (lane < 2 * QPG) asm volatile("prefetch.global.L1 [%0];" ::"l"(qn + lane * 32));
                    }
                }
                for (; r0 + PB <= len; r0 += PB) {
                    prefetch_rows16_l1<PB>(tv, r0 + 2 * PB, len, lane);
                    mix_rows<QPG, PB, false>(tv, r0, len, Sw, o, lane);
                }
                for (; r0 < len; r0 += 4) mix_rows<QPG, 4, true>(tv, r0, len, Sw, o, lane);
                if (appa)
#pragma unroll
                    for (int h = 0; h < QPG; ++h) {
                        const float p = Sw[h * SST + len];
                        o[h].x = fmaf(p, nvv.x, o[h].x);
                        o[h].y = fmaf(p, nvv.y, o[h].y);
                    }
                if (pw == 0 && lane == 0) TC_TRACE(ti * 16 + (ai == first ? 10 : 13));
                if (OP_BUFS == 1 && !op_free) {  // single O_priv buffer: last tile's epilogue must be done
                    wait_epilogues(epi_done, ti);
                    op_free = true;
                }
#pragma unroll
                for (int h = 0; h < QPG; ++h) {
                    const int r = ai * QPG + h;
                    reinterpret_cast<float2*>(Op + ((size_t)(OP_BUFS == 2 ? tpar : 0) * TM + r) * OPS)[lane] = o[h];
                }
                if (appa) {  // the fused append of the new token's K/V (row len; never read above)
                    if (lane < 8) {
                        reinterpret_cast<float4*>(b.tail_keys + toff + (size_t)len * TD)[2 * lane] = nka;
                        reinterpret_cast<float4*>(b.tail_keys + toff + (size_t)len * TD)[2 * lane + 1] = nkb;
                    }
                    reinterpret_cast<float2*>(b.tail_values + toff + (size_t)len * TD)[lane] = nvv;
                }
                __syncwarp();  // Sw reuse
            }
            // Arrive only once the epilogue two tiles back is done, even with no agents: the
            // barrier of this tile's parity then never runs a phase ahead of the synapse warps.
            if (!published) wait_epilogues(epi_done, ti - 1);
            if (lane == 0 && pw == 0) TC_TRACE(ti * 16 + 11);
            if (lane == 0 && pw == PWARPS - 1) TC_TRACE(ti * 16 + 14);
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&mbar[2 + tpar])) : "memory");
            tpar ^= 1u;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
#ifdef CX_EXPERIMENTS
    if (trc && threadIdx.x == 0) trc[2048 + 2 * (blockIdx.y * gridDim.x + blockIdx.x) + 1] = gtime();
#endif
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tbase_s), "r"(512));
}

}  // namespace

bool decode_tc_launch(cx_ctx* ctx, const cx_decode_batch& b, cudaStream_t s) {
    const int qpg = b.n_q / b.n_kv;
    if (b.d_k != TD || b.k_syn < 1 || b.k_syn > TNS_MAX || b.t_cap > TTAIL) return false;
    // 256-bit loads of q, K rows, the new key and K_syn; 16-byte accesses elsewhere
    auto al = [](const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; };
    if (!al(b.q, 32) || !al(b.tail_keys, 32) || !al(b.new_keys, 32) || !al(b.syn_keys, 32) || !al(b.out, 16) ||
        !al(b.tail_values, 16) || !al(b.new_values, 16) || !al(b.syn_values, 16))
        return false;
    const TcLayout lay = tc_layout(b.k_syn, qpg);
    static int max_optin = -1;
    if (max_optin < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    }
    if (lay.total > (size_t)max_optin) return false;
    void (*kern)(cx_decode_batch, float, int*, unsigned long long*, int) = nullptr;
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
    // one resident CTA per SM: fill the SMs in a single wave
    int per_lh = std::max(1, std::min(n_tiles, sms / n_lh));
    if (ctx->opt.decode_ctas_per_lh > 0) per_lh = std::max(1, std::min(n_tiles, ctx->opt.decode_ctas_per_lh));
    size_t smem = lay.total;
    unsigned long long* trc_arg = nullptr;
    int skip = 0;
#ifdef CX_EXPERIMENTS
    // CX_TC_SMEM_PAD=bytes: reserve extra shared memory, i.e. shrink the L1 carveout, to
    // measure how the private-row stream depends on L1 capacity
    if (getenv("CX_TC_SMEM_PAD")) smem += (size_t)atol(getenv("CX_TC_SMEM_PAD"));
    if (smem > (size_t)max_optin) return false;
    static unsigned long long* trc = nullptr;
    const bool tracing = getenv("CX_TC_TRACE") != nullptr;
    if (tracing && !trc) {
        CX_CUDA(cudaMalloc(&trc, 8192 * sizeof(unsigned long long)));
        CX_CUDA(cudaMemset(trc, 0, 8192 * sizeof(unsigned long long)));
    }
    if (tracing) trc_arg = trc;
    skip = getenv("CX_TC_SKIP") ? atoi(getenv("CX_TC_SKIP")) : 0;
    if (skip) {  // timing experiments only: say so once, loudly
        static bool warned = false;
        if (!warned) {
            fprintf(stderr, "cortex_b200: CX_TC_SKIP=%d is set -- decode outputs are NOT valid (timing experiments only)\n",
                    skip);
            warned = true;
        }
    }
#endif
    kernel_smem(kern, smem);
    {
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3((unsigned)n_lh, (unsigned)per_lh);
        lc.blockDim = dim3(TTHREADS);
        lc.dynamicSmemBytes = smem;
        lc.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (griddepcontrol in the kernel)
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = attr;
        lc.numAttrs = 1;
        CX_CUDA(cudaLaunchKernelEx(&lc, kern, b, (float)(1.0 / std::sqrt((double)b.d_k)), ctx->d_flag, trc_arg, skip));
        count_launch();
    }
#ifdef CX_EXPERIMENTS
    if (tracing) {  // debugging only: per-tile phase times of CTA (0, 0), us since the staging ended
        std::vector<unsigned long long> h(8192);
        CX_CUDA(cudaStreamSynchronize(s));
        CX_CUDA(cudaMemcpy(h.data(), trc, h.size() * sizeof(h[0]), cudaMemcpyDeviceToHost));
        const double t0 = (double)h[1000];
        fprintf(stderr, "decode_tc trace: grid %d x %d, K/V_syn staging %.2f us\n", n_lh, per_lh,
                (h[1000] - h[1001]) / 1e3);
        for (int ti = 0; ti < 62 && h[ti * 16]; ++ti) {
            fprintf(stderr, "tile %2d syn:", ti);
            for (int k = 0; k < 8; ++k) fprintf(stderr, " %7.2f", (h[ti * 16 + k] - t0) / 1e3);
            fprintf(stderr, " pv-issued %7.2f", (h[ti * 16 + 15] - t0) / 1e3);
            fprintf(stderr, " | priv0:");
            for (int k = 8; k < 15; ++k) fprintf(stderr, " %7.2f", h[ti * 16 + k] ? (h[ti * 16 + k] - t0) / 1e3 : -1.0);
            fprintf(stderr, "\n");
        }
        {  // every CTA's start / end (us, from the first start)
            const int nc = n_lh * per_lh;
            unsigned long long s0 = ~0ull, s1 = 0, e0 = ~0ull, e1 = 0;
            double dur = 0;
            for (int i = 0; i < nc; ++i) {
                const unsigned long long a = h[2048 + 2 * i], b = h[2048 + 2 * i + 1];
                s0 = std::min(s0, a); s1 = std::max(s1, a); e0 = std::min(e0, b); e1 = std::max(e1, b);
                dur += (double)(b - a);
            }
            fprintf(stderr, "decode_tc CTAs: starts %.2f..%.2f us, ends %.2f..%.2f us, mean duration %.2f us\n", 0.0,
                    (s1 - s0) / 1e3, (e0 - s0) / 1e3, (e1 - s0) / 1e3, dur / nc / 1e3);
        }
        CX_CUDA(cudaMemset(trc, 0, 8192 * sizeof(unsigned long long)));
    }
#endif
    return true;
}

}  // namespace cx

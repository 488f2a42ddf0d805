// tcgen05.mma issue-rate microbenchmark (tools only): one CTA per SM, thread 0
// issues `reps` x `tiles` kind::f16 MMAs (M = 128, K = 16, N given) with A from
// shared memory (SS) or tensor memory (TS), k-step-major order over `tiles`
// independent accumulators, then commit + wait.  Prints cycles per MMA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
__global__ void rate(int n, int tiles, int ts, int reps, long long* out, int issuers, int elect) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tbase_s;
    __shared__ __align__(8) uint64_t mbar;
    const int tid = threadIdx.x;
    for (int e = tid; e < (12 * 16384 + 8192) / 16; e += blockDim.x) reinterpret_cast<uint4*>(sm)[e] = make_uint4(0, 0, 0, 0);
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tbase_s)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tb = tbase_s;
    const uint32_t idesc = (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    unsigned char* bop = sm + 12 * 16384;
    long long t0 = 0, t1 = 0, tiss = 0;
    const int me = tid >> 5;
    if (((tid & 31) == 0 || elect) && me < issuers) {
        uint32_t ph = 0;
        for (int it = 0; it < 2; ++it) {  // it 0 warms up
            t0 = clock64();
            for (int r = 0; r < reps; ++r) {
                for (int kk = 0; kk < 4; ++kk) {
                    const uint64_t bd = sdesc(su32(bop) + kk * 2 * 128 * (n / 8), 128 * (n / 8), 128);
                    for (int j = me; j < tiles; j += issuers) {
                        const uint32_t dt = tb + (uint32_t)(n * j) % 256;
                        if (!ts) {
                            const uint64_t ad = sdesc(su32(sm + (j % 12) * 16384) + kk * 2 * 2048, 2048, 128);
                            if (elect)
                                asm volatile("{ .reg .pred p, e; setp.ne.b32 p, %4, 0; elect.sync _|e, 0xffffffff;\n"
                                             "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                                             ::"r"(dt), "l"(ad), "l"(bd), "r"(idesc), "r"(kk > 0 ? 1u : 0u) : "memory");
                            else
                                asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                                             ::"r"(dt), "l"(ad), "l"(bd), "r"(idesc), "r"(kk > 0 ? 1u : 0u) : "memory");
                        } else {
                            const uint32_t at = tb + 256 + 32 * (j % 8) + 8 * kk;
                            if (elect)
                                asm volatile("{ .reg .pred p, e; setp.ne.b32 p, %4, 0; elect.sync _|e, 0xffffffff;\n"
                                             "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }"
                                             ::"r"(dt), "r"(at), "l"(bd), "r"(idesc), "r"(kk > 0 ? 1u : 0u) : "memory");
                            else
                                asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }"
                                             ::"r"(dt), "r"(at), "l"(bd), "r"(idesc), "r"(kk > 0 ? 1u : 0u) : "memory");
                        }
                    }
                }
            }
            tiss = clock64();
            if (me == 0 && (tid & 31) == 0) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar)) : "memory");
            uint32_t ok = 0;
            do {
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(ok) : "r"(su32(&mbar)), "r"(ph) : "memory");
            } while (!ok && tid == 0);
            if (elect) __syncwarp();
            ph ^= 1u;
            t1 = clock64();
        }
        if (tid == 0) { out[blockIdx.x] = t1 - t0; out[148 + blockIdx.x] = tiss - t0; }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}
// precomputed operands: 8 MMAs (2 tiles x 4 k-steps) per iteration, no address math in the loop
__global__ void rate_pre(int reps, long long* out) {
    __shared__ uint32_t tbase_s;
    __shared__ __align__(8) uint64_t mbar;
    __shared__ __align__(1024) unsigned char bop[1024];
    const int tid = threadIdx.x;
    for (int e = tid; e < 64; e += blockDim.x) reinterpret_cast<uint4*>(bop)[e] = make_uint4(0, 0, 0, 0);
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tbase_s)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tb = tbase_s;
    const uint32_t idesc = (1u << 4) | (1u << 17) | ((uint32_t)(128 >> 4) << 24);
    if (tid < 32) {
        uint64_t bd[4];
        for (int kk = 0; kk < 4; ++kk) bd[kk] = sdesc(su32(bop) + kk * 256, 128, 128);
        long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                for (int j = 0; j < 2; ++j)
                    asm volatile("{ .reg .pred p, e; setp.ne.b32 p, %4, 0; elect.sync _|e, 0xffffffff;\n"
                                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }"
                                 ::"r"(tb + 8 * j), "r"(tb + 256 + 32 * j + 8 * kk), "l"(bd[kk]), "r"(idesc), "r"(kk)
                                 : "memory");
        }
        if (tid == 0) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar)) : "memory");
        uint32_t ok = 0;
        do {
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(ok) : "r"(su32(&mbar)), "r"(0u) : "memory");
        } while (!ok);
        long long t1 = clock64();
        if (tid == 0) out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

int main() {
    long long* d;
    cudaMalloc(&d, sizeof(long long) * 296);
    cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384 + 8192);
    {
        rate_pre<<<148, 128>>>(64, d);
        long long h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("TS precomputed, warp-uniform: %7.1f cycles / MMA  err=%s\n", (double)h[0] / (64 * 8),
               cudaGetErrorString(cudaGetLastError()));
    }
    for (int ts = 0; ts < 2; ++ts)
        for (int el = 0; el < 2; ++el)
            for (int iss : {1, 4}) {
                const int n = 8, reps = 8, tiles = 22;
                rate<<<148, 128, 12 * 16384 + 8192>>>(n, tiles, ts, reps, d, iss, el);
                long long h[296];
                cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
                const double per = (double)h[0] / (reps * tiles * 4);
                printf("%s N=%3d tiles=%2d issuers=%d elect=%d: %7.1f cycles / MMA, issue loop %7.1f / MMA  err=%s\n",
                       ts ? "TS" : "SS", n, tiles, iss, el, per, (double)h[148] / (reps * tiles * 4),
                       cudaGetErrorString(cudaGetLastError()));
            }
    return 0;
}

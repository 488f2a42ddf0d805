// Standalone tcgen05 check (tools only): D[128 x N] = A[128 x 64] . B[N x 64]^T,
// bf16 operands in the K-major SWIZZLE_NONE core-matrix layout, fp32 accumulator
// in TMEM, read back with tcgen05.ld.32x32b.  Validates descriptor encodings.
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <vector>

constexpr int M = 128, K = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// core-matrix layout offset (bytes) of element (r, k) in an R x K bf16 K-major tile:
// core matrices of 8 rows x 16 B; row groups contiguous (SBO = 128 B), K chunks of 8
// elements at stride LBO = (R/8) * 128 B.
__host__ __device__ inline uint32_t cm_off(int r, int k, int R) {
    return ((k >> 3) * (R >> 3) + (r >> 3)) * 128 + (r & 7) * 16 + (k & 7) * 2;
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version (sm_100)
    return d;                // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

__host__ __device__ inline uint32_t idesc_bf16(int m, int n) {
    uint32_t d = 0;
    d |= 1u << 4;          // c_format F32
    d |= 1u << 7;          // a_format BF16
    d |= 1u << 10;         // b_format BF16
    d |= (uint32_t)(n >> 3) << 17;
    d |= (uint32_t)(m >> 4) << 24;
    return d;
}

template <int N>
__global__ void umma_gemm(const float* A, const float* B, float* D, int swap_lbo_sbo) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __nv_bfloat16* As = reinterpret_cast<__nv_bfloat16*>(sm);
    __nv_bfloat16* Bs = reinterpret_cast<__nv_bfloat16*>(sm + M * K * 2);
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t mbar;
    const int tid = threadIdx.x;
    for (int e = tid; e < M * K; e += blockDim.x) {
        const int r = e / K, k = e % K;
        As[cm_off(r, k, M) / 2] = __float2bfloat16_rn(A[e]);
    }
    for (int e = tid; e < N * K; e += blockDim.x) {
        const int r = e / K, k = e % K;
        Bs[cm_off(r, k, N) / 2] = __float2bfloat16_rn(B[e]);
    }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = tmem_base;
    if (tid == 0) {
        const uint32_t idesc = idesc_bf16(M, N);
        const uint32_t a_lbo = (M / 8) * 128, b_lbo = (N / 8) * 128, sbo = 128;
        for (int ks = 0; ks < K / 16; ++ks) {
            const uint32_t a_addr = smem_u32(As) + ks * 2 * a_lbo;
            const uint32_t b_addr = smem_u32(Bs) + ks * 2 * b_lbo;
            const uint64_t ad = swap_lbo_sbo ? sdesc(a_addr, sbo, a_lbo) : sdesc(a_addr, a_lbo, sbo);
            const uint64_t bd = swap_lbo_sbo ? sdesc(b_addr, sbo, b_lbo) : sdesc(b_addr, b_lbo, sbo);
            const uint32_t acc = ks > 0 ? 1u : 0u;
            asm volatile(
                "{ .reg .pred p; setp.ne.b32 p, %4, 0; "
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(tbase),
                "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&mbar))
                     : "memory");
    }
    // wait for the MMAs
    {
        uint32_t ok = 0;
        do {
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                         : "=r"(ok)
                         : "r"(smem_u32(&mbar))
                         : "memory");
        } while (!ok);
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // epilogue: warp w (w < 4) reads lanes 32w..32w+31, 16 columns at a time
    const int w = tid >> 5, lane = tid & 31;
    if (w < 4) {
        const int row = 32 * w + lane;
        for (int c0 = 0; c0 < N; c0 += 16) {
            uint32_t v[16];
            const uint32_t taddr = tbase + ((uint32_t)(32 * w) << 16) + (uint32_t)c0;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = __uint_as_float(v[j]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(256));
}

static float bf(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

template <int N>
int run(int swap) {
    std::vector<float> A(M * K), B(N * K), D(M * N, -1.f);
    srand(1);
    for (auto& x : A) x = (rand() / (float)RAND_MAX) * 2 - 1;
    for (auto& x : B) x = (rand() / (float)RAND_MAX) * 2 - 1;
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    const int smem = (M + N) * K * 2;
    cudaFuncSetAttribute(umma_gemm<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    umma_gemm<N><<<1, 128, smem>>>(dA, dB, dD, swap);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("N=%d swap=%d: CUDA error %s\n", N, swap, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
            double r = 0;
            for (int k = 0; k < K; ++k) r += (double)bf(A[i * K + k]) * bf(B[j * K + k]);
            maxerr = fmax(maxerr, fabs(r - D[i * N + j]));
        }
    printf("N=%d swap=%d: max abs err %.3e  (D[0]=%f D[last]=%f)\n", N, swap, maxerr, D[0], D[M * N - 1]);
    cudaFree(dA); cudaFree(dB); cudaFree(dD);
    return 0;
}

int main() {
    run<64>(0);
    run<64>(1);
    run<176>(0);
    return 0;
}

// Standalone tcgen05 check (tools only): D[128 x N] = A[128 x K] . B[N x K]^T with
// the A operand in TENSOR MEMORY (written by tcgen05.st as packed bf16x2, row =
// TMEM lane, two consecutive k per 32-bit column) and B in shared memory
// (K-major SWIZZLE_NONE core-matrix layout).  Validates the ".kind::f16 [d], [a],
// b_desc" form used for P.V in decode_tc.cu.
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <vector>

constexpr int M = 128, K = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__host__ __device__ inline uint32_t cm_off(int r, int k, int R) {
    return ((k >> 3) * (R >> 3) + (r >> 3)) * 128 + (r & 7) * 16 + (k & 7) * 2;
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

__host__ __device__ inline uint32_t idesc_bf16(int m, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

template <int N>
__global__ void umma_ts(const float* A, const float* B, float* D) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __nv_bfloat16* Bs = reinterpret_cast<__nv_bfloat16*>(sm);
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t mbar;
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    for (int e = tid; e < N * K; e += blockDim.x) {
        const int r = e / K, k = e % K;
        Bs[cm_off(r, k, N) / 2] = __float2bfloat16_rn(B[e]);
    }
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(256));
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
    const uint32_t tA = tbase + 128;  // A occupies K/2 = 32 columns from column 128
    // A row (32 w + lane) -> TMEM lane, packed bf16x2 (k even in the low half)
    {
        const int row = 32 * w + lane;
        uint32_t v[K / 2];
        for (int c = 0; c < K / 2; ++c) {
            __nv_bfloat162 h2 = __floats2bfloat162_rn(A[row * K + 2 * c], A[row * K + 2 * c + 1]);
            v[c] = *reinterpret_cast<uint32_t*>(&h2);
        }
        for (int c0 = 0; c0 < K / 2; c0 += 8) {
            const uint32_t taddr = tA + ((uint32_t)(32 * w) << 16) + (uint32_t)c0;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
                         "r"(v[c0]), "r"(v[c0 + 1]), "r"(v[c0 + 2]), "r"(v[c0 + 3]), "r"(v[c0 + 4]), "r"(v[c0 + 5]),
                         "r"(v[c0 + 6]), "r"(v[c0 + 7]));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t idesc = idesc_bf16(M, N);
        const uint32_t b_lbo = (N / 8) * 128;
        for (int ks = 0; ks < K / 16; ++ks) {
            const uint64_t bd = sdesc(smem_u32(Bs) + ks * 2 * b_lbo, b_lbo, 128);
            const uint32_t a_t = tA + (uint32_t)(ks * 8);
            const uint32_t acc = ks > 0 ? 1u : 0u;
            asm volatile(
                "{ .reg .pred p; setp.ne.b32 p, %4, 0; "
                "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }" ::"r"(tbase),
                "r"(a_t), "l"(bd), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar))
                     : "memory");
    }
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
    {
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
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(256));
}

static float bf(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

template <int N>
int run() {
    std::vector<float> A(M * K), B(N * K), D(M * N, -1.f);
    srand(3);
    for (auto& x : A) x = (rand() / (float)RAND_MAX) * 2 - 1;
    for (auto& x : B) x = (rand() / (float)RAND_MAX) * 2 - 1;
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    const int smem = N * K * 2;
    cudaFuncSetAttribute(umma_ts<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    umma_ts<N><<<1, 128, smem>>>(dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("N=%d: CUDA error %s\n", N, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
            double r = 0;
            for (int k = 0; k < K; ++k) r += (double)bf(A[i * K + k]) * bf(B[j * K + k]);
            maxerr = fmax(maxerr, fabs(r - D[i * N + j]));
        }
    printf("TS N=%d: max abs err %.3e (D[0]=%f D[last]=%f)\n", N, maxerr, D[0], D[M * N - 1]);
    cudaFree(dA); cudaFree(dB); cudaFree(dD);
    return maxerr < 1e-3 ? 0 : 2;
}

int main() {
    int rc = run<64>();
    rc |= run<128>();
    return rc;
}

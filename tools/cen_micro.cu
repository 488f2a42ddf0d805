// Centroid-kernel bound finder (tools only): the TMA ring of centroid_tma_kernel with
// (A) the fp64 add chain, (B) the ring alone (one add per stage), (C) the add chain over
// shared memory without waiting for any copy.  48 groups x 8192 rows x 64 dims.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int ROWS = 32, NST = 16, DIM = 64;
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int MODE>
__global__ void __launch_bounds__(256) k(const float* X, double* out, int L) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm);
    float* ring = reinterpret_cast<float*>(sm + 256);
    const int g = blockIdx.x, j = threadIdx.x;
    const float* base = X + (size_t)g * L * DIM;
    const int nst = L / ROWS;
    if (j == 0) {
        for (int i = 0; i < NST; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(full + i)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    auto issue = [&](int st, int slot) {
        const uint32_t bytes = ROWS * DIM * 4;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(full + slot)), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su(ring + (size_t)slot * ROWS * DIM)), "l"(base + (size_t)st * ROWS * DIM), "r"(bytes), "r"(su(full + slot))
                     : "memory");
    };
    if (MODE != 2 && j == 0)
        for (int st = 0; st < NST; ++st) issue(st, st);
    double acc = 0.0;
    int slot = 0;
    uint32_t par = 0;
    for (int st = 0; st < nst; ++st) {
        if (MODE != 2) {
            uint32_t ok = 0;
            do {
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(ok) : "r"(su(full + slot)), "r"(par) : "memory");
            } while (!ok);
        }
        const float* buf = ring + (size_t)slot * ROWS * DIM;
        if (MODE == 1) {
            acc = __dadd_rn(acc, (double)buf[j]);
        } else {
#pragma unroll
            for (int r = 0; r < ROWS; ++r) acc = __dadd_rn(acc, (double)buf[r * DIM + j]);
        }
        __syncthreads();
        if (MODE != 2 && j == 0 && st + NST < nst) issue(st + NST, slot);
        if (++slot == NST) { slot = 0; par ^= 1u; }
    }
    out[g * DIM + j] = acc;
}
int main() {
    const int G = 48, L = 8192;
    float* X; double* o;
    cudaMalloc(&X, sizeof(float) * G * L * DIM);
    cudaMemset(X, 0, sizeof(float) * G * L * DIM);
    cudaMalloc(&o, sizeof(double) * G * DIM);
    const size_t smem = 256 + (size_t)NST * ROWS * DIM * 4;
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    const char* names[3] = {"ring + add chain", "ring only", "add chain only"};
    for (int rep = 0; rep < 2; ++rep)
        for (int m = 0; m < 3; ++m) {
            cudaEventRecord(a);
            for (int i = 0; i < 5; ++i) {
                if (m == 0) k<0><<<G, DIM, smem>>>(X, o, L);
                if (m == 1) k<1><<<G, DIM, smem>>>(X, o, L);
                if (m == 2) k<2><<<G, DIM, smem>>>(X, o, L);
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("%-18s %.1f us\n", names[m], ms * 1000 / 5);
        }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}

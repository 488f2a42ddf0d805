// Microbenchmark (tools only): dependent-chain latency and throughput of the
// fp64 / fp32 ops the selection uses, on the GPU box.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_dadd(double* out, double x, int n, long long* cyc) {
    double a = x, b = x * 0.5;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { a = __dadd_rn(a, b); }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_dmul(double* out, double x, int n, long long* cyc) {
    double a = x, b = 1.0000001;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { a = __dmul_rn(a, b); }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_fadd(float* out, float x, int n, long long* cyc) {
    float a = x, b = x * 0.5f;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { a = __fadd_rn(a, b); }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_dsqrt(double* out, double x, int n, long long* cyc) {
    double a = x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { a = __dsqrt_rn(a) + 1.0; }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_ddiv(double* out, double x, int n, long long* cyc) {
    double a = x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { a = __ddiv_rn(1.5, a); }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
// throughput: 8 independent chains per thread, many warps
__global__ void tput_dadd(double* out, double x, int n) {
    double a0 = x, a1 = x + 1, a2 = x + 2, a3 = x + 3, a4 = x + 4, a5 = x + 5, a6 = x + 6, a7 = x + 7, b = 0.5;
    for (int i = 0; i < n; ++i) {
        a0 = __dadd_rn(a0, b); a1 = __dadd_rn(a1, b); a2 = __dadd_rn(a2, b); a3 = __dadd_rn(a3, b);
        a4 = __dadd_rn(a4, b); a5 = __dadd_rn(a5, b); a6 = __dadd_rn(a6, b); a7 = __dadd_rn(a7, b);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void tput_ffma(float* out, float x, int n) {
    float a0 = x, a1 = x + 1, a2 = x + 2, a3 = x + 3, a4 = x + 4, a5 = x + 5, a6 = x + 6, a7 = x + 7, b = 0.5f;
    for (int i = 0; i < n; ++i) {
        a0 = __fmaf_rn(a0, b, b); a1 = __fmaf_rn(a1, b, b); a2 = __fmaf_rn(a2, b, b); a3 = __fmaf_rn(a3, b, b);
        a4 = __fmaf_rn(a4, b, b); a5 = __fmaf_rn(a5, b, b); a6 = __fmaf_rn(a6, b, b); a7 = __fmaf_rn(a7, b, b);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

int main1() {
    double* dd; float* df; long long* cyc;
    cudaMalloc(&dd, 1 << 26); cudaMalloc(&df, 1 << 26); cudaMallocManaged(&cyc, 8);
    const int n = 4096;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    lat_dadd<<<1, 32>>>(dd, 1.0, n, cyc); cudaDeviceSynchronize();
    lat_dadd<<<1, 32>>>(dd, 1.0, n, cyc); cudaDeviceSynchronize();
    printf("DADD latency  %.2f cyc\n", (double)*cyc / n);
    lat_dmul<<<1, 32>>>(dd, 1.0, n, cyc); cudaDeviceSynchronize();
    printf("DMUL latency  %.2f cyc\n", (double)*cyc / n);
    lat_fadd<<<1, 32>>>(df, 1.0f, n, cyc); cudaDeviceSynchronize();
    printf("FADD latency  %.2f cyc\n", (double)*cyc / n);
    lat_dsqrt<<<1, 32>>>(dd, 2.0, n, cyc); cudaDeviceSynchronize();
    printf("DSQRT(+add) latency %.2f cyc\n", (double)*cyc / n);
    lat_ddiv<<<1, 32>>>(dd, 2.0, n, cyc); cudaDeviceSynchronize();
    printf("DDIV latency  %.2f cyc\n", (double)*cyc / n);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    const int blocks = sms * 8, threads = 256, it = 4096;
    tput_dadd<<<blocks, threads>>>(dd, 1.0, 16); cudaDeviceSynchronize();
    cudaEventRecord(e0); tput_dadd<<<blocks, threads>>>(dd, 1.0, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * it * 8;
    printf("DADD throughput %.1f Gop/s = %.1f /clk/SM (clock %d MHz attr)\n", ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    tput_ffma<<<blocks, threads>>>(df, 1.0f, 16); cudaDeviceSynchronize();
    cudaEventRecord(e0); tput_ffma<<<blocks, threads>>>(df, 1.0f, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA throughput %.1f Gop/s = %.1f /clk/SM\n", ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk * 1e3));
    return 0;
}

// ---- exact squared-distance chain microbench (appended) ----
__global__ void chain_sq(const float* __restrict__ xin, const float* __restrict__ bin, double* out, int reps,
                         long long* cyc) {
    __shared__ float xs[64 * 65];
    __shared__ float bs[64];
    for (int i = threadIdx.x; i < 64 * 65; i += blockDim.x) xs[i] = xin[i % 256];
    for (int i = threadIdx.x; i < 64; i += blockDim.x) bs[i] = bin[i];
    __syncthreads();
    const float* row = xs + threadIdx.x * 65;
    double acc = 0.0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int c = 0; c < 64; ++c) {
            const double d = __dsub_rn((double)row[c], (double)bs[c]);
            acc = __dadd_rn(acc, __dmul_rn(d, d));
        }
    }
    long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void tput_f2f(double* out, float x, int n) {
    float a0 = x, a1 = x + 1, a2 = x + 2, a3 = x + 3;
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    for (int i = 0; i < n; ++i) {
        s0 = (double)a0; s1 = (double)a1; s2 = (double)a2; s3 = (double)a3;
        a0 = __uint_as_float(__double2hiint(s0) ^ 1); a1 = __uint_as_float(__double2hiint(s1) ^ 1);
        a2 = __uint_as_float(__double2hiint(s2) ^ 1); a3 = __uint_as_float(__double2hiint(s3) ^ 1);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}
int main2() {
    float *x, *b; double* o; long long* cyc;
    cudaMalloc(&x, 4096); cudaMalloc(&b, 4096); cudaMalloc(&o, 1 << 20); cudaMallocManaged(&cyc, 8);
    cudaMemset(x, 0, 4096); cudaMemset(b, 0, 4096);
    for (int th : {1, 32, 64}) {
        chain_sq<<<1, th>>>(x, b, o, 1, cyc); cudaDeviceSynchronize();
        chain_sq<<<1, th>>>(x, b, o, 16, cyc); cudaDeviceSynchronize();
        printf("exact_sq chain, %d threads: %.1f cycles per 64-term sum\n", th, (double)*cyc / 16);
    }
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
    tput_f2f<<<sms * 8, 256>>>(o, 1.0f, 16); cudaDeviceSynchronize();
    cudaEventRecord(e0); tput_f2f<<<sms * 8, 256>>>(o, 1.0f, 4096); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)sms * 8 * 256 * 4096 * 4;
    printf("F2F.F64.F32 (+int ops) throughput %.1f /clk/SM\n", ops / (ms * 1e-3) / sms / 1.965e9);
    return 0;
}
int main() { main1(); return main2(); }

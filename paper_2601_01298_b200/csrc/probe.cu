// probe.cu -- on-box peak measurement for the selection roofline (SURVEY.md §8(d):
// "measure the fp64/fp32 peaks on the box; only HBM and BF16 are in
// MEASURED_PEAKS.json").  The selection's exact arithmetic is unfused fp64
// add / mul (the reference's operation order, no FMA), so its ceiling is the
// DADD / DMUL issue rate, measured here with independent dependency chains on
// every SM.
#include "cx_internal.cuh"

namespace cx {
namespace {

constexpr int CHAINS = 8;

__global__ void __launch_bounds__(256) fp64_rate_kernel(double* out, double x, int n) {
    double a[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) a[c] = x + c;
    const double b = 0.5, m = 1.0000000001;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) a[c] = (c & 1) ? __dmul_rn(a[c], m) : __dadd_rn(a[c], b);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += a[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace
}  // namespace cx

using namespace cx;

// fp64 add / mul operations per second (one op per DADD or DMUL), whole device.
extern "C" cx_status cx_probe_fp64_rate(cx_ctx* c, double* ops_per_s) {
    return guard(__func__, [&] {
        if (!c || !ops_per_s) fail(CX_INVALID_ARGUMENT, "null ctx/out");
        CX_CUDA(cudaSetDevice(c->device));
        const int blocks = c->num_sms * 8, threads = 256, n = 4096;
        double* out = nullptr;
        CX_CUDA(cudaMalloc(&out, sizeof(double) * blocks * threads));
        cudaEvent_t e0, e1;
        CX_CUDA(cudaEventCreate(&e0));
        CX_CUDA(cudaEventCreate(&e1));
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
            CX_CUDA(cudaEventRecord(e0, c->stream));
            fp64_rate_kernel<<<blocks, threads, 0, c->stream>>>(out, 1.0, n);
            check_launch("fp64_rate_kernel");
            CX_CUDA(cudaEventRecord(e1, c->stream));
            CX_CUDA(cudaEventSynchronize(e1));
            float ms = 0.f;
            CX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            if (rep > 0) best = std::min(best, ms);  // rep 0 warms up
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaFree(out);
        *ops_per_s = (double)blocks * threads * n * CHAINS / (best * 1e-3);
    });
}

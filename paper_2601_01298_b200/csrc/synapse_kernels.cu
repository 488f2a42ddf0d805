// synapse_kernels.cu -- sm_100a kernels for the Topological Synapse compress
// path: attention mass, centroid coverage (A2), the greedy
// hybrid selection (A4/A6), landmark gather (A5) and the metric reductions (A7).
//
// Exactness contract: every value the reference's DECISIONS
// depend on is computed with the reference's fp64 operations in the
// reference's order, using __d*_rn intrinsics so nvcc never contracts them
// into FMAs (the reference is built without -march => no FMA).  The fp32
// distance filter in the selection loop is conservative: it only skips a
// (row, pick) pair when a proven lower bound says the fp64 distance cannot
// lower that row's running minimum, so its output is bit-identical.
#include <cooperative_groups.h>
#include <float.h>

#include "cx_internal.cuh"

namespace cg = cooperative_groups;

namespace cx {

namespace {

constexpr int kMaxCluster = 16;

__device__ __forceinline__ double dmin_std(double a, double b) { return (b < a) ? b : a; }  // std::min
__device__ __forceinline__ double dmax_std(double a, double b) { return (a < b) ? b : a; }  // std::max

// ----------------------------------------------------------------------------
// A3: attention mass.  K1: scores[g][p][i] = (sum_c q_c * k_ic) * (1/sqrt(d_k))
// with the reference's sequential fp64 dot (synapse.cpp:76-86).
// ----------------------------------------------------------------------------
__global__ void attn_scores_kernel(GroupView gv, double inv_sqrt_dk, double* __restrict__ scores,
                                   int* flag) {
    const int g = blockIdx.y;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= gv.L) return;
    const float* row = gv.X + g * gv.gstride + i * gv.rstride;
    for (int p = 0; p < gv.P; ++p) {
        const float* q = gv.Q + ((int64_t)g * gv.P + p) * gv.d_k;
        const float* kp = row + (int64_t)p * gv.col_step;
        double dot = 0.0;
#pragma unroll 8
        for (int c = 0; c < gv.d_k; ++c)
            dot = __dadd_rn(dot, __dmul_rn((double)__ldg(q + c), (double)__ldg(kp + c)));
        const double s = __dmul_rn(dot, inv_sqrt_dk);
        if (!isfinite(s)) atomicOr(flag, FLAG_NONFINITE);
        scores[((int64_t)g * gv.P + p) * gv.L + i] = s;
    }
}

// dim-64 fast path for the same scores (GQA groups, or a single pass): the row
// is loaded once into registers (16 x float4) and all passes are accumulated
// in one sweep over the coordinates -- P independent fp64 chains per thread,
// each still summed in the reference's coordinate order.
constexpr int kAttnMaxP = 8;
__global__ void __launch_bounds__(256) attn64_scores_kernel(GroupView gv, double inv_sqrt_dk,
                                                          double* __restrict__ scores, int* flag) {
    __shared__ double qs[kAttnMaxP][64];
    const int g = blockIdx.y;
    for (int e = threadIdx.x; e < gv.P * 64; e += blockDim.x)
        qs[e / 64][e % 64] = (double)__ldg(gv.Q + (int64_t)g * gv.P * 64 + e);
    __syncthreads();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= gv.L) return;
    const float4* row = reinterpret_cast<const float4*>(gv.X + g * gv.gstride + i * gv.rstride);
    float x[64];
#pragma unroll
    for (int c4 = 0; c4 < 16; ++c4) {
        const float4 v = __ldg(row + c4);
        x[4 * c4] = v.x; x[4 * c4 + 1] = v.y; x[4 * c4 + 2] = v.z; x[4 * c4 + 3] = v.w;
    }
    double acc[kAttnMaxP];
#pragma unroll
    for (int p = 0; p < kAttnMaxP; ++p) acc[p] = 0.0;
#pragma unroll
    for (int c = 0; c < 64; ++c) {
        const double xc = (double)x[c];
        // fused multiply-add: half the fp64 instructions of the reference's dmul + dadd, and one
        // rounding per term instead of two (the attention mass contract is 1e-12 relative,
        // DESIGN.md §3.1; the selection's decisions are certified by the gap monitor)
#pragma unroll
        for (int p = 0; p < kAttnMaxP; ++p)
            if (p < gv.P) acc[p] = __fma_rn(qs[p][c], xc, acc[p]);
    }
#pragma unroll
    for (int p = 0; p < kAttnMaxP; ++p) {
        if (p < gv.P) {
            const double s = __dmul_rn(acc[p], inv_sqrt_dk);
            if (!isfinite(s)) atomicOr(flag, FLAG_NONFINITE);
            scores[((int64_t)g * gv.P + p) * gv.L + i] = s;
        }
    }
}

template <class T, class Op>
__device__ __forceinline__ T warp_reduce(T v, Op op) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide reduction with a fixed combination tree (deterministic run to run).
template <class T, class Op>
__device__ T block_reduce(T v, Op op, T identity, T* smem /* >= 32 */) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_reduce(v, op);
    __syncthreads();
    if (lane == 0) smem[wid] = v;
    __syncthreads();
    T r = (threadIdx.x < nw) ? smem[threadIdx.x] : identity;
    if (wid == 0) r = warp_reduce(r, op);
    if (threadIdx.x == 0) smem[0] = r;
    __syncthreads();
    r = smem[0];
    __syncthreads();
    return r;
}

// K2: per (group, pass): max, e_i = exp(s_i - max) in place, sum (kernels.cpp:66-81).
__global__ void attn_softmax_kernel(int64_t L, int P, double* __restrict__ scores,
                                    double* __restrict__ sums) {
    __shared__ double red[32];
    const int gp = blockIdx.x;
    double* s = scores + (int64_t)gp * L;
    double m = -INFINITY;
    for (int64_t i = threadIdx.x; i < L; i += blockDim.x) m = dmax_std(m, s[i]);
    m = block_reduce(m, [](double a, double b) { return dmax_std(a, b); }, -(double)INFINITY, red);
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < L; i += blockDim.x) {
        const double e = exp(__dsub_rn(s[i], m));
        s[i] = e;
        acc = __dadd_rn(acc, e);
    }
    acc = block_reduce(acc, [](double a, double b) { return __dadd_rn(a, b); }, 0.0, red);
    if (threadIdx.x == 0) sums[gp] = acc;
}

// K3: total_i = ((0 + e_0i/sum_0) + e_1i/sum_1) + ...  (pass order, synapse.cpp:87-90)
__global__ void attn_total_kernel(int64_t L, int P, const double* __restrict__ e,
                                  const double* __restrict__ sums, double* __restrict__ out) {
    const int g = blockIdx.y;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= L) return;
    double t = 0.0;
    for (int p = 0; p < P; ++p)
        t = __dadd_rn(t, __ddiv_rn(e[((int64_t)g * P + p) * L + i], sums[(int64_t)g * P + p]));
    out[(int64_t)g * L + i] = t;
}

// ----------------------------------------------------------------------------
// A2: centroid_of (synapse.cpp:36-44) -- summed sequentially over rows, as
// the reference does; one thread per coordinate.
// ----------------------------------------------------------------------------
__global__ void centroid_kernel(GroupView gv, double* __restrict__ cen) {
    const int g = blockIdx.x;
    const int j = threadIdx.x;
    if (j >= gv.dim) return;
    const float* base = gv.X + g * gv.gstride + j;
    double c = 0.0;
    int64_t i = 0;
    for (; i + 8 <= gv.L; i += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(base + (i + u) * gv.rstride);
#pragma unroll
        for (int u = 0; u < 8; ++u) c = __dadd_rn(c, (double)v[u]);
    }
    for (; i < gv.L; ++i) c = __dadd_rn(c, (double)__ldg(base + i * gv.rstride));
    cen[(int64_t)g * gv.dim + j] = __ddiv_rn(c, (double)gv.L);
}

// Same sum with the loads off the critical path: one warp per 32 coordinates
// of one group; rows stream through an 8-stage cp.async ring (32 rows x 128 B
// per stage) so the only serial cost is the fp64 add chain (L x 8.4 cycles).
constexpr int kCpStages = 12;  // 12 x 32 rows x 128 B = 48 KB static: ~2 us of loads in flight per warp
constexpr int kCpRows = 32;
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}
__global__ void __launch_bounds__(32) centroid_pipe_kernel(GroupView gv, double* __restrict__ cen) {
    __shared__ __align__(16) float ring[kCpStages][kCpRows][32];
    const int g = blockIdx.y;
    const int c0 = blockIdx.x * 32;
    const int lane = threadIdx.x;
    const float* base = gv.X + g * gv.gstride + c0;
    const int64_t nst = (gv.L + kCpRows - 1) / kCpRows;
    auto issue = [&](int64_t st) {
        if (st < nst) {
            const int64_t r0 = st * kCpRows;
            const int rows = (int)min((int64_t)kCpRows, gv.L - r0);
            float(*buf)[32] = ring[st % kCpStages];
            for (int e = lane; e < rows * 8; e += 32) {  // 8 x 16 B per row
                const int r = e >> 3, q = e & 7;
                cp_async16(&buf[r][q * 4], base + (r0 + r) * gv.rstride + q * 4);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int st = 0; st < kCpStages - 1; ++st) issue(st);
    double acc = 0.0;
    for (int64_t st = 0; st < nst; ++st) {
        issue(st + kCpStages - 1);
        asm volatile("cp.async.wait_group %0;" ::"n"(kCpStages - 1) : "memory");
        __syncwarp();
        const float(*buf)[32] = ring[st % kCpStages];
        const int rows = (int)min((int64_t)kCpRows, gv.L - st * kCpRows);
        if (c0 + lane < gv.dim) {
#pragma unroll 8
            for (int r = 0; r < rows; ++r) acc = __dadd_rn(acc, (double)buf[r][lane]);
        }
        __syncwarp();
    }
    if (c0 + lane < gv.dim) cen[(int64_t)g * gv.dim + c0 + lane] = __ddiv_rn(acc, (double)gv.L);
}

// The same sum with the rows streamed by TMA bulk copies: one CTA per group, one thread
// per coordinate; a ring of stages of kTmaRows contiguous rows (rstride == dim), ONE
// cp.async.bulk per stage completing on the stage's mbarrier (per-row copies measured
// 2.5x slower than the cp.async ring: small TMA requests are expensive).  ~128 KB of rows in flight per SM keeps the loads
// ahead of the only serial cost, the fp64 add chain (L x ~8.4 cycles).
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int kTmaRows>
__global__ void __launch_bounds__(256) centroid_tma_kernel(GroupView gv, double* __restrict__ cen, int n_stages) {
    extern __shared__ __align__(128) unsigned char csm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(csm);  // [n_stages]
    float* ring = reinterpret_cast<float*>(csm + 128 * ((n_stages * 8 + 127) / 128));  // [n_stages][32][dim]
    const int g = blockIdx.x, j = threadIdx.x, dim = gv.dim;
    const float* base = gv.X + g * gv.gstride;
    const int64_t nst = (gv.L + kTmaRows - 1) / kTmaRows;
    const uint32_t row_bytes = (uint32_t)dim * 4u;
    if (j == 0) {
        for (int i = 0; i < n_stages; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + i)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int64_t st, int slot) {  // thread 0: the stage's rows are contiguous (rstride == dim)
        const int64_t r0 = st * kTmaRows;
        const uint32_t bytes = row_bytes * (uint32_t)min((int64_t)kTmaRows, gv.L - r0);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + slot)), "r"(bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(ring + (size_t)slot * kTmaRows * dim)),
            "l"(base + r0 * dim), "r"(bytes), "r"(smem_u32(full + slot))
            : "memory");
    };
    if (j == 0)
        for (int64_t st = 0; st < min((int64_t)n_stages, nst); ++st) issue(st, (int)st);
    double acc = 0.0;
    // slot and phase parity advance incrementally (a 64-bit % and / per stage cost more than
    // the stage's 32 adds)
    int slot = 0;
    uint32_t par = 0;
    for (int64_t st = 0; st < nst; ++st) {
        uint32_t ok = 0;
        do {
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(ok)
                         : "r"(smem_u32(full + slot)), "r"(par)
                         : "memory");
        } while (!ok);
        const float* buf = ring + (size_t)slot * kTmaRows * dim;
        const int rows = (int)min((int64_t)kTmaRows, gv.L - st * kTmaRows);
        if (rows == kTmaRows) {
#pragma unroll
            for (int r = 0; r < kTmaRows; ++r) acc = __dadd_rn(acc, (double)buf[r * dim + j]);
        } else {
            for (int r = 0; r < rows; ++r) acc = __dadd_rn(acc, (double)buf[r * dim + j]);
        }
        __syncthreads();  // every thread is done with the slot
        if (j == 0 && st + n_stages < nst) issue(st + n_stages, slot);
        if (++slot == n_stages) {
            slot = 0;
            par ^= 1u;
        }
    }
    cen[(int64_t)g * dim + j] = __ddiv_rn(acc, (double)gv.L);
}

constexpr int kCenRows = 64;
__global__ void __launch_bounds__(256) centroid_staged_kernel(GroupView gv, double* __restrict__ cen) {
    extern __shared__ __align__(16) float cbuf[];  // [2][kCenRows][dim]
    const int g = blockIdx.x;
    const int dim = gv.dim;
    const float* base = gv.X + g * gv.gstride;
    const int64_t nchunks = (gv.L + kCenRows - 1) / kCenRows;
    auto load = [&](int64_t ch, float* dst) {
        const int64_t r0 = ch * kCenRows;
        const int rows = (int)min((int64_t)kCenRows, gv.L - r0);
        for (int e = threadIdx.x; e < rows * dim; e += blockDim.x) {
            const int r = e / dim, c = e % dim;
            dst[r * dim + c] = __ldg(base + (r0 + r) * gv.rstride + c);
        }
    };
    double acc = 0.0;
    load(0, cbuf);
    __syncthreads();
    for (int64_t ch = 0; ch < nchunks; ++ch) {
        float* cur = cbuf + (ch & 1) * kCenRows * dim;
        if (ch + 1 < nchunks) load(ch + 1, cbuf + ((ch + 1) & 1) * kCenRows * dim);
        if (threadIdx.x < dim) {
            const int rows = (int)min((int64_t)kCenRows, gv.L - ch * kCenRows);
            for (int r = 0; r < rows; ++r) acc = __dadd_rn(acc, (double)cur[r * dim + threadIdx.x]);
        }
        __syncthreads();
    }
    if (threadIdx.x < dim) cen[(int64_t)g * dim + threadIdx.x] = __ddiv_rn(acc, (double)gv.L);
}

// sq_dist(span<float>, vector<double>) / sq_dist(span<float>, span<float>)
// (synapse.cpp:18-34): sequential over coordinates, no FMA.
__device__ __forceinline__ double sq_dist_exact(const float* x, int64_t xs, const double* b, int dim) {
    double acc = 0.0;
    for (int c = 0; c < dim; ++c) {
        const double d = __dsub_rn((double)x[c * xs], b[c]);
        acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
    return acc;
}

__device__ __forceinline__ double sq_dist_exact_ff(const float* a, const float* b, int dim) {
    double acc = 0.0;
    for (int c = 0; c < dim; ++c) {
        const double d = __dsub_rn((double)a[c], (double)b[c]);
        acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
    return acc;
}

// coverage with empty selection: sqrt(sq_dist(x_i, centroid))  (synapse.cpp:107-112)
__global__ void coverage_centroid_kernel(GroupView gv, const double* __restrict__ cen,
                                         double* __restrict__ out) {
    extern __shared__ double cs[];
    const int g = blockIdx.y;
    for (int c = threadIdx.x; c < gv.dim; c += blockDim.x) cs[c] = cen[(int64_t)g * gv.dim + c];
    __syncthreads();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= gv.L) return;
    out[(int64_t)g * gv.L + i] =
        __dsqrt_rn(sq_dist_exact(gv.X + g * gv.gstride + i * gv.rstride, 1, cs, gv.dim));
}

// coverage with a selection: sqrt(min_s sq_dist(x_i, x_s))  (synapse.cpp:114-119)
__global__ void coverage_selected_kernel(GroupView gv, const int64_t* __restrict__ sel, int64_t n_sel,
                                         double* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= gv.L) return;
    const float* xi = gv.X + i * gv.rstride;
    double best = INFINITY;
    for (int64_t s = 0; s < n_sel; ++s) best = dmin_std(best, sq_dist_exact_ff(xi, gv.X + sel[s] * gv.rstride, gv.dim));
    out[i] = __dsqrt_rn(best);
}

// ----------------------------------------------------------------------------
// A4/A6: greedy hybrid selection (synapse.cpp:216-284).
//
// One thread-block cluster per group; CTA r owns rows [r*S, r*S+S).  Rows are
// staged once into shared memory, column-major (conflict-free), when they fit;
// otherwise read in place from global memory (L2-resident).  Per round:
//   1. local min/max of attention and running-min distance over REMAINING rows
//      (fused into the previous round's update), exchanged across the cluster
//      through DSMEM + one cluster barrier;
//   2. local argmax of the hybrid score (strict >, lowest row on ties),
//      exchanged with the candidate's coordinates + one cluster barrier;
//   3. distance update of every remaining row against the pick: fp32 lower
//      bound first, exact fp64 (reference order) only where the bound cannot
//      rule out a new minimum.  Removed rows are never read again by the
//      reference, so they are skipped.
// ----------------------------------------------------------------------------
struct SelectParams {
    GroupView gv;
    const double* attn;  // [G][L]
    const double* cen;   // [G][dim]
    int take;
    double lambda;
    int S;               // rows per CTA
    int smem_rows;       // rows staged in shared memory
    int filter;          // fp32 lower-bound filter on/off
    int64_t* pick_rows;  // [G][take] unsorted (selection order)
    double* pick_scores;
    int64_t* out_rows;   // [G][take] ascending
    double* out_scores;
};

struct alignas(16) BestSlot {
    double score;
    long long row;
};

struct SelectSmem {
    // offsets (bytes) into dynamic shared memory
    size_t mind, attn, thr, rem, xs, bvec, bf, mm, best, coords, red_d, red_b, total;
};

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline SelectSmem select_smem_layout(int S, int dim, int smem_rows) {
    SelectSmem L;
    size_t o = 0;
    L.mind = o;   o = align_up(o + sizeof(double) * S, 16);
    L.attn = o;   o = align_up(o + sizeof(double) * S, 16);
    L.thr = o;    o = align_up(o + sizeof(float) * S, 16);
    L.rem = o;    o = align_up(o + S, 16);
    L.xs = o;     o = align_up(o + (smem_rows ? sizeof(float) * (size_t)S * dim : 0), 16);
    L.bvec = o;   o = align_up(o + sizeof(double) * dim, 16);
    L.bf = o;     o = align_up(o + sizeof(float) * dim, 16);
    L.mm = o;     o = align_up(o + sizeof(double) * 4 * kMaxCluster, 16);
    L.best = o;   o = align_up(o + sizeof(BestSlot) * kMaxCluster, 16);
    L.coords = o; o = align_up(o + sizeof(float) * kMaxCluster * dim, 16);
    L.red_d = o;  o = align_up(o + sizeof(double) * 4 * 32, 16);
    L.red_b = o;  o = align_up(o + sizeof(BestSlot) * 32, 16);
    L.total = o;
    return L;
}

__device__ __forceinline__ bool better(double s, long long r, double bs, long long br) {
    return s > bs || (s == bs && r < br);
}

__global__ void __launch_bounds__(512, 1) select_kernel(SelectParams p) {
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned C = cluster.num_blocks();
    const unsigned rank = cluster.block_rank();
    const int g = blockIdx.y;
    const GroupView& gv = p.gv;
    const int dim = gv.dim;
    const int64_t L = gv.L;
    const int S = p.S;
    const int64_t r0 = (int64_t)rank * S;
    const int nrows = (int)max((int64_t)0, min((int64_t)S, L - r0));
    const int tid = threadIdx.x, nt = blockDim.x;

    extern __shared__ __align__(16) unsigned char smem[];
    const SelectSmem lay = select_smem_layout(S, dim, p.smem_rows);
    double* mind = reinterpret_cast<double*>(smem + lay.mind);
    double* attn = reinterpret_cast<double*>(smem + lay.attn);
    float* thr = reinterpret_cast<float*>(smem + lay.thr);
    unsigned char* rem = smem + lay.rem;
    float* xs = reinterpret_cast<float*>(smem + lay.xs);
    double* bvec = reinterpret_cast<double*>(smem + lay.bvec);
    float* bf = reinterpret_cast<float*>(smem + lay.bf);
    double* mm = reinterpret_cast<double*>(smem + lay.mm);          // [C][4]
    BestSlot* bests = reinterpret_cast<BestSlot*>(smem + lay.best);  // [C]
    float* coords = reinterpret_cast<float*>(smem + lay.coords);     // [C][dim]
    double* red_d = reinterpret_cast<double*>(smem + lay.red_d);     // [4][32]
    BestSlot* red_b = reinterpret_cast<BestSlot*>(smem + lay.red_b);

    const float* gX = gv.X + g * gv.gstride + r0 * gv.rstride;
    // element (li, c): smem column-major or global row-major
    const float* xbase = p.smem_rows ? xs : gX;
    const int64_t xcs = p.smem_rows ? (int64_t)S : 1;          // stride between coordinates
    const int64_t xrs = p.smem_rows ? (int64_t)1 : gv.rstride;  // stride between rows

    // ---- stage rows + attention; coverage init = distance to the centroid ----
    if (p.smem_rows) {
        for (int64_t e = tid; e < (int64_t)nrows * dim; e += nt) {
            const int li = (int)(e / dim), c = (int)(e % dim);
            xs[(int64_t)c * S + li] = __ldg(gX + li * gv.rstride + c);
        }
    }
    for (int c = tid; c < dim; c += nt) bvec[c] = p.cen[(int64_t)g * dim + c];
    for (int li = tid; li < nrows; li += nt) {
        attn[li] = p.attn[(int64_t)g * L + r0 + li];
        rem[li] = 1;
    }
    __syncthreads();

    // local min/max over remaining rows (all rows at round 0)
    double amin = INFINITY, amax = -INFINITY, cmin = INFINITY, cmax = -INFINITY;
    for (int li = tid; li < nrows; li += nt) {
        const double d = __dsqrt_rn(sq_dist_exact(xbase + li * xrs, xcs, bvec, dim));
        mind[li] = d;
        thr[li] = INFINITY;
        amin = dmin_std(amin, attn[li]);
        amax = dmax_std(amax, attn[li]);
        cmin = dmin_std(cmin, d);
        cmax = dmax_std(cmax, d);
    }

    const double lam = p.lambda;
    const double one_m_lam = __dsub_rn(1.0, lam);
    int64_t* pick_rows = p.pick_rows + (int64_t)g * p.take;
    double* pick_scores = p.pick_scores + (int64_t)g * p.take;

    for (int round = 0; round < p.take; ++round) {
        // ---- 1. cluster-wide min/max over remaining rows ----
        {
            const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
            amin = warp_reduce(amin, [](double a, double b) { return dmin_std(a, b); });
            amax = warp_reduce(amax, [](double a, double b) { return dmax_std(a, b); });
            cmin = warp_reduce(cmin, [](double a, double b) { return dmin_std(a, b); });
            cmax = warp_reduce(cmax, [](double a, double b) { return dmax_std(a, b); });
            if (lane == 0) {
                red_d[0 * 32 + wid] = amin;
                red_d[1 * 32 + wid] = amax;
                red_d[2 * 32 + wid] = cmin;
                red_d[3 * 32 + wid] = cmax;
            }
            __syncthreads();
            if (wid == 0) {
                double v0 = lane < nw ? red_d[0 * 32 + lane] : INFINITY;
                double v1 = lane < nw ? red_d[1 * 32 + lane] : -INFINITY;
                double v2 = lane < nw ? red_d[2 * 32 + lane] : INFINITY;
                double v3 = lane < nw ? red_d[3 * 32 + lane] : -INFINITY;
                v0 = warp_reduce(v0, [](double a, double b) { return dmin_std(a, b); });
                v1 = warp_reduce(v1, [](double a, double b) { return dmax_std(a, b); });
                v2 = warp_reduce(v2, [](double a, double b) { return dmin_std(a, b); });
                v3 = warp_reduce(v3, [](double a, double b) { return dmax_std(a, b); });
                if (lane < (int)C) {  // push my CTA's partials to CTA `lane`
                    double* dst = cluster.map_shared_rank(mm, lane) + rank * 4;
                    dst[0] = v0; dst[1] = v1; dst[2] = v2; dst[3] = v3;
                }
            }
        }
        cluster.sync();
        amin = INFINITY; amax = -INFINITY; cmin = INFINITY; cmax = -INFINITY;
        for (unsigned r = 0; r < C; ++r) {
            amin = dmin_std(amin, mm[r * 4 + 0]);
            amax = dmax_std(amax, mm[r * 4 + 1]);
            cmin = dmin_std(cmin, mm[r * 4 + 2]);
            cmax = dmax_std(cmax, mm[r * 4 + 3]);
        }

        // ---- 2. hybrid argmax (synapse.cpp:247-260) ----
        const bool a_span = amax > amin, c_span = cmax > cmin;
        const double ar = __dsub_rn(amax, amin), cr = __dsub_rn(cmax, cmin);
        double bs = -1.0;
        long long br = LLONG_MAX;
        for (int li = tid; li < nrows; li += nt) {
            if (!rem[li]) continue;
            const double na = a_span ? __ddiv_rn(__dsub_rn(attn[li], amin), ar) : 0.0;
            const double nc = c_span ? __ddiv_rn(__dsub_rn(mind[li], cmin), cr) : 0.0;
            const double h = __dadd_rn(__dmul_rn(lam, nc), __dmul_rn(one_m_lam, na));
            if (h > bs) { bs = h; br = r0 + li; }  // rows visited ascending per thread
        }
        {
            const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double os = __shfl_xor_sync(0xffffffffu, bs, o);
                const long long orr = __shfl_xor_sync(0xffffffffu, br, o);
                if (better(os, orr, bs, br)) { bs = os; br = orr; }
            }
            if (lane == 0) { red_b[wid].score = bs; red_b[wid].row = br; }
            __syncthreads();
            if (tid == 0) {
                for (int w = 1; w < nw; ++w)
                    if (better(red_b[w].score, red_b[w].row, bs, br)) { bs = red_b[w].score; br = red_b[w].row; }
                red_b[0].score = bs;
                red_b[0].row = br;
            }
            __syncthreads();
            bs = red_b[0].score;
            br = red_b[0].row;
            // push (score,row) and the candidate's coordinates to every CTA
            if (tid < (int)C) {
                BestSlot* dst = cluster.map_shared_rank(bests, tid) + rank;
                dst->score = bs;
                dst->row = br;
            }
            if (br != LLONG_MAX) {
                const int lb = (int)(br - r0);
                for (int e = tid; e < (int)C * dim; e += nt) {
                    const int r = e / dim, c = e % dim;
                    float* dst = cluster.map_shared_rank(coords, r) + rank * dim;
                    dst[c] = xbase[lb * xrs + c * xcs];
                }
            }
        }
        cluster.sync();
        unsigned w = 0;
        bs = bests[0].score;
        br = bests[0].row;
        for (unsigned r = 1; r < C; ++r)
            if (better(bests[r].score, bests[r].row, bs, br)) { bs = bests[r].score; br = bests[r].row; w = r; }
        for (int c = tid; c < dim; c += nt) {
            const float v = coords[w * dim + c];
            bf[c] = v;
            bvec[c] = (double)v;
        }
        if (rank == 0 && tid == 0) {
            pick_rows[round] = br;
            pick_scores[round] = bs;
        }
        if (br >= r0 && br < r0 + nrows && tid == 0) rem[br - r0] = 0;
        __syncthreads();

        // ---- 3. distance update against the pick (synapse.cpp:265-273) ----
        amin = INFINITY; amax = -INFINITY; cmin = INFINITY; cmax = -INFINITY;
        if (round + 1 < p.take) {
            for (int li = tid; li < nrows; li += nt) {
                if (!rem[li]) continue;
                const float* x = xbase + li * xrs;
                bool need_exact = true;
                if (p.filter && round > 0) {
                    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
                    int c = 0;
                    for (; c + 4 <= dim; c += 4) {
                        const float t0 = __fsub_rn(x[(c + 0) * xcs], bf[c + 0]);
                        const float t1 = __fsub_rn(x[(c + 1) * xcs], bf[c + 1]);
                        const float t2 = __fsub_rn(x[(c + 2) * xcs], bf[c + 2]);
                        const float t3 = __fsub_rn(x[(c + 3) * xcs], bf[c + 3]);
                        s0 = __fmaf_rn(t0, t0, s0);
                        s1 = __fmaf_rn(t1, t1, s1);
                        s2 = __fmaf_rn(t2, t2, s2);
                        s3 = __fmaf_rn(t3, t3, s3);
                    }
                    for (; c < dim; ++c) {
                        const float t = __fsub_rn(x[c * xcs], bf[c]);
                        s0 = __fmaf_rn(t, t, s0);
                    }
                    const float s = __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3));
                    // |s - S| <= (dim + 5) u S for S = exact sum (u = 2^-24), plus an
                    // absolute underflow allowance; fp64 sum >= S (1 - (dim+2) 2^-53).
                    const float lb = __fsub_rd(__fmul_rd(s, 1.0f - 0x1p-15f), 0x1p-100f);
                    need_exact = !(lb > thr[li]);
                }
                double d2, d;
                if (need_exact) {
                    d2 = sq_dist_exact(x, xcs, bvec, dim);
                    d = __dsqrt_rn(d2);
                    if (round == 0) {
                        mind[li] = d;
                        thr[li] = __double2float_ru(d2);
                    } else if (d < mind[li]) {  // std::min(mindist, d)
                        mind[li] = d;
                        thr[li] = __double2float_ru(d2);
                    }
                }
                amin = dmin_std(amin, attn[li]);
                amax = dmax_std(amax, attn[li]);
                cmin = dmin_std(cmin, mind[li]);
                cmax = dmax_std(cmax, mind[li]);
            }
        }
    }

    // ---- sort picks ascending by row (synapse.cpp:276-277) ----
    cluster.sync();
    if (rank == 0) {
        __syncthreads();
        int64_t* out_rows = p.out_rows + (int64_t)g * p.take;
        double* out_scores = p.out_scores + (int64_t)g * p.take;
        for (int s = tid; s < p.take; s += nt) {
            const int64_t r = pick_rows[s];
            int pos = 0;
            for (int t = 0; t < p.take; ++t) pos += pick_rows[t] < r;
            out_rows[pos] = r;
            out_scores[pos] = pick_scores[s];
        }
    }
}

// ----------------------------------------------------------------------------
// A5: landmark gather dst[g][s][:] = src[g][rows[g][s]][:]
// ----------------------------------------------------------------------------
// landmark gather (synapse.cpp:303-318 copy): dst[g][s] = src row rows[g][s] of group g, for
// up to two sources (keys and values) in one launch (blockIdx.z); dst group blocks dst_gstride
// floats apart (take * dim when dense; the decode layout [layer][kv head][k][d] otherwise)
__global__ void gather_rows_kernel(GroupView gv, const float* __restrict__ src0, const float* __restrict__ src1,
                                   const int64_t* __restrict__ rows, int take, float* __restrict__ dst0,
                                   float* __restrict__ dst1, int64_t dst_gstride, int rpb) {
    const int g = blockIdx.y;
    const float* src = blockIdx.z ? src1 : src0;
    float* dst = blockIdx.z ? dst1 : dst0;
    // rpb rows per block, tpr = blockDim.x / rpb threads per row (one 16-B chunk each when
    // dim % 4 == 0): every row of a group's selection is in flight at once (one thread-block
    // per row left 3/4 of each block idle and took ~3 waves of blocks: 11 us for cfg2)
    const int tpr = (int)blockDim.x / rpb;
    const int s = (int)blockIdx.x * rpb + (int)threadIdx.x / tpr, t = (int)threadIdx.x % tpr;
    if (s >= take) return;
    const int64_t r = rows[(int64_t)g * take + s];
    const float* in = src + g * gv.gstride + r * gv.rstride;
    float* out = dst + (int64_t)g * dst_gstride + (int64_t)s * gv.dim;
    if ((gv.dim & 3) == 0 && ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0) {
        for (int c = t; c < gv.dim / 4; c += tpr)
            reinterpret_cast<float4*>(out)[c] = __ldg(reinterpret_cast<const float4*>(in) + c);
    } else {
        for (int c = t; c < gv.dim; c += tpr) out[c] = __ldg(in + c);
    }
}

// ----------------------------------------------------------------------------
// A7 metrics.  hausdorff: per-row min over landmarks of sq_dist, max over rows
// (order-free, hence bit-exact); rows==nullptr means landmarks are a separate
// set `lm`.  mean_pairwise: sum over i<j of sqrt(sq_dist) (fp64; reduction
// order differs from the reference's serial loop -> 1e-12 relative).
// ----------------------------------------------------------------------------
__global__ void hausdorff_kernel(const float* __restrict__ cloud, int64_t count, int dim,
                                 const float* __restrict__ lm, int64_t m, const int64_t* __restrict__ rows,
                                 unsigned long long* __restrict__ worst_bits) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double best = INFINITY;
    if (i < count) {
        const float* xi = cloud + i * dim;
        for (int64_t j = 0; j < m; ++j) {
            const float* y = rows ? cloud + rows[j] * dim : lm + j * dim;
            best = dmin_std(best, sq_dist_exact_ff(xi, y, dim));
        }
    } else {
        best = 0.0;
    }
    // non-negative doubles order like their bit patterns
    best = warp_reduce(best, [](double a, double b) { return dmax_std(a, b); });
    if ((threadIdx.x & 31) == 0) atomicMax(worst_bits, (unsigned long long)__double_as_longlong(best));
}

// Tiled form (dim <= 128): a CTA stages its 128 cloud rows and then 32-landmark tiles as
// fp64 in shared memory (converted once), so a pair costs shared-memory reads and the
// sequential fp64 sum only; min / max are order-free, so the result stays bitwise.
constexpr int HD_ROWS = 128, HD_T = 32, HD_MAXDIM = 128;
__global__ void __launch_bounds__(HD_ROWS) hausdorff_tile_kernel(const float* __restrict__ cloud, int64_t count, int dim,
                                                                 const float* __restrict__ lm, int64_t m,
                                                                 const int64_t* __restrict__ rows,
                                                                 unsigned long long* __restrict__ worst_bits) {
    extern __shared__ double hd_sm[];
    const int pitch = dim + 1;
    double* sx = hd_sm;                      // [HD_ROWS][pitch]
    double* sl = hd_sm + HD_ROWS * pitch;    // [HD_T][pitch]
    const int64_t r0 = (int64_t)blockIdx.x * HD_ROWS;
    for (int e = threadIdx.x; e < HD_ROWS * dim; e += HD_ROWS) {
        const int r = e / dim, c = e % dim;
        sx[r * pitch + c] = r0 + r < count ? (double)cloud[(r0 + r) * dim + c] : 0.0;
    }
    const double* x = sx + threadIdx.x * pitch;
    double best = INFINITY;
    for (int64_t j0 = 0; j0 < m; j0 += HD_T) {
        __syncthreads();  // previous tile consumed (and the cloud rows staged)
        for (int e = threadIdx.x; e < HD_T * dim; e += HD_ROWS) {
            const int r = e / dim, c = e % dim;
            const int64_t j = j0 + r;
            sl[r * pitch + c] = j < m ? (double)(rows ? cloud[rows[j] * dim + c] : lm[j * dim + c]) : 0.0;
        }
        __syncthreads();
        const int nt = (int)min((int64_t)HD_T, m - j0);
        for (int jj = 0; jj < nt; ++jj) {
            const double* y = sl + jj * pitch;  // broadcast
            double acc = 0.0;
            for (int c = 0; c < dim; ++c) {
                const double d = __dsub_rn(x[c], y[c]);
                acc = __dadd_rn(acc, __dmul_rn(d, d));
            }
            best = dmin_std(best, acc);
        }
    }
    if (r0 + threadIdx.x >= count) best = 0.0;
    best = warp_reduce(best, [](double a, double b) { return dmax_std(a, b); });
    if ((threadIdx.x & 31) == 0) atomicMax(worst_bits, (unsigned long long)__double_as_longlong(best));
}

__global__ void mean_pairwise_kernel(const float* __restrict__ pts, int64_t count, int dim,
                                     const int64_t* __restrict__ rows, double* __restrict__ partial) {
    __shared__ double red[32];
    const int64_t i = blockIdx.x;
    double acc = 0.0;
    const float* xi = pts + (rows ? rows[i] : i) * dim;
    for (int64_t j = i + 1 + threadIdx.x; j < count; j += blockDim.x)
        acc = __dadd_rn(acc, __dsqrt_rn(sq_dist_exact_ff(xi, pts + (rows ? rows[j] : j) * dim, dim)));
    acc = block_reduce(acc, [](double a, double b) { return __dadd_rn(a, b); }, 0.0, red);
    if (threadIdx.x == 0) partial[i] = acc;
}

// Tiled form: the points are converted to fp64 once (rows gathered), then each CTA takes a
// 32 x 32 tile of the upper triangle (bi <= bj) with both tiles' rows staged in shared
// memory; every pair's squared distance is still the sequential fp64 sum of the reference
// (coordinates in order), only the sum over pairs is reordered (1e-12 relative).
constexpr int MP_T = 32;
constexpr int MP_MAXDIM = 256;
__global__ void to_f64_kernel(const float* __restrict__ pts, int64_t n, int dim, const int64_t* __restrict__ rows,
                              double* __restrict__ out) {
    const int64_t tot = n * dim;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / dim, c = e % dim;
        out[e] = (double)pts[(rows ? rows[i] : i) * dim + c];
    }
}
__global__ void __launch_bounds__(256) mean_pairwise_tile_kernel(const double* __restrict__ p64, int64_t n, int dim,
                                                                 double* __restrict__ partial) {
    extern __shared__ double mp_sm[];  // [2][MP_T][dim + 1]
    __shared__ double red[32];
    const int bi = blockIdx.y, bj = blockIdx.x;
    const int64_t slot = (int64_t)bi * gridDim.x + bj;
    if (bj < bi) {  // lower triangle: nothing (uniform per CTA)
        if (threadIdx.x == 0) partial[slot] = 0.0;
        return;
    }
    const int pitch = dim + 1;
    double* si = mp_sm;
    double* sj = mp_sm + MP_T * pitch;
    const int64_t i0 = (int64_t)bi * MP_T, j0 = (int64_t)bj * MP_T;
    for (int e = threadIdx.x; e < MP_T * dim; e += blockDim.x) {
        const int r = e / dim, c = e % dim;
        si[r * pitch + c] = i0 + r < n ? p64[(i0 + r) * dim + c] : 0.0;
        sj[r * pitch + c] = j0 + r < n ? p64[(j0 + r) * dim + c] : 0.0;
    }
    __syncthreads();
    const int ti = threadIdx.x & 31, tw = threadIdx.x >> 5;  // lane -> i row, warp -> j rows tw + 8u
    double acc = 0.0;
    for (int u = 0; u < MP_T / 8; ++u) {
        const int tj = tw + 8 * u;
        if (i0 + ti < n && j0 + tj < n && (bi < bj || tj > ti)) {
            const double* a = si + ti * pitch;
            const double* b = sj + tj * pitch;  // warp-uniform row: broadcast reads
            double d2 = 0.0;
            for (int c = 0; c < dim; ++c) {
                const double d = __dsub_rn(a[c], b[c]);
                d2 = __dadd_rn(d2, __dmul_rn(d, d));
            }
            acc = __dadd_rn(acc, __dsqrt_rn(d2));
        }
    }
    acc = block_reduce(acc, [](double x, double y) { return __dadd_rn(x, y); }, 0.0, red);
    if (threadIdx.x == 0) partial[slot] = acc;
}

__global__ void sum_partials_kernel(const double* __restrict__ partial, int64_t n, double* __restrict__ out) {
    __shared__ double red[32];
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc = __dadd_rn(acc, partial[i]);
    acc = block_reduce(acc, [](double a, double b) { return __dadd_rn(a, b); }, 0.0, red);
    if (threadIdx.x == 0) *out = acc;
}

}  // namespace

// ============================================================================
// host launchers
// ============================================================================

void plan_attention(ArenaPlan& p, const GroupView& g) {
    p.take<double>((size_t)g.G * g.P * g.L);
    p.take<double>((size_t)g.G * g.P);
}

void attention_grouped(cx_ctx* ctx, const GroupView& g, double* out, cudaStream_t s) {
    double* scores = ctx->arena.take<double>((size_t)g.G * g.P * g.L);
    double* sums = ctx->arena.take<double>((size_t)g.G * g.P);
    const double inv = 1.0 / std::sqrt((double)g.d_k);
    dim3 grid((unsigned)((g.L + 255) / 256), (unsigned)g.G);
    const bool fast = g.dim == 64 && g.d_k == 64 && g.P <= kAttnMaxP && (g.col_step == 0 || g.P == 1) &&
                      (g.rstride & 3) == 0 && (g.gstride & 3) == 0 && (reinterpret_cast<uintptr_t>(g.X) & 15) == 0;
    if (fast) {
        attn64_scores_kernel<<<grid, 256, 0, s>>>(g, inv, scores, ctx->d_flag);
        check_launch("attn64_scores_kernel");
    } else {
        attn_scores_kernel<<<grid, 256, 0, s>>>(g, inv, scores, ctx->d_flag);
        check_launch("attn_scores_kernel");
    }
    attn_softmax_kernel<<<g.G * g.P, 1024, 0, s>>>(g.L, g.P, scores, sums);
    check_launch("attn_softmax_kernel");
    attn_total_kernel<<<grid, 256, 0, s>>>(g.L, g.P, scores, sums, out);
    check_launch("attn_total_kernel");
}

namespace {

struct SelectPlan {
    int C, S, smem_rows;
    size_t smem;
};

SelectPlan plan_select_shape(const GroupView& g) {
    static int max_optin = -1;
    if (max_optin < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) v = 232448;
        max_optin = v;
    }
    SelectPlan pl;
    const int64_t want_rows = 512;
    pl.C = (int)std::min<int64_t>(kMaxCluster, std::max<int64_t>(1, (g.L + want_rows - 1) / want_rows));
    pl.S = (int)((g.L + pl.C - 1) / pl.C);
    pl.smem_rows = 1;
    size_t need = select_smem_layout(pl.S, g.dim, 1).total;
    if (need > (size_t)max_optin - 1024) {
        pl.smem_rows = 0;
        need = select_smem_layout(pl.S, g.dim, 0).total;
        if (need > (size_t)max_optin - 1024)
            fail(CX_DEVICE_ERROR, "select: group too large for one cluster (rows per CTA " + std::to_string(pl.S) + ")");
    }
    pl.smem = need;
    return pl;
}

}  // namespace

void plan_select(ArenaPlan& p, const GroupView& g, int k) {
    const int64_t take = std::min<int64_t>(k, g.L);
    p.take<double>((size_t)g.G * g.dim);        // centroids
    p.take<int64_t>((size_t)g.G * take);        // pick rows
    p.take<double>((size_t)g.G * take);         // pick scores
    p.take<double>((size_t)g.G * take * kGapRecStride);  // gap-monitor records
    p.take<char>(select_tc_scratch(g.G));               // select_tc cooperative exchanges
}

void centroid_launch(const GroupView& g, double* cen, cudaStream_t s) {
    if (g.dim > 1024) fail(CX_DEVICE_ERROR, "select: dim > 1024 unsupported");
    if (g.dim % 4 == 0 && g.dim <= 256 && g.rstride == g.dim && (g.gstride & 3) == 0 &&
        (reinterpret_cast<uintptr_t>(g.X) & 15) == 0) {
        // 128-row stages when rows are <= 256 B: every stage boundary costs ~200 cycles (mbarrier
        // wait, refilling the load -> widen pipeline, the block barrier, the refill issue), so
        // longer stages amortise it (32-row stages: 142 -> 110 us after removing a 64-bit % and
        // / per stage; see tools/cen_micro.cu)
        const int rows = g.dim <= 64 ? 128 : 32;
        const size_t stage_bytes = (size_t)rows * g.dim * sizeof(float);
        const int n_stages = (int)std::max<size_t>(2, std::min<size_t>(16, (160 * 1024) / stage_bytes));
        const size_t smem = 128 * (((size_t)n_stages * 8 + 127) / 128) + (size_t)n_stages * stage_bytes;
        if (rows == 128) {
            kernel_smem(centroid_tma_kernel<128>, smem);
            centroid_tma_kernel<128><<<(unsigned)g.G, (unsigned)g.dim, smem, s>>>(g, cen, n_stages);
        } else {
            kernel_smem(centroid_tma_kernel<32>, smem);
            centroid_tma_kernel<32><<<(unsigned)g.G, (unsigned)g.dim, smem, s>>>(g, cen, n_stages);
        }
        check_launch("centroid_tma_kernel");
    } else if (g.dim % 32 == 0 && (g.rstride & 3) == 0 && (g.gstride & 3) == 0 &&
        (reinterpret_cast<uintptr_t>(g.X) & 15) == 0) {
        centroid_pipe_kernel<<<dim3((unsigned)(g.dim / 32), (unsigned)g.G), 32, 0, s>>>(g, cen);
        check_launch("centroid_pipe_kernel");
    } else if (g.dim <= 256) {
        const size_t smem = sizeof(float) * 2 * kCenRows * g.dim;
        if (smem > 48 * 1024)
            kernel_smem(centroid_staged_kernel, smem);
        centroid_staged_kernel<<<g.G, 256, smem, s>>>(g, cen);
        check_launch("centroid_staged_kernel");
    } else {
        centroid_kernel<<<g.G, ((g.dim + 31) / 32) * 32, 0, s>>>(g, cen);
        check_launch("centroid_kernel");
    }
}

bool select_grouped(cx_ctx* ctx, const GroupView& g, const double* attn, int k, double lambda,
                    unsigned flags, int64_t* rows, double* scores, cudaStream_t s, const double* cen_in,
                    const SynGather* gat) {
    const int take = (int)std::min<int64_t>(k, g.L);
    if (take <= 0 || g.G <= 0) return true;  // nothing to gather either
    double* cen = ctx->arena.take<double>((size_t)g.G * g.dim);
    int64_t* pr = ctx->arena.take<int64_t>((size_t)g.G * take);
    double* ps = ctx->arena.take<double>((size_t)g.G * take);
    double* grec = ctx->arena.take<double>((size_t)g.G * take * kGapRecStride);
    char* tc_scratch = ctx->arena.take<char>(select_tc_scratch(g.G));

    if (cen_in) cen = const_cast<double*>(cen_in);
    else centroid_launch(g, cen, s);

    // decision-gap monitor output (cx_selection_gaps): one value per group, ctx-owned so it
    // outlives the call's arena scratch
    if (ctx->gaps_cap < g.G) {
        if (ctx->gaps) CX_CUDA(cudaFree(ctx->gaps));
        ctx->gaps = nullptr;
        ctx->gaps_cap = 0;
        CX_CUDA(cudaMalloc(&ctx->gaps, sizeof(double) * (size_t)g.G));
        ctx->gaps_cap = g.G;
    }
    ctx->gaps_n = g.G;
    const int impl = ctx->opt.select_impl;
    bool gathered = false;
    if (!(flags & CX_SELECT_GENERIC) && impl != CX_SELECT_IMPL_CUDA_CORE &&
        select_tc_launch(g, ctx->opt, attn, cen, take, lambda, flags, pr, ps, rows, scores, ctx->gaps, tc_scratch, s,
                         gat, &gathered))
        return gathered;
    if (impl == CX_SELECT_IMPL_TC && !(flags & CX_SELECT_GENERIC))
        fail(CX_PRECONDITION_ERROR, "select: the pinned tensor-core selection does not apply to this shape");
    if (!(flags & CX_SELECT_GENERIC) &&
        (select64_launch(g, ctx->opt, attn, cen, take, lambda, flags, pr, ps, rows, scores, ctx->gaps, grec, s) ||
         select128_launch(g, ctx->opt, attn, cen, take, lambda, flags, pr, ps, rows, scores, ctx->gaps, grec, s)))
        return false;
    // the generic kernel does not monitor: NaN (all-ones bits) = not measured
    CX_CUDA(cudaMemsetAsync(ctx->gaps, 0xFF, sizeof(double) * (size_t)g.G, s));

    SelectPlan pl = plan_select_shape(g);
    SelectParams prm;
    prm.gv = g;
    prm.attn = attn;
    prm.cen = cen;
    prm.take = take;
    prm.lambda = lambda;
    prm.S = pl.S;
    prm.smem_rows = pl.smem_rows;
    prm.filter = (flags & CX_SELECT_EXACT_ONLY) ? 0 : 1;
    prm.pick_rows = pr;
    prm.pick_scores = ps;
    prm.out_rows = rows;
    prm.out_scores = scores;

    kernel_smem(select_kernel, pl.smem, pl.C > 8);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)pl.C, (unsigned)g.G, 1);
    cfg.blockDim = dim3(512, 1, 1);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)pl.C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CX_CUDA(cudaLaunchKernelEx(&cfg, select_kernel, prm));
    count_launch();
    return false;
}

void gather_rows(const GroupView& g, const float* src, const int64_t* rows, int take, float* dst,
                 cudaStream_t s) {
    gather_rows2(g, src, nullptr, rows, take, dst, nullptr, (int64_t)take * g.dim, s);
}

void gather_rows2(const GroupView& g, const float* src0, const float* src1, const int64_t* rows, int take, float* dst0,
                  float* dst1, int64_t dst_gstride, cudaStream_t s) {
    if (take <= 0 || g.G <= 0) return;
    // several rows per 256-thread block when a row is <= 64 chunks of 16 B (dim <= 256, % 4)
    const bool multi = (g.dim & 3) == 0 && g.dim <= 256 && take > 1;
    const int rpb = multi ? 256 / (g.dim / 4) : 1;
    const unsigned gx = multi ? (unsigned)((take + rpb - 1) / rpb) : (unsigned)take;
    gather_rows_kernel<<<dim3(gx, (unsigned)g.G, src1 ? 2u : 1u), multi ? 256 : 64, 0, s>>>(g, src0, src1, rows, take,
                                                                                          dst0, dst1, dst_gstride, rpb);
    check_launch("gather_rows_kernel");
}

void coverage_selected(const GroupView& g, const int64_t* sel, int64_t n_sel, double* out, cudaStream_t s) {
    if (g.L <= 0) return;
    coverage_selected_kernel<<<(unsigned)((g.L + 255) / 256), 256, 0, s>>>(g, sel, n_sel, out);
    check_launch("coverage_selected_kernel");
}

void coverage_centroid(cx_ctx* ctx, const GroupView& g, double* out, cudaStream_t s) {
    if (g.L <= 0) return;
    double* cen = ctx->arena.take<double>((size_t)g.G * g.dim);
    centroid_launch(g, cen, s);
    coverage_centroid_kernel<<<dim3((unsigned)((g.L + 255) / 256), (unsigned)g.G), 256, sizeof(double) * g.dim, s>>>(
        g, cen, out);
    check_launch("coverage_centroid_kernel");
}

void hausdorff(const float* cloud, int64_t count, int dim, const float* lm, int64_t m, const int64_t* rows,
               double* out_worst_sq, cudaStream_t s) {
    CX_CUDA(cudaMemsetAsync(out_worst_sq, 0, sizeof(double), s));
    if (dim <= HD_MAXDIM) {
        const size_t smem = sizeof(double) * (size_t)(HD_ROWS + HD_T) * (size_t)(dim + 1);
        if (smem > 48 * 1024)
            kernel_smem(hausdorff_tile_kernel, smem);
        hausdorff_tile_kernel<<<(unsigned)((count + HD_ROWS - 1) / HD_ROWS), HD_ROWS, smem, s>>>(
            cloud, count, dim, lm, m, rows, reinterpret_cast<unsigned long long*>(out_worst_sq));
        check_launch("hausdorff_tile_kernel");
        return;
    }
    hausdorff_kernel<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(
        cloud, count, dim, lm, m, rows, reinterpret_cast<unsigned long long*>(out_worst_sq));
    check_launch("hausdorff_kernel");
}

size_t mean_pairwise_scratch(int64_t count, int dim) {
    if (dim > MP_MAXDIM) return (size_t)count + 1;
    const int64_t nt = (count + MP_T - 1) / MP_T;
    return 1 + (size_t)count * dim + (size_t)(nt * nt);
}

void mean_pairwise(const float* pts, int64_t count, int dim, const int64_t* rows, double* out_sum,
                   cudaStream_t s) {
    // scratch right after out_sum: mean_pairwise_scratch(count, dim) - 1 doubles
    if (dim > MP_MAXDIM) {  // wide rows: a CTA per row i (partial sums per row)
        double* partial = out_sum + 1;
        mean_pairwise_kernel<<<(unsigned)count, 256, 0, s>>>(pts, count, dim, rows, partial);
        check_launch("mean_pairwise_kernel");
        sum_partials_kernel<<<1, 1024, 0, s>>>(partial, count, out_sum);
        check_launch("sum_partials_kernel");
        return;
    }
    double* p64 = out_sum + 1;
    double* partial = p64 + (size_t)count * dim;
    const int64_t nt = (count + MP_T - 1) / MP_T;
    to_f64_kernel<<<(unsigned)std::min<int64_t>((count * dim + 255) / 256, 4096), 256, 0, s>>>(pts, count, dim, rows, p64);
    check_launch("to_f64_kernel");
    const size_t smem = sizeof(double) * 2 * MP_T * (size_t)(dim + 1);
    if (smem > 48 * 1024)
        kernel_smem(mean_pairwise_tile_kernel, smem);
    mean_pairwise_tile_kernel<<<dim3((unsigned)nt, (unsigned)nt), 256, smem, s>>>(p64, count, dim, partial);
    check_launch("mean_pairwise_tile_kernel");
    sum_partials_kernel<<<1, 1024, 0, s>>>(partial, nt * nt, out_sum);
    check_launch("sum_partials_kernel");
}

}  // namespace cx

// select64.cu -- the greedy hybrid selection (SURVEY.md §8(a) A4/A6,
// synapse.cpp:216-284) specialised for d = 64, the per-(layer, KV-head) key
// width of the 0.5B-class shape.  select128.cu compiles the same kernel for
// d = 128 (the head-concatenated reference-mode cloud) with no register rows.
//
// Layout: one thread-block cluster of C CTAs per group; CTA r owns rows
// [r*S, r*S+S).  Thread t owns rows t, 512+t, 1024+t, ...; row t lives in 64
// fp32 REGISTERS, the others in shared memory as fp32 (float4-interleaved,
// conflict-free) or as an fp16 SKETCH (the filter reads the sketch, the exact
// evaluations read the fp32 row from L2), or in L2 only.  C and the row mode
// come from a measured cost model (waves x per-round cost; a partial last wave
// is a separate launch).  All per-row state (running min distance, attention,
// bound threshold, removed flag) is in the owner's registers.  Per round:
//   U  distance update against the previous pick.  A Gram-form fp32 lower
//      bound (packed fma.rn.f32x2) rules out rows whose min cannot change;
//      the rest are queued and evaluated exactly in fp64 in the reference's
//      operation order by otherwise idle threads;
//   X1 cluster exchange of (amin, amax, cmin, cmax) over remaining rows;
//   H  hybrid argmax: a multiply-by-reciprocal fp64 approximation ranks all
//      rows; only rows within 1e-12 of the approximate maximum evaluate the
//      reference's exact divisions; exact argmax via two shared atomics
//      (max score bits, then min row among ties);
//   X2 cluster exchange of every CTA's (score, row, |b|^2, coordinates).
// Exchanges are DSMEM st.async pushes completing on a per-CTA mbarrier (no
// cluster-wide barrier per round).  Every decision is bit-identical to the
// reference.
#include <cooperative_groups.h>
#include <cuda_fp16.h>

#include <map>
#include <mutex>

#include "cx_internal.cuh"

namespace cg = cooperative_groups;

// entry points of this instantiation: select64_* (d = 64) or select128_* (select128.cu)
#define SEL_CAT2(a, b, c) a##b##_##c
#define SEL_CAT(a, b, c) SEL_CAT2(a, b, c)
#define SEL_FN(name) SEL_CAT(select, SEL_D, name)

namespace cx {

namespace {

#ifndef SEL_D
#define SEL_D 64
#endif
constexpr int D = SEL_D;         // row width of this instantiation (64; 128 via select128.cu)
constexpr int NT = 512;          // threads per CTA
constexpr int NW = NT / 32;
// d = 64: thread t keeps row t in 64 registers (RR = 512 register rows per CTA);
// d = 128 has no register rows: every row is a shared-memory (fp32 / sketch) row
constexpr bool REG = D == 64;
constexpr int RR = REG ? NT : 0;
constexpr int QCAP = D == 64 ? 160 : 96;  // exact-evaluation queue capacity per pass
#ifndef CX_QCAP_SK
#define CX_QCAP_SK 64
#endif
constexpr int QCAP_SK = CX_QCAP_SK;  // ... in sketch mode (64 leaves room for 1536 sketch rows)
// Rows beyond the 512 register rows of a CTA live in shared memory as fp32
// (ROWS_SMEM), or as an fp16 SKETCH there with the exact fp32 rows read from L2
// by the few exact evaluations (ROWS_SKETCH), or are read from L2 every round.
enum : int { ROWS_L2 = 0, ROWS_SMEM = 1, ROWS_SKETCH = 2 };
// staged-row pitch: 16-byte aligned rows (cp.async / float4 stores); the evaluators'
// float4 reads (thread t, row t) hit 8 distinct 16-byte slots per quarter warp
constexpr int SPITCH = D + 4;
constexpr int MAXC = 16;
static_assert(MAXC == kGapRecStride, "gap-monitor record stride");
constexpr int MAXRPT_ALL = 4;    // rows per thread (S <= 2048)
// decision-gap monitor window: rows whose approximate hybrid is within GAP_WINDOW of the
// CTA maximum are scored exactly, so the top-1 / top-2 gap of every round is known
// exactly when it is below GAP_WINDOW (and reported as GAP_WINDOW otherwise)
#ifndef CX_GAP_WINDOW
#define CX_GAP_WINDOW 1e-10
#endif
constexpr double GAP_WINDOW = CX_GAP_WINDOW;

__device__ __forceinline__ double dmin_std(double a, double b) { return (b < a) ? b : a; }  // std::min
__device__ __forceinline__ double dmax_std(double a, double b) { return (a < b) ? b : a; }  // std::max

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* m, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
    const uint32_t a = smem_u32(m);
    uint32_t ok = 0;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!ok);
}
// global -> shared 16 bytes without registers (L2 only); completes at cp.async.wait_all
__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t raddr, uint64_t a, uint64_t b, uint32_t rmbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
                 "l"(a), "l"(b), "r"(rmbar)
                 : "memory");
}
__device__ __forceinline__ void st_async_v4(uint32_t raddr, float4 v, uint32_t rmbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                     raddr),
                 "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y)), "r"(__float_as_uint(v.z)),
                 "r"(__float_as_uint(v.w)), "r"(rmbar)
                 : "memory");
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

struct Sel64Params {
    const float* X;
    int64_t gstride, rstride;
    int64_t L;
    const double* attn;  // [G][L]
    const double* cen;   // [G][D]
    int take;
    double lambda;
    int S;               // rows per CTA
    int Rs;              // rows per CTA beyond the register rows (S - RR, >= 0)
    int filter;
    int64_t* pick_rows;
    double* pick_scores;
    int64_t* out_rows;
    double* out_scores;
    long long* trace;    // optional per-round phase timestamps (CX_SEL_TRACE=1)
    double* gaps;        // [G]: smallest top-1 / top-2 hybrid gap over the rounds (capped at GAP_WINDOW)
    double* gap_rec;     // [G][take][MAXC] scratch: per round, each CTA's runner-up candidate
};

#ifdef CX_EXPERIMENTS  // per-round phase cycles (CX_SEL_TRACE=1; debugging builds only)
#define STAMP(k)                                                        \
    do {                                                                \
        if (p.trace && p.trace != (long long*)1 && tid == 0 && rank == 0 && g == 0 && round < 4096) \
            p.trace[round * 16 + (k)] = clock64();                      \
    } while (0)
#else
#define STAMP(k) \
    do {         \
    } while (0)
#endif

// X2 payload header: (score, row) + (|b|^2 of the candidate row, the CTA's second-best
// exact score in its gap window, -1 if none)
struct alignas(16) Hdr {
    double score;
    long long row;
    double nb;
    double second;
};

struct Sel64Layout {
    size_t mbar, mm, hdr, bc, cand, hw, misc, qown, qres, stage, xs, total;
};

__host__ __device__ inline size_t al(size_t x, size_t a = 16) { return (x + a - 1) / a * a; }

__host__ __device__ inline Sel64Layout sel64_layout(int Rs, int mode) {
    const int qcap = mode == ROWS_SKETCH ? QCAP_SK : QCAP;
    Sel64Layout l;
    size_t o = 0;
    l.mbar = o;  o = al(o + 2 * sizeof(uint64_t));
    l.mm = o;    o = al(o + sizeof(double) * 4 * MAXC);       // X1 slots
    l.hdr = o;   o = al(o + sizeof(Hdr) * MAXC);              // X2 headers
    l.bc = o;    o = al(o + sizeof(float) * D * MAXC);        // X2 coordinates
    l.cand = o;  o = al(o + sizeof(float) * D + sizeof(Hdr)); // this CTA's candidate (coords + header)
    l.hw = o;    o = al(o + sizeof(double) * 4 * NW);         // per-warp partials
    l.misc = o;  o = al(o + sizeof(unsigned long long) * 8);  // counters / atomics
    l.qown = o;  o = al(o + sizeof(int) * qcap);
    l.qres = o;  o = al(o + sizeof(double) * 2 * qcap);
    l.stage = o; o = al(o + sizeof(float) * qcap * SPITCH);
    l.xs = o;    o = al(o + (mode == ROWS_SMEM ? sizeof(float) * (size_t)Rs * D
                             : mode == ROWS_SKETCH ? sizeof(__half) * (size_t)Rs * D : 0));
    l.total = o;
    return l;
}

// exact sq_dist(point, pick) in the reference's order (synapse.cpp:18-25);
// the row is read through get4(c4) -> float4, the pick as floats (exact in fp64).
template <int UNR = 16, class Get4>
__device__ __forceinline__ double exact_sq(Get4 get4, const float* b) {
    double acc = 0.0;
#pragma unroll UNR
    for (int c4 = 0; c4 < D / 4; ++c4) {
        const float4 v = get4(c4);
        const float4 w = reinterpret_cast<const float4*>(b)[c4];
        double d = __dsub_rn((double)v.x, (double)w.x);
        acc = __dadd_rn(acc, __dmul_rn(d, d));
        d = __dsub_rn((double)v.y, (double)w.y);
        acc = __dadd_rn(acc, __dmul_rn(d, d));
        d = __dsub_rn((double)v.z, (double)w.z);
        acc = __dadd_rn(acc, __dmul_rn(d, d));
        d = __dsub_rn((double)v.w, (double)w.w);
        acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
    return acc;
}

// same against the fp64 centroid (sq_dist(span<float>, vector<double>), synapse.cpp:27-34)
template <int UNR = 16, class Get4>
__device__ __forceinline__ double exact_sq_d(Get4 get4, const double* b) {
    double acc = 0.0;
#pragma unroll UNR
    for (int c4 = 0; c4 < D / 4; ++c4) {
        const float4 v = get4(c4);
        double d = __dsub_rn((double)v.x, b[4 * c4]);
        acc = __dadd_rn(acc, __dmul_rn(d, d));
        d = __dsub_rn((double)v.y, b[4 * c4 + 1]);
        acc = __dadd_rn(acc, __dmul_rn(d, d));
        d = __dsub_rn((double)v.z, b[4 * c4 + 2]);
        acc = __dadd_rn(acc, __dmul_rn(d, d));
        d = __dsub_rn((double)v.w, b[4 * c4 + 3]);
        acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
    return acc;
}

// squared norm in fp64 (each square of an fp32 value is exact)
template <int UNR = 16, class Get4>
__device__ __forceinline__ double norm2(Get4 get4) {
    double acc = 0.0;
#pragma unroll UNR
    for (int c4 = 0; c4 < D / 4; ++c4) {
        const float4 v = get4(c4);
        acc += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
    }
    return acc;
}

// x . b in fp32 with packed FMAs (4 independent chains)
template <int UNR = 16, class Get4>
__device__ __forceinline__ float dot_f32x2(Get4 get4, const float* b) {
    float2 s0 = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f);
#pragma unroll UNR
    for (int c4 = 0; c4 < D / 4; ++c4) {
        const float4 v = get4(c4);
        const float4 w = reinterpret_cast<const float4*>(b)[c4];
        s0 = ffma2(make_float2(v.x, v.y), make_float2(w.x, w.y), s0);
        s1 = ffma2(make_float2(v.z, v.w), make_float2(w.z, w.w), s1);
    }
    return (s0.x + s0.y) + (s1.x + s1.y);
}

// Lower bound of the fp64 squared distance from the Gram form
// S = |x|^2 + |b|^2 - 2 x.b: every fp32 rounding above is
// covered by D u (|x|^2 + |b|^2), u = 2^-24 (64 u at d = 64, 128 u at d = 128),
// plus an underflow allowance.
constexpr float GRAM_SLACK = D * 0x1p-24f;
constexpr float SKETCH_SUB = D <= 64 ? 0x1p-21f : 0x1p-20f;
static_assert(D <= 128, "sketch subnormal term derived for d <= 128");
__device__ __forceinline__ float gram_lower_bound(float nx, float nb, float dot) {
    const float sum = __fadd_rn(nx, nb);
    const float s = __fsub_rn(sum, __fmul_rn(2.0f, dot));
    const float e = __fmaf_ru(GRAM_SLACK, sum, 0x1p-100f);
    // a non-finite dot (overflow; -inf would make the bound +inf) bounds nothing: -inf
    return isfinite(dot) ? __fsub_rd(s, e) : -INFINITY;
}

// The same bound when x is only known through its fp16 rounding x~ (the sketch):
// |x_c - x~_c| <= 2^-11 |x_c| + 2^-25 (subnormals), so |2 (x - x~).b| <= 2^-11 (|x|^2 +
// |b|^2) + 2^-24 sqrt(D) |b| (<= 2^-21 |b| at d = 64, 2^-20 |b| at d = 128), added to the slack.  An fp16 overflow makes the dot +-inf/NaN,
// the comparison false, and the row is evaluated exactly.
__device__ __forceinline__ float gram_lower_bound_sketch(float nx, float nb, float dot) {
    const float sum = __fadd_rn(nx, nb);
    const float s = __fsub_rn(sum, __fmul_rn(2.0f, dot));
    const float e = __fadd_ru(__fmaf_ru(GRAM_SLACK + 0x1p-11f, sum, 0x1p-100f), __fmul_ru(SKETCH_SUB, __fsqrt_ru(nb)));
    return isfinite(dot) ? __fsub_rd(s, e) : -INFINITY;  // fp16 overflow (+-inf / NaN): evaluate exactly
}

template <int RPT, int ROWMODE>
__global__ void __launch_bounds__(NT, 1) select64_kernel(Sel64Params p) {
    constexpr bool SMEM_ROWS = ROWMODE == ROWS_SMEM;
    constexpr int qcap = ROWMODE == ROWS_SKETCH ? QCAP_SK : QCAP;
    constexpr int MAXRPT = RPT;  // rows per thread of this instantiation
    cg::cluster_group cluster = cg::this_cluster();
    const uint32_t C = cluster.num_blocks();
    const uint32_t rank = cluster.block_rank();
    const int g = blockIdx.y;
    const int tid = threadIdx.x;
    const int lane = tid & 31, wid = tid >> 5;
    const int S = p.S;
    const int64_t r0 = (int64_t)rank * S;
    const int nrows = (int)max((int64_t)0, min((int64_t)S, p.L - r0));
    int round = -1;  // for STAMP outside the loop

    extern __shared__ __align__(16) unsigned char smem[];
    const Sel64Layout lay = sel64_layout(p.Rs, ROWMODE);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + lay.mbar);
    double* mm = reinterpret_cast<double*>(smem + lay.mm);
    Hdr* hdr = reinterpret_cast<Hdr*>(smem + lay.hdr);
    float* bc = reinterpret_cast<float*>(smem + lay.bc);
    float* cand = reinterpret_cast<float*>(smem + lay.cand);
    Hdr* cand_hdr = reinterpret_cast<Hdr*>(cand + D);
    double* hw = reinterpret_cast<double*>(smem + lay.hw);
    unsigned long long* misc = reinterpret_cast<unsigned long long*>(smem + lay.misc);
    int* qown = reinterpret_cast<int*>(smem + lay.qown);
    double* qres = reinterpret_cast<double*>(smem + lay.qres);
    float* stage = reinterpret_cast<float*>(smem + lay.stage);
    float4* xs4 = reinterpret_cast<float4*>(smem + lay.xs);  // [D/4][Rs] float4
    uint4* xh8 = reinterpret_cast<uint4*>(smem + lay.xs);    // sketch: [D/8][Rs] x 8 halves
    int* qn = reinterpret_cast<int*>(&misc[0]);              // queue length
    unsigned long long* hkey = &misc[1];                      // max exact score bits
    unsigned long long* hrow = &misc[2];                      // min row among ties
    unsigned long long* hkey2 = &misc[3];                     // [2] by round parity: second-best score bits
    unsigned long long* min_gap = &misc[5];                   // gap monitor: bits of the smallest gap (rank 0)
    unsigned long long* ties = &misc[6];                      // [2] by round parity: rows scoring the CTA max

    const float* gX = p.X + g * p.gstride + r0 * p.rstride;

    // ---- stage rows ---------------------------------------------------------
    float xr[D];
    if (REG && tid < nrows) {
        const float4* src = reinterpret_cast<const float4*>(gX + (int64_t)tid * p.rstride);
#pragma unroll
        for (int c4 = 0; c4 < D / 4; ++c4) {
            const float4 v = __ldg(src + c4);
            xr[4 * c4 + 0] = v.x; xr[4 * c4 + 1] = v.y; xr[4 * c4 + 2] = v.z; xr[4 * c4 + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int c = 0; c < D; ++c) xr[c] = 0.f;
    }
    const int nsm = max(0, nrows - RR);
    if (SMEM_ROWS) {
        for (int e = tid; e < nsm * (D / 4); e += NT) {
            const int j = e / (D / 4), c4 = e % (D / 4);
            xs4[(size_t)c4 * p.Rs + j] = __ldg(reinterpret_cast<const float4*>(gX + (int64_t)(RR + j) * p.rstride) + c4);
        }
    }
    if (ROWMODE == ROWS_SKETCH) {
        for (int e = tid; e < nsm * (D / 8); e += NT) {
            const int j = e / (D / 8), c8 = e % (D / 8);
            const float4* src = reinterpret_cast<const float4*>(gX + (int64_t)(RR + j) * p.rstride) + 2 * c8;
            const float4 u = __ldg(src), v = __ldg(src + 1);
            const __half2 h0 = __floats2half2_rn(u.x, u.y), h1 = __floats2half2_rn(u.z, u.w);
            const __half2 h2 = __floats2half2_rn(v.x, v.y), h3 = __floats2half2_rn(v.z, v.w);
            xh8[(size_t)c8 * p.Rs + j] = make_uint4(*reinterpret_cast<const uint32_t*>(&h0), *reinterpret_cast<const uint32_t*>(&h1),
                                                    *reinterpret_cast<const uint32_t*>(&h2), *reinterpret_cast<const uint32_t*>(&h3));
        }
    }
    __syncthreads();  // staged rows are written and read by different threads
    // x~ . b over the fp16 sketch of row RR + j
    auto sketch_dot = [&](int j, const float* b) {
        float2 s0 = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f);
#pragma unroll 4
        for (int c8 = 0; c8 < D / 8; ++c8) {
            const uint4 u = xh8[(size_t)c8 * p.Rs + j];
            const float4 w0 = reinterpret_cast<const float4*>(b)[2 * c8], w1 = reinterpret_cast<const float4*>(b)[2 * c8 + 1];
            const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
            const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
            const float2 f2 = __half22float2(*reinterpret_cast<const __half2*>(&u.z));
            const float2 f3 = __half22float2(*reinterpret_cast<const __half2*>(&u.w));
            s0 = ffma2(f0, make_float2(w0.x, w0.y), s0);
            s1 = ffma2(f1, make_float2(w0.z, w0.w), s1);
            s0 = ffma2(f2, make_float2(w1.x, w1.y), s0);
            s1 = ffma2(f3, make_float2(w1.z, w1.w), s1);
        }
        return (s0.x + s0.y) + (s1.x + s1.y);
    };
    auto reg4 = [&](int c4) { return make_float4(xr[4 * c4], xr[4 * c4 + 1], xr[4 * c4 + 2], xr[4 * c4 + 3]); };
    auto far4 = [&](int j) {  // row RR + j
        return [&, j](int c4) -> float4 {
            if (SMEM_ROWS) return xs4[(size_t)c4 * p.Rs + j];
            return __ldg(reinterpret_cast<const float4*>(gX + (int64_t)(RR + j) * p.rstride) + c4);
        };
    };

    // ---- per-row state in registers: rows tid + k*NT -------------------------
    const int nr = tid < nrows ? 1 + (nrows - 1 - tid) / NT : 0;
    double m[MAXRPT], a[MAXRPT];
    float th[MAXRPT], nx[MAXRPT];
    uint32_t remm = 0;
    {
        const double* cen = p.cen + (int64_t)g * D;  // L1-resident broadcast reads
#pragma unroll
        for (int k = 0; k < MAXRPT; ++k) {
            m[k] = 0.0; a[k] = 0.0; th[k] = INFINITY; nx[k] = 0.f;
            if (k < nr) {
                const int li = tid + k * NT;
                a[k] = p.attn[(int64_t)g * p.L + r0 + li];
                // coverage init: distance to the centroid (synapse.cpp:107-112)
                if (REG && k == 0) {
                    m[k] = __dsqrt_rn(exact_sq_d(reg4, cen));
                    nx[k] = (float)norm2(reg4);
                } else {
                    m[k] = __dsqrt_rn(exact_sq_d<2>(far4(li - RR), cen));
                    nx[k] = (float)norm2<2>(far4(li - RR));
                }
                remm |= 1u << k;
            }
        }
    }
    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        qn[0] = 0;
        *hkey = 0ull;
        *hrow = ~0ull;
        hkey2[0] = hkey2[1] = 0ull;
        ties[0] = ties[1] = 0ull;
        *min_gap = (unsigned long long)__double_as_longlong(GAP_WINDOW);
    }
    __syncthreads();
    cluster.sync();  // mbarriers visible cluster-wide before any remote push
    const uint32_t tx1 = C * 32u, tx2 = C * (uint32_t)(sizeof(Hdr) + D * sizeof(float));
    if (tid == 0) {
        mbar_arrive_expect(&mbar[0], tx1);
        mbar_arrive_expect(&mbar[1], tx2);
    }

    const double lam = p.lambda;
    const double one_m_lam = __dsub_rn(1.0, lam);
    int64_t* pick_rows = p.pick_rows + (int64_t)g * p.take;
    double* pick_scores = p.pick_scores + (int64_t)g * p.take;
    uint32_t ph1 = 0, ph2 = 0;
    const float* bw = nullptr;  // winner coordinates of the previous round (in bc)
    float nbw = 0.f;

    for (round = 0; round < p.take; ++round) {
        STAMP(0);
        // ======== U: distance update against the previous pick ========
        if (round > 0) {
            const bool assign = (round == 1);  // the first pick REPLACES the centroid distances
            int slot[MAXRPT];
#pragma unroll
            for (int k = 0; k < MAXRPT; ++k) {
                slot[k] = -1;
                if (k >= nr || !(remm >> k & 1u)) continue;
                bool need;
                if (assign || !p.filter) {
                    need = true;
                } else {
                    if (ROWMODE == ROWS_SKETCH && !(REG && k == 0)) {
                        need = !(gram_lower_bound_sketch(nx[k], nbw, sketch_dot(tid + k * NT - RR, bw)) > th[k]);
                    } else {
                        const float dt = (REG && k == 0) ? dot_f32x2(reg4, bw) : dot_f32x2<4>(far4(tid + k * NT - RR), bw);
                        need = !(gram_lower_bound(nx[k], nbw, dt) > th[k]);
                    }
                }
                if (!need) continue;
                const int sl = atomicAdd(qn, 1);
                if (sl < qcap) {
                    slot[k] = sl;
                    qown[sl] = tid;
                    float* st = stage + sl * SPITCH;
                    if (!SMEM_ROWS && !(REG && k == 0)) {
                        // sketch / L2 rows: the fp32 row comes from L2 asynchronously, so the
                        // owner moves on and all queued rows' fetches overlap in one round trip
                        const float* src = gX + (int64_t)(tid + k * NT) * p.rstride;
#pragma unroll
                        for (int c4 = 0; c4 < D / 4; ++c4) cp_async16(st + 4 * c4, src + 4 * c4);
                    } else {
#pragma unroll
                        for (int c4 = 0; c4 < D / 4; ++c4)
                            reinterpret_cast<float4*>(st)[c4] = (REG && k == 0) ? reg4(c4) : far4(tid + k * NT - RR)(c4);
                    }
                } else {  // queue full: evaluate in place
                    const double d2 = (REG && k == 0) ? exact_sq(reg4, bw) : exact_sq<2>(far4(tid + k * NT - RR), bw);
                    const double d = __dsqrt_rn(d2);
                    if (assign || d < m[k]) {
                        m[k] = d;
                        th[k] = __double2float_ru(d2);
                    }
                }
            }
            if (p.trace && p.trace != (long long*)1) {  // tracing only: split filter / staging wait
                __syncthreads();
                STAMP(9);
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncthreads();
            STAMP(6);
            if (p.trace && p.trace != (long long*)1 && tid == 0 && rank == 0 && g == 0 && round < 4096)
                p.trace[round * 16 + 8] = qn[0];  // rows queued for exact evaluation (before the cap)
            const int nq = min(qn[0], qcap);
            if (tid < nq) {
                const float4* st = reinterpret_cast<const float4*>(stage + tid * SPITCH);
                const double d2 = exact_sq<2>([&](int c4) { return st[c4]; }, bw);
                qres[2 * tid] = d2;
                qres[2 * tid + 1] = __dsqrt_rn(d2);
            }
            __syncthreads();
            STAMP(7);
            if (tid == 0) qn[0] = 0;  // next use is after >= 2 more barriers
#pragma unroll
            for (int k = 0; k < MAXRPT; ++k) {
                if (slot[k] < 0) continue;
                const double d2 = qres[2 * slot[k]], d = qres[2 * slot[k] + 1];
                if (assign || d < m[k]) {  // round 1 assigns; later rounds take std::min
                    m[k] = d;
                    th[k] = __double2float_ru(d2);
                }
            }
        }
        STAMP(1);

        // ======== X1: cluster-wide min/max over remaining rows ========
        double amin = INFINITY, amax = -INFINITY, cmin = INFINITY, cmax = -INFINITY;
#pragma unroll
        for (int k = 0; k < MAXRPT; ++k) {
            if (!(remm >> k & 1u)) continue;
            amin = dmin_std(amin, a[k]);
            amax = dmax_std(amax, a[k]);
            cmin = dmin_std(cmin, m[k]);
            cmax = dmax_std(cmax, m[k]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            amin = dmin_std(amin, __shfl_xor_sync(0xffffffffu, amin, o));
            amax = dmax_std(amax, __shfl_xor_sync(0xffffffffu, amax, o));
            cmin = dmin_std(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
            cmax = dmax_std(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
        }
        if (lane == 0) {
            hw[wid] = amin; hw[NW + wid] = amax; hw[2 * NW + wid] = cmin; hw[3 * NW + wid] = cmax;
        }
        __syncthreads();
        if (wid == 0) {
            double v0 = lane < NW ? hw[lane] : INFINITY;
            double v1 = lane < NW ? hw[NW + lane] : -INFINITY;
            double v2 = lane < NW ? hw[2 * NW + lane] : INFINITY;
            double v3 = lane < NW ? hw[3 * NW + lane] : -INFINITY;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                v0 = dmin_std(v0, __shfl_xor_sync(0xffffffffu, v0, o));
                v1 = dmax_std(v1, __shfl_xor_sync(0xffffffffu, v1, o));
                v2 = dmin_std(v2, __shfl_xor_sync(0xffffffffu, v2, o));
                v3 = dmax_std(v3, __shfl_xor_sync(0xffffffffu, v3, o));
            }
            if (lane < (int)C) {
                const uint32_t dst = mapa(smem_u32(mm + rank * 4), lane);
                const uint32_t mb = mapa(smem_u32(&mbar[0]), lane);
                st_async_v2(dst, __double_as_longlong(v0), __double_as_longlong(v1), mb);
                st_async_v2(dst + 16, __double_as_longlong(v2), __double_as_longlong(v3), mb);
            }
        }
        STAMP(2);
        mbar_wait(&mbar[0], ph1);
        ph1 ^= 1u;
        if (tid == 0 && round + 1 < p.take) mbar_arrive_expect(&mbar[0], tx1);
        {
            double v0 = lane < (int)C ? mm[lane * 4 + 0] : INFINITY;
            double v1 = lane < (int)C ? mm[lane * 4 + 1] : -INFINITY;
            double v2 = lane < (int)C ? mm[lane * 4 + 2] : INFINITY;
            double v3 = lane < (int)C ? mm[lane * 4 + 3] : -INFINITY;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                v0 = dmin_std(v0, __shfl_xor_sync(0xffffffffu, v0, o));
                v1 = dmax_std(v1, __shfl_xor_sync(0xffffffffu, v1, o));
                v2 = dmin_std(v2, __shfl_xor_sync(0xffffffffu, v2, o));
                v3 = dmax_std(v3, __shfl_xor_sync(0xffffffffu, v3, o));
            }
            amin = v0; amax = v1; cmin = v2; cmax = v3;
        }
        STAMP(3);

        // ======== H: hybrid argmax (synapse.cpp:247-260) ========
        const bool a_span = amax > amin, c_span = cmax > cmin;
        const double ar = __dsub_rn(amax, amin), cr = __dsub_rn(cmax, cmin);
        const double iar = a_span ? __drcp_rn(ar) : 0.0, icr = c_span ? __drcp_rn(cr) : 0.0;
        double happ[MAXRPT];
        double hmax = -1.0;
#pragma unroll
        for (int k = 0; k < MAXRPT; ++k) {
            happ[k] = -1.0;
            if (!(remm >> k & 1u)) continue;
            const double na = __dmul_rn(__dsub_rn(a[k], amin), iar);
            const double nc = __dmul_rn(__dsub_rn(m[k], cmin), icr);
            happ[k] = __dadd_rn(__dmul_rn(lam, nc), __dmul_rn(one_m_lam, na));
            hmax = dmax_std(hmax, happ[k]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) hmax = dmax_std(hmax, __shfl_xor_sync(0xffffffffu, hmax, o));
        if (lane == 0) hw[wid] = hmax;  // hw (X1 partials) is dead: every warp passed the X1 wait
        __syncthreads();
        {
            double v = lane < NW ? hw[lane] : -1.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v = dmax_std(v, __shfl_xor_sync(0xffffffffu, v, o));
            hmax = v;
        }
        // the reciprocal form is within ~1e-15 of the exact hybrid unless a range
        // is so small that 1/range leaves the normal range: then rank exactly
        const bool approx_ok = (!a_span || ar >= 1e-290) && (!c_span || cr >= 1e-290);
        const double cut = approx_ok ? hmax - GAP_WINDOW : -INFINITY;
        double hex[MAXRPT];
#pragma unroll
        for (int k = 0; k < MAXRPT; ++k) {
            hex[k] = -1.0;
            if (!(remm >> k & 1u) || happ[k] < cut) continue;
            const double na = a_span ? __ddiv_rn(__dsub_rn(a[k], amin), ar) : 0.0;
            const double nc = c_span ? __ddiv_rn(__dsub_rn(m[k], cmin), cr) : 0.0;
            hex[k] = __dadd_rn(__dmul_rn(lam, nc), __dmul_rn(one_m_lam, na));
            // hybrid >= 0 (both terms are), so the bit pattern orders like the value
            atomicMax(hkey, (unsigned long long)__double_as_longlong(hex[k]));
        }
        __syncthreads();
        const unsigned long long kbest = *hkey;
#pragma unroll
        for (int k = 0; k < MAXRPT; ++k) {
            if (!(remm >> k & 1u) || hex[k] < 0.0) continue;
            const unsigned long long kb = (unsigned long long)__double_as_longlong(hex[k]);
            if (kb == kbest) {
                atomicMin(hrow, (unsigned long long)(r0 + tid + k * NT));  // strict >: lowest row wins ties
                atomicAdd(&ties[round & 1], 1ull);  // gap monitor: > 1 means a runner-up equal to the winner
            } else {
                atomicMax(&hkey2[round & 1], kb);  // gap monitor: the CTA's best below the winner
            }
        }
        __syncthreads();
        const unsigned long long rbest = *hrow;
#ifdef CX_EXPERIMENTS
        if (p.trace == (long long*)1 && round < 3 && tid < 64 && (remm & 1u))
            printf("r%d tid%d a=%.17g m=%.17g happ=%.17g hex=%.17g | amin=%.17g amax=%.17g cmin=%.17g cmax=%.17g hmax=%.17g kbest=%llx rbest=%llx\n",
                   round, tid, a[0], m[0], happ[0], hex[0], amin, amax, cmin, cmax, hmax, kbest, rbest);
#endif
        if (rbest != ~0ull) {  // owner of the local winner publishes its coordinates
            const int li = (int)((long long)rbest - r0);
            if (REG && li < NT) {
                if (tid == li) {
#pragma unroll
                    for (int c4 = 0; c4 < D / 4; ++c4) reinterpret_cast<float4*>(cand)[c4] = reg4(c4);
                    cand_hdr->nb = (double)nx[0];
                }
            } else if (tid == (li & (NT - 1))) {
                const int k = li / NT;
                auto get = far4(li - RR);
#pragma unroll
                for (int c4 = 0; c4 < D / 4; ++c4) reinterpret_cast<float4*>(cand)[c4] = get(c4);
#pragma unroll
                for (int kk = REG ? 1 : 0; kk < MAXRPT; ++kk)
                    if (kk == k) cand_hdr->nb = (double)nx[kk];
            }
        } else if (tid < D) {
            cand[tid] = 0.f;
            if (tid == 0) cand_hdr->nb = 0.0;
        }
        __syncthreads();
        STAMP(4);

        // ======== X2: push (score, row, |b|^2, coordinates) to every CTA ========
        if (tid < (int)C) {
            const uint32_t dst = mapa(smem_u32(hdr + rank), tid);
            const uint32_t mb = mapa(smem_u32(&mbar[1]), tid);
            const double sc = rbest != ~0ull ? __longlong_as_double((long long)kbest) : -1.0;
            const long long rw = rbest != ~0ull ? (long long)rbest : LLONG_MAX;
            st_async_v2(dst, __double_as_longlong(sc), (uint64_t)rw, mb);
            const unsigned long long k2 = ties[round & 1] > 1ull ? kbest : hkey2[round & 1];  // after the barrier above
            st_async_v2(dst + 16, __double_as_longlong(cand_hdr->nb),
                        (uint64_t)__double_as_longlong(k2 ? __longlong_as_double((long long)k2) : -1.0), mb);
        }
        for (int e = tid - 32; tid >= 32 && e < (int)C * (D / 4); e += NT - 32) {
            const int dst_rank = e / (D / 4), c4 = e % (D / 4);
            const uint32_t dst = mapa(smem_u32(bc + rank * D + 4 * c4), dst_rank);
            st_async_v4(dst, reinterpret_cast<const float4*>(cand)[c4], mapa(smem_u32(&mbar[1]), dst_rank));
        }
        if (tid == 0) {  // reset the argmax atomics (next use is after >= 2 more barriers)
            *hkey = 0ull;
            *hrow = ~0ull;
            hkey2[(round + 1) & 1] = 0ull;  // next round's; this round's may still be read above
            ties[(round + 1) & 1] = 0ull;
        }
        mbar_wait(&mbar[1], ph2);
        ph2 ^= 1u;
        if (tid == 0 && round + 1 < p.take) mbar_arrive_expect(&mbar[1], tx2);
        // winner across the cluster (every warp, same order -> same answer)
        double bs = lane < (int)C ? hdr[lane].score : -1.0;
        long long br = lane < (int)C ? hdr[lane].row : LLONG_MAX;
        int w = lane;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double os = __shfl_xor_sync(0xffffffffu, bs, o);
            const long long orow = __shfl_xor_sync(0xffffffffu, br, o);
            const int ow = __shfl_xor_sync(0xffffffffu, w, o);
            if (os > bs || (os == bs && orow < br)) { bs = os; br = orow; w = ow; }
        }
        if (rank == 0 && lane < (int)C && wid == 0 && p.gap_rec)  // gap monitor record (see below)
            p.gap_rec[((int64_t)g * p.take + round) * MAXC + lane] = lane == w ? hdr[lane].second : hdr[lane].score;
        bw = bc + w * D;
        nbw = (float)hdr[w].nb;
        if (br >= r0 && br < r0 + nrows) {
            const int li = (int)(br - r0);
            if (tid == (li & (NT - 1))) remm &= ~(1u << (li / NT));
        }
        if (tid == 0 && rank == 0) {
            pick_rows[round] = br;
            pick_scores[round] = bs;
        }
        STAMP(5);
    }

    // ---- sort the picks ascending by row (synapse.cpp:276-277) ----
    __syncthreads();
    // ---- decision-gap monitor: per round, the runner-up is the winning CTA's second or
    // another CTA's best (recorded above, a tie with the winner included); a row outside
    // every CTA's window scores < winner - GAP_WINDOW (+ ~1e-15) ----
    if (rank == 0 && p.gaps) {
        for (int r = tid; r < p.take; r += NT) {
            const double* rec = p.gap_rec + ((int64_t)g * p.take + r) * MAXC;
            double b2 = -1.0;
            for (int c = 0; c < (int)C; ++c) b2 = dmax_std(b2, rec[c]);
            if (b2 >= 0.0) {
                const double gap = dmin_std(__dsub_rn(pick_scores[r], b2), GAP_WINDOW);
                atomicMin(min_gap, (unsigned long long)__double_as_longlong(gap));  // gap >= 0: bits order
            }
        }
        __syncthreads();
        if (tid == 0) p.gaps[g] = __longlong_as_double((long long)*min_gap);
    }
    if (rank == 0) {
        int64_t* out_rows = p.out_rows + (int64_t)g * p.take;
        double* out_scores = p.out_scores + (int64_t)g * p.take;
        for (int s = tid; s < p.take; s += NT) {
            const int64_t r = pick_rows[s];
            int pos = 0;
            for (int t = 0; t < p.take; ++t) pos += pick_rows[t] < r;
            out_rows[pos] = r;
            out_scores[pos] = pick_scores[s];
        }
    }
    cluster.sync();  // no CTA exits while a peer may still push into it
}

}  // namespace

// Host side: choose the cluster size and residency, launch.  Returns false
// when the dim-64 kernel does not apply (caller uses the generic kernel).
// co-resident clusters of size C for the on-chip (shared-memory rows) kernel, cached
static void (*sel64_kernel_for(int rpt, int mode))(Sel64Params) {
    if (mode == ROWS_SMEM)
        return rpt <= 1 ? select64_kernel<1, ROWS_SMEM> : rpt <= 2 ? select64_kernel<2, ROWS_SMEM> : select64_kernel<4, ROWS_SMEM>;
    if (mode == ROWS_SKETCH)
        return rpt <= 1 ? select64_kernel<1, ROWS_SKETCH> : rpt <= 2 ? select64_kernel<2, ROWS_SKETCH>
                                                              : select64_kernel<4, ROWS_SKETCH>;
    return rpt <= 1 ? select64_kernel<1, ROWS_L2> : rpt <= 2 ? select64_kernel<2, ROWS_L2> : select64_kernel<4, ROWS_L2>;
}

static int active_clusters(int C, int Rs, int S, int mode = ROWS_SMEM) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, int> cache;
    const size_t smem = sel64_layout(Rs, mode).total;
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_pair(C * 4 + mode, (int)smem);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    const int rpt = (S + NT - 1) / NT;
    void (*kern)(Sel64Params) = sel64_kernel_for(rpt, mode);
    int n = 0;
    bool attr_ok = true;
    try {
        kernel_smem(kern, smem, C > 8);  // the attribute only ever grows (a later launch may need more)
    } catch (const Failure&) {
        attr_ok = false;
    }
    if (attr_ok) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)C, 1, 1);
        cfg.blockDim = dim3(NT, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) n = 0;
    }
    cudaGetLastError();  // an unsupported query leaves no sticky error behind
    cache[key] = n;
    return n;
}

// Among the on-chip cluster sizes >= c_min, the one minimising waves x per-round cost
// for G groups.  Per-round cost was measured to be ~3.6 us + 0.0037 us per row per CTA
// on B200 (C=8: 7.4 us, C=9: 7.2 us, C=16: 5.5 us at L=8192); waves = ceil(G /
// co-resident clusters).  cfg2 (G=48): C=9 (4.71 vs 4.86 ms at C=8); G <= 7 (one
// group, or cfg2 over 8 GPUs): C=16.  Returns the estimated cost (us per round).
static double best_cluster(int G, int64_t L, size_t budget, int* C, int* S, int* Rs, int* mode, int* act_out,
                           bool sketch_ok = true) {
    double best = 1e300;
    for (int c = 1; c <= MAXC; ++c) {
        const int s_ = (int)((L + c - 1) / c), rs = std::max(0, s_ - RR);
        if (s_ > MAXRPT_ALL * NT) continue;
        // fp32 rows on chip if they fit, else the fp16 sketch (rows re-read from L2 only
        // by the exact evaluations): measured ~15% more per round (C=6: 10.1 us, C=5:
        // 11.6 us per round against 8.7 / 9.7 us for fp32 rows of the same count)
        int md = ROWS_SMEM;
        double per = 3.6 + 0.0037 * s_;
        if (sel64_layout(rs, ROWS_SMEM).total > budget) {
            if (!sketch_ok || sel64_layout(rs, ROWS_SKETCH).total > budget) continue;
            md = ROWS_SKETCH;
            per *= 1.15;
        }
        const int act = active_clusters(c, rs, s_, md);
        if (act <= 0) continue;
        const double cost = (double)((G + act - 1) / act) * per;
        if (cost < best * (1.0 - 1e-9)) {
            best = cost;
            *C = c; *S = s_; *Rs = rs; *mode = md;
            *act_out = act;
        }
    }
    return best;
}

// groups per wave of the configuration the cost model picks for G groups of L rows
// (0 when the dim-64 kernel would not run on chip)
int SEL_FN(wave)(int64_t L, int G) {
    static int max_optin = -1;
    if (max_optin < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
            max_optin = 232448;
    }
    int C = 0, S = 0, Rs = 0, mode = 0, act = 0;
    best_cluster(G, L, (size_t)max_optin - 2048, &C, &S, &Rs, &mode, &act);
    return C > 0 ? act : 0;
}

bool SEL_FN(launch)(const GroupView& g, const Options& o, const double* attn, const double* cen, int take,
                     double lambda, unsigned flags, int64_t* pick_rows, double* pick_scores, int64_t* rows, double* scores,
                     double* gaps, double* gap_rec, cudaStream_t s) {
    if (g.dim != D || (g.rstride & 3) != 0 || (g.gstride & 3) != 0 ||
        (reinterpret_cast<uintptr_t>(g.X) & 15) != 0 || g.L < 1)
        return false;
    static int max_optin = -1;
    if (max_optin < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
            max_optin = 232448;
    }
    const size_t budget = (size_t)max_optin - 2048;
    // Cluster size and row mode by the cost model (best_cluster): waves x per-round cost
    // over every C whose rows fit on chip as fp32 or as the fp16 sketch.  A partial last
    // wave (e.g. 48 = 15 + 15 + 15 + 3 clusters) runs as its own launch with the
    // configuration best for that many groups, after the full waves.
    int C = 0, S = 0, Rs = 0, mode = ROWS_SMEM, act = 0;
    if (o.select_cluster > 0) {  // CX_OPT_SELECT_CLUSTER (tests / tuning): force a cluster size
        const int c = o.select_cluster;
        const int s_ = (int)((g.L + c - 1) / c), rs = std::max(0, s_ - RR);
        if (c >= 1 && c <= MAXC && s_ <= MAXRPT_ALL * NT) {
            C = c; S = s_; Rs = rs;
            mode = sel64_layout(rs, ROWS_SMEM).total <= budget                        ? ROWS_SMEM
                   : !o.select_no_sketch && sel64_layout(rs, ROWS_SKETCH).total <= budget ? ROWS_SKETCH
                                                                                         : ROWS_L2;
        }
    } else {
        const bool sk = !o.select_no_sketch;
        const double cost = best_cluster(g.G, g.L, budget, &C, &S, &Rs, &mode, &act, sk);
        const int full = act > 0 ? (g.G / act) * act : 0, rem = g.G - full;
        if (C > 0 && full > 0 && rem > 0) {
            int c1, s1, r1, m1, a1, c2, s2, r2, m2, a2;
            const double cost2 = best_cluster(full, g.L, budget, &c1, &s1, &r1, &m1, &a1, sk) +
                                 best_cluster(rem, g.L, budget, &c2, &s2, &r2, &m2, &a2, sk);
            if (cost2 < cost * 0.98) {
                GroupView ga = g, gb = g;
                ga.G = full;
                gb.G = rem;
                gb.X = g.X + (int64_t)full * g.gstride;
                const int64_t off = (int64_t)full * take;
                return SEL_FN(launch)(ga, o, attn, cen, take, lambda, flags, pick_rows, pick_scores, rows, scores,
                                      gaps, gap_rec, s) &&
                       SEL_FN(launch)(gb, o, attn + (int64_t)full * g.L, cen + (int64_t)full * D, take, lambda, flags,
                                       pick_rows + off, pick_scores + off, rows + off, scores + off,
                                       gaps ? gaps + full : nullptr, gap_rec ? gap_rec + off * MAXC : nullptr, s);
            }
        }
    }
    if (C == 0) {  // nothing fits on chip: rows beyond 512 per CTA are read from L2 every round
        C = MAXC;
        S = (int)((g.L + C - 1) / C);
        Rs = std::max(0, S - RR);
        if (S > MAXRPT_ALL * NT) return false;
        mode = ROWS_L2;
    }
    Sel64Params prm;
    prm.X = g.X;
    prm.gstride = g.gstride;
    prm.rstride = g.rstride;
    prm.L = g.L;
    prm.attn = attn;
    prm.cen = cen;
    prm.take = take;
    prm.lambda = lambda;
    prm.S = S;
    prm.Rs = Rs;
    prm.filter = (flags & CX_SELECT_EXACT_ONLY) ? 0 : 1;
    prm.pick_rows = pick_rows;
    prm.pick_scores = pick_scores;
    prm.out_rows = rows;
    prm.out_scores = scores;
    prm.trace = nullptr;
    prm.gaps = gap_rec ? gaps : nullptr;
    prm.gap_rec = gap_rec;
#ifdef CX_EXPERIMENTS  // build-time debugging only (CX_NVCC_EXTRA=-DCX_EXPERIMENTS): per-phase cycles
    const char* tr = getenv("CX_SEL_TRACE");
    if (tr && tr[0] == '1') CX_CUDA(cudaMallocManaged(&prm.trace, sizeof(long long) * 16 * 4096));
    if (tr && tr[0] == 'p') prm.trace = (long long*)1;
#endif
    const size_t smem = sel64_layout(Rs, mode).total;
    const int rpt = (S + NT - 1) / NT;
    void (*kern)(Sel64Params) = sel64_kernel_for(rpt, mode);
    kernel_smem(kern, smem, C > 8);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)C, (unsigned)g.G, 1);
    cfg.blockDim = dim3(NT, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
#ifdef CX_EXPERIMENTS
    if (getenv("CX_SEL_OCC")) {  // debugging: co-resident clusters for this configuration
        int ncl = 0;
        cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
        fprintf(stderr, "select64: C=%d S=%d Rs=%d smem=%zu max active clusters=%d groups=%d\n", C, S, Rs, smem, ncl, g.G);
    }
#endif
    CX_CUDA(cudaLaunchKernelEx(&cfg, kern, prm));
    count_launch();
#ifdef CX_EXPERIMENTS
    const char* dump = getenv("CX_SEL_DUMP");
    if (dump && dump[0] == '1') {  // debugging aid: picks in selection order (group 0)
        CX_CUDA(cudaStreamSynchronize(s));
        std::vector<int64_t> pr(take);
        std::vector<double> ps(take);
        CX_CUDA(cudaMemcpy(pr.data(), pick_rows, sizeof(int64_t) * take, cudaMemcpyDeviceToHost));
        CX_CUDA(cudaMemcpy(ps.data(), pick_scores, sizeof(double) * take, cudaMemcpyDeviceToHost));
        for (int i = 0; i < std::min(take, 12); ++i) fprintf(stderr, "pick %d: row %lld score %.17g\n", i, (long long)pr[i], ps[i]);
    }
    if (prm.trace && prm.trace != (long long*)1) {  // debugging aid: average cycles per phase over rounds 2..take-2
        CX_CUDA(cudaStreamSynchronize(s));
        double acc[11] = {0};
        int n = 0;
        for (int r = 2; r < std::min(take, 4096) - 1; ++r, ++n) {
            const long long* t = prm.trace + r * 16;
            for (int k = 0; k < 5; ++k) acc[k] += (double)(t[k + 1] - t[k]);
            acc[5] += (double)(prm.trace[(r + 1) * 16] - t[0]);
            acc[6] += (double)(t[6] - t[0]);  // filter + staging
            acc[10] += (double)(t[9] - t[0]);  // filter + staging issue (before the cp.async wait)
            acc[7] += (double)(t[7] - t[6]);  // exact evaluation
            acc[8] += (double)(t[1] - t[7]);  // apply
            acc[9] += (double)t[8];           // queued rows
        }
        if (n > 0)
            fprintf(stderr, "select%d C=%d S=%d Rs=%d rows=%d cycles/round: U=%.0f (filter+stage %.0f, exact %.0f, "
                            "apply %.0f; %.1f rows queued; filter+issue %.0f) X1send=%.0f X1wait=%.0f H=%.0f X2=%.0f total=%.0f\n",
                    D, C, S, Rs, mode, acc[0] / n, acc[6] / n, acc[7] / n, acc[8] / n, acc[9] / n, acc[10] / n, acc[1] / n,
                    acc[2] / n, acc[3] / n, acc[4] / n, acc[5] / n);
        cudaFree(prm.trace);
    }
#endif
    return true;
}

}  // namespace cx

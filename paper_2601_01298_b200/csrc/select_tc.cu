// select_tc.cu -- the greedy hybrid selection (SURVEY.md §8(a) A4/A6,
// synapse.cpp:216-284) for d = 64 with the distance filter on the 5th-generation
// tensor cores and every row on chip, so that cfg2's 48 groups run in ONE wave.
//
// Why: the selection is k dependent rounds; per round every remaining row needs
// min(m_i, |x_i - b|) against the new pick b.  On-chip capacity decides the wave
// count: cfg2 holds 48 x 8192 rows, 2657 rows per SM for a single wave -- 340 KB
// as fp16, more than shared memory.  Here a CTA keeps its rows as an fp16 SKETCH
// split between shared memory (UMMA core-matrix tiles) and TENSOR MEMORY (the A
// operand of tcgen05.mma may live in TMEM), up to 22 tiles of 128 rows = 2816
// rows per CTA.  Per round ONE thread issues the filter GEMV on the tensor cores:
// D[row] = x~ . [b_hi | b_lo] (M = 128 rows per MMA, N = 8, K = 64 in 4 steps,
// fp32 accumulate in TMEM), every thread reads its rows' dots with tcgen05.ld and
// forms the conservative lower bound of the Gram form; only rows
// the bound cannot rule out are evaluated exactly -- in fp64, in the reference's
// operation order, from the fp32 row in global memory (L2).  No fp32 row is kept
// in registers, so the 512 threads carry just the per-row state.
//
// The cluster exchanges (X1 min / max, X2 candidates) and the exact hybrid argmax
// are the select64 protocol: every decision is bit-identical to
// the reference.
//
// Rows: thread (warp w, lane l) owns rows tile*128 + 32 (w % 4) + l of the tiles
// j = w / 4 + (NW / 4) k, k = 0..RPT-1 (tcgen05.ld: a warp reads the TMEM lanes of its
// sub-partition w % 4).  NT = 512 threads (CX_SEL_NT=1024 builds a 3-rows-per-thread variant:
// 1.3-2.5 KB of spills at 64 registers, cfg2 selection 2.27 ms against 1.66 ms; not used).  Tiles [0, n_smem) are in shared memory, [n_smem, n_tiles)
// in TMEM columns [tm_rows_col + 32 (j - n_smem), +32).
#include <cooperative_groups.h>
#include <cuda_fp16.h>

#include <map>
#include <tuple>
#include <mutex>

#include "cx_internal.cuh"

namespace cg = cooperative_groups;

namespace cx {

namespace {

constexpr int D = 64;
#ifndef CX_SEL_NT
#define CX_SEL_NT 512
#endif
constexpr int NT = CX_SEL_NT;  // threads per CTA (1024: 3 rows per thread at 22 tiles, 64 registers)
constexpr int NW = NT / 32;
constexpr int TILE = 128;         // rows per MMA (M)
constexpr int MAXT = 22;          // tiles per CTA: 2816 rows
constexpr int DC = 8;             // TMEM columns of one D block (N = 8)
// D packing: the 4 tiles of a block share one 8-column D block; tile q of the block multiplies
// B operand q = [0 ... b_hi b_lo (columns 2q, 2q+1) ... 0], so its two dots land in columns
// 2q, 2q+1 and the other tiles add exact zeros there.  One warp issues a block's 4 tiles in
// order (the first MMA overwrites, the rest accumulate).  D then takes 8 columns per 4 tiles
// instead of per tile, and TMEM holds 14 row tiles instead of 10 at 22 tiles (fewer A reads
// from shared memory: an SS MMA moves 4 KB through shared memory, a TS one none)
#ifndef CX_SEL_NO_DPACK
constexpr int DPACK = 4;
#else
constexpr int DPACK = 1;
#endif
constexpr int MAXC = 16;
constexpr int TILE_BYTES = TILE * D * 2;  // one fp16 A tile: 16 KB
constexpr double GAP_WINDOW = 1e-10;      // as select64.cu (gap monitor + exact window)
static_assert(MAXC == kGapRecStride, "gap-monitor record stride");
static_assert((MAXT + DPACK - 1) / DPACK * DC <= 512 - 32 * 10, "D and 10 row tiles fill TMEM at 22 tiles");
// first TMEM column of the row tiles: after the D blocks (8 columns per DPACK tiles)
__host__ __device__ inline int tm_rows_col(int n_tiles) { return (DC * ((n_tiles + DPACK - 1) / DPACK) + 31) / 32 * 32; }
__host__ __device__ inline int n_dblocks(int n_tiles) { return (n_tiles + DPACK - 1) / DPACK; }

__device__ __forceinline__ double dmin_std(double a, double b) { return (b < a) ? b : a; }
// Every value reduced below is a non-negative double (attention mass, distances, hybrid
// scores in [0, 1]; never -0.0), and those order like their bit patterns as unsigned
// integers: warp min / max are two redux.sync on the 32-bit halves.
__device__ __forceinline__ unsigned long long dbits(double x) { return (unsigned long long)__double_as_longlong(x); }
__device__ __forceinline__ double bitsd(unsigned long long b) { return __longlong_as_double((long long)b); }
__device__ __forceinline__ unsigned long long wmax64(unsigned long long v) {
    const uint32_t hi = (uint32_t)(v >> 32), lo = (uint32_t)v;
    const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
    const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    return ((unsigned long long)mh << 32) | ml;
}
__device__ __forceinline__ unsigned long long wmin64(unsigned long long v) {
    const uint32_t hi = (uint32_t)(v >> 32), lo = (uint32_t)v;
    const uint32_t mh = __reduce_min_sync(0xffffffffu, hi);
    const uint32_t ml = __reduce_min_sync(0xffffffffu, hi == mh ? lo : 0xffffffffu);
    return ((unsigned long long)mh << 32) | ml;
}
constexpr unsigned long long BITS_INF = 0x7FF0000000000000ull;  // +inf: the min identity (max: 0)

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* m, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
    const uint32_t a = su32(m);
    uint32_t ok = 0;
    do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok)
                     : "r"(a), "r"(parity)
                     : "memory");
    } while (!ok);
}
// TMA bulk copy global -> shared completing on an mbarrier (transaction bytes)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(mbar))
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(su32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* m) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(m)) : "memory");
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

// ---- tcgen05 helpers ----
// K-major SWIZZLE_NONE core-matrix layout: 8 rows x 16 B core matrices, row groups
// 128 B apart (SBO), 8-element K chunks (R / 8) * 128 B apart (LBO)
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
// kind::f16 instruction descriptor: A = B = fp16 (format 0), D = fp32, K-major A and B
__host__ __device__ __forceinline__ uint32_t idesc_f16_f32(int m, int n) {
    return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
// warp-uniform issue: the whole warp runs the code (operands stay in uniform registers),
// one elected lane issues -- ~10x cheaper per MMA than a divergent single thread (measured)
__device__ __forceinline__ void mma_ss_elect(uint32_t dt, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{ .reg .pred p, e; setp.ne.b32 p, %4, 0; elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(dt),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_ts_elect(uint32_t dt, uint32_t at, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{ .reg .pred p, e; setp.ne.b32 p, %4, 0; elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }" ::"r"(dt),
        "r"(at), "l"(bd), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_commit_elect(uint64_t* mbar) {
    asm volatile(
        "{ .reg .pred e; elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0]; }" ::"r"(su32(mbar))
        : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
__device__ __forceinline__ void tmem_ld2(uint32_t taddr, uint32_t& a, uint32_t& b) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(taddr));
}

// exact sq_dist(x, b) in the reference's order (synapse.cpp:18-25); x read as float4
template <class Get4>
__device__ __forceinline__ double exact_sq(Get4 get4, const float* b) {
    double acc = 0.0;
#pragma unroll
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

// Lower bound of the fp64 squared distance from the tensor-core Gram form.
// dot = x~ . (b_hi + b_lo): x~ = fp16(x) (|x_c - x~_c| <= 2^-11 |x_c| + 2^-25), b_hi + b_lo
// = b to 2^-22 |b_c| + 2^-25, products exact in fp32, 64 fp32 accumulations (<= 2^-17 of the
// absolute sum even with truncating adds).  With 2 |x.b| <= |x|^2 + |b|^2 and |x| + |b| <=
// 1 + (|x|^2 + |b|^2) / 2, every term is covered by 2^-9.9 (|x|^2 + |b|^2) + 2^-19, plus the
// fp32 roundings of the bound itself.  An fp16 overflow (|x_c| or |b_c| > 65504) makes the
// dot non-finite: then nothing is bounded and the row is evaluated exactly.
__device__ __forceinline__ float tc_lower_bound(float nx, float nb, float dot) {
    const float sum = __fadd_rn(nx, nb);
    const float s = __fsub_rn(sum, __fmul_rn(2.0f, dot));
    const float e = __fmaf_ru(0x1.1p-10f, sum, 0x1p-19f);
    return isfinite(dot) ? __fsub_rd(s, e) : -INFINITY;
}

struct alignas(16) Hdr {
    double score;
    long long row;
    double nb;
    double second;
};

struct SelxParams {
    const float* X;
    int64_t gstride, rstride;
    int64_t L;
    const double* attn;  // [G][L]
    const double* cen;   // [G][D]
    int take;
    double lambda;
    int S;               // rows per CTA
    int n_tiles;         // ceil(S / 128)
    int n_smem;          // tiles in shared memory (the rest in TMEM)
    int n_stage;         // staging slots for the exact rows (TMA bulk copies)
    int filter;
    int64_t* pick_rows;
    double* pick_scores;
    int64_t* out_rows;
    double* out_scores;
    double* gaps;
    long long* trace;
    // cooperative (non-cluster) mode: the exchanges go through global memory
    unsigned long long* x1g;  // [G][2 parity][C * NW][4]: (amin, amax, cmin, cmax) bits
    Hdr* x2h;                 // [G][2][C * NW]: (score, row, |b|^2, runner-up)
    float* x2c;               // [G][2][C * NW][D]: the candidates' coordinates
    unsigned* cnt;            // [G][2]: monotonic arrival counters (zeroed per launch)
    int C;                    // CTAs per group  // CX_EXPERIMENTS builds: per-round phase clocks of group 0, rank 0
    // the fused landmark gather (A5, synapse.cpp:303-318): rank 0 copies the sorted picks'
    // key rows (from X) and value rows (from V, the keys' group layout) into syn_k / syn_v
    const float* V;
    float* syn_k;
    float* syn_v;
    int64_t syn_gs;
};

#ifdef CX_EXPERIMENTS
#define XSTAMP(k)                                                                         \
    do {                                                                                  \
        if (p.trace && tid == 0 && rank == 0 && g == 0 && round < 4096) p.trace[round * 16 + (k)] = clock64(); \
    } while (0)
#else
#define XSTAMP(k) \
    do {          \
    } while (0)
#endif


struct SelxLayout {
    size_t mbar, mm, hdr, bc, loc, misc, qrow, qres, bop, stage, tiles, total;
};

__host__ __device__ inline size_t al(size_t x, size_t a = 16) { return (x + a - 1) / a * a; }

__host__ __device__ inline SelxLayout selx_layout(int n_smem, int C, int n_stage) {
    SelxLayout l;
    size_t o = 0;
    l.mbar = o;  o = al(o + 5 * sizeof(uint64_t));
    l.mm = o;    o = al(o + sizeof(double) * 4 * C * NW);  // X1: one slot per (CTA, warp)
    l.hdr = o;   o = al(o + sizeof(Hdr) * C * NW);        // X2: one candidate per (CTA, warp)
    l.bc = o;    o = al(o + sizeof(float) * D * C * NW);
    l.loc = o;   o = al(o + NW * (4 * sizeof(unsigned long long) + sizeof(Hdr) + D * sizeof(float)));  // per-warp partials
    l.misc = o;  o = al(o + sizeof(unsigned long long) * 8);
    l.qrow = o;  o = al(o + sizeof(int) * NT);         // exact-evaluation queue: local row
    l.qres = o;  o = al(o + sizeof(double) * 2 * NT);  // ... and its (d^2, d)
    l.bop = o;   o = al(o + DPACK * 8 * D * 2, 1024);  // DPACK B operands: 8 rows (b_hi, b_lo at 2q, 2q+1; 0...) x 64 fp16
    l.stage = o; o = al(o + (size_t)n_stage * D * sizeof(float), 1024);  // exact rows (fp32)
    l.tiles = o; o = al(o + (size_t)n_smem * TILE_BYTES, 1024);
    l.total = o;
    return l;
}

// CL: the group's CTAs form a thread-block cluster and exchange through DSMEM pushes.
// !CL: a cooperative launch (all CTAs co-resident, any SMs: one wave when C x G <= 148, which
// clusters cannot reach -- 45 co-resident clusters of 3 on B200) and the exchanges go through
// global memory: every warp writes its slot and bumps the group's counter; one poller per CTA
// waits for the count, then one TMA bulk copy brings the whole exchange into shared memory,
// completing on the same mbarrier the cluster pushes would.
template <int RPT, bool CL>
__global__ void __launch_bounds__(NT, 1) selx_kernel(SelxParams p) {
    const uint32_t C = CL ? cg::this_cluster().num_blocks() : (uint32_t)p.C;
    const uint32_t rank = CL ? cg::this_cluster().block_rank() : blockIdx.x;
    const int g = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int sub = wid & 3, quad = wid >> 2;  // TMEM sub-partition, tile phase
    const int64_t r0 = (int64_t)rank * p.S;
    const int nrows = (int)max((int64_t)0, min((int64_t)p.S, p.L - r0));

    extern __shared__ __align__(1024) unsigned char smem[];
    const SelxLayout lay = selx_layout(p.n_smem, (int)C, p.n_stage);
    float* stage = reinterpret_cast<float*>(smem + lay.stage);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + lay.mbar);  // [0] X1, [1] X2, [2] MMA, [3] TMEM base, [4] stage
    double* mm = reinterpret_cast<double*>(smem + lay.mm);
    Hdr* hdr = reinterpret_cast<Hdr*>(smem + lay.hdr);
    float* bc = reinterpret_cast<float*>(smem + lay.bc);
    unsigned long long* misc = reinterpret_cast<unsigned long long*>(smem + lay.misc);
    unsigned long long* loc1 = reinterpret_cast<unsigned long long*>(smem + lay.loc);  // [NW][4]
    Hdr* locH = reinterpret_cast<Hdr*>(loc1 + 4 * NW);                                 // [NW]
    float* locC = reinterpret_cast<float*>(locH + NW);                                 // [NW][D]
    int* qrow = reinterpret_cast<int*>(smem + lay.qrow);
    double* qres = reinterpret_cast<double*>(smem + lay.qres);
    unsigned char* bop = smem + lay.bop;
    unsigned char* tiles = smem + lay.tiles;
    uint32_t* tbase_s = reinterpret_cast<uint32_t*>(&mbar[3]);
    int* qn = reinterpret_cast<int*>(&misc[0]);
    unsigned long long* min_gap = &misc[5];

    const float* gX = p.X + g * p.gstride + r0 * p.rstride;
    // a split plan's cooperative part may launch once every CTA of this grid is resident
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    // the CTA's fp32 rows -> L2 (the exact evaluations and the winners' coordinates read them
    // from global memory every round: an L2 hit instead of an HBM round trip)
    if (p.rstride == D) {
        const char* base = reinterpret_cast<const char*>(gX);
        const size_t bytes = (size_t)nrows * D * sizeof(float);
        for (size_t o = (size_t)tid * 4096; o < bytes; o += (size_t)NT * 4096)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + o), "r"((uint32_t)min((size_t)4096, bytes - o))
                         : "memory");
    }
    if (wid == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tbase_s)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int e = tid; e < DPACK * 8 * D * 2 / 16; e += NT) reinterpret_cast<uint4*>(bop)[e] = make_uint4(0, 0, 0, 0);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = *tbase_s;

    // ---- rows: per-row state in registers, fp16 sketch in shared memory / TMEM ----
    double m[RPT], a[RPT];
    float th[RPT], nx[RPT];
    uint32_t remm = 0;
    {
        const double* cen = p.cen + (int64_t)g * D;
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
            m[k] = 0.0; a[k] = 0.0; th[k] = INFINITY; nx[k] = 0.f;
            const int j = quad + (NW / 4) * k;
            if (j >= p.n_tiles) continue;
            const int li = j * TILE + 32 * sub + lane;
            const bool valid = li < nrows;
            float x[D];
            if (valid) {
                const float4* src = reinterpret_cast<const float4*>(gX + (int64_t)li * p.rstride);
#pragma unroll
                for (int c4 = 0; c4 < D / 4; ++c4) {
                    const float4 v = __ldg(src + c4);
                    x[4 * c4] = v.x; x[4 * c4 + 1] = v.y; x[4 * c4 + 2] = v.z; x[4 * c4 + 3] = v.w;
                }
                a[k] = p.attn[(int64_t)g * p.L + r0 + li];
                // coverage init: distance to the centroid (synapse.cpp:107-112, sq_dist :27-34)
                double acc = 0.0, n2 = 0.0;
#pragma unroll
                for (int c = 0; c < D; ++c) {
                    const double d = __dsub_rn((double)x[c], cen[c]);
                    acc = __dadd_rn(acc, __dmul_rn(d, d));
                    n2 += (double)x[c] * x[c];
                }
                m[k] = __dsqrt_rn(acc);
                nx[k] = (float)n2;
                remm |= 1u << k;
            } else {
#pragma unroll
                for (int c = 0; c < D; ++c) x[c] = 0.f;
            }
            // the fp16 sketch (padding rows are zero and never enter a decision)
            uint32_t h[32];
#pragma unroll
            for (int u = 0; u < 32; ++u) {
                const __half2 v = __floats2half2_rn(x[2 * u], x[2 * u + 1]);
                h[u] = *reinterpret_cast<const uint32_t*>(&v);
            }
            if (j < p.n_smem) {
                unsigned char* t = tiles + (size_t)j * TILE_BYTES;
                const int r = 32 * sub + lane;
#pragma unroll
                for (int c = 0; c < D / 8; ++c)
                    *reinterpret_cast<uint4*>(t + cm_off(r, 8 * c, TILE)) =
                        make_uint4(h[4 * c], h[4 * c + 1], h[4 * c + 2], h[4 * c + 3]);
            } else {
                tmem_st32(tbase + ((uint32_t)(32 * sub) << 16) + (uint32_t)(tm_rows_col(p.n_tiles) + 32 * (j - p.n_smem)), h);
            }
        }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        mbar_init(&mbar[2], (uint32_t)min(n_dblocks(p.n_tiles), NW));  // one commit per MMA-issuing warp
        mbar_init(&mbar[4], 1);  // the exact rows' bulk copies (tx bytes) + one arrival
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        *qn = 0;
        *min_gap = (unsigned long long)__double_as_longlong(GAP_WINDOW);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (CL) cg::this_cluster().sync();  // mbarriers visible cluster-wide before any remote push
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tx1 = C * NW * 32u, tx2 = C * NW * (uint32_t)(sizeof(Hdr) + D * sizeof(float));
    if (CL && tid == 0) {
        mbar_arrive_expect(&mbar[0], tx1);
        mbar_arrive_expect(&mbar[1], tx2);
    }
    // Cooperative mode (CX_SEL_COOP_COUNTER: the previous protocol, kept for A/B).  Warp 0
    // writes the CTA's slot, then bumps the group's counter with a release add; one poller per
    // CTA (thread 0) acquires the count, then ONE TMA bulk copy brings the whole exchange into
    // shared memory, completing on the same mbarrier the cluster pushes would.  The default
    // stamped protocol below needs one L2 round trip instead of three: cooperative round
    // 19.1K -> 16.0K cycles (4 CTAs), cfg2 compression 1.81 -> 1.70 ms.
#ifndef CX_SEL_COOP_COUNTER
    // Stamped exchange (the default).  Every 64-bit word of a slot carries the round's stamp in
    // bit 63 (all payload words are non-negative double bit patterns or row indices, so the bit
    // is free): stamp = 1 - ((round >> 1) & 1), the slots are zeroed per launch, and each slot
    // buffer (round parity) is rewritten only two rounds later, after every CTA has read it.
    // A writer stores its words relaxed -- no fence, no counter -- and warp 0 of every CTA
    // polls the C slots' words until all carry this round's stamp: one L2 round trip after the
    // last writer, instead of fence + counter add + counter poll + bulk copy.
    constexpr unsigned long long TOPB = 1ull << 63;
    constexpr unsigned long long SENT = 0x7FF8000000000001ull;  // encodes -1.0 (no candidate)
    auto stamp_of = [](int round_) { return (unsigned long long)(1 - ((round_ >> 1) & 1)) << 63; };
    auto st_word = [](unsigned long long* a, unsigned long long v) {
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
    };
    auto ld_word = [](const unsigned long long* a) {
        unsigned long long v;
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
        return v;
    };
    // warp 0: the C slots' 4 C words of this round -> out[0 .. 4C) with the stamps removed
    auto poll_slots = [&](const unsigned long long* slots, int round_, unsigned long long* out) {
        const unsigned long long want = stamp_of(round_);
        const int nwd = 4 * (int)C;
        unsigned long long v0, v1;
        bool ok;
        do {
            v0 = lane < nwd ? ld_word(slots + lane) : want;
            v1 = lane + 32 < nwd ? ld_word(slots + lane + 32) : want;
            ok = (v0 & TOPB) == want && (v1 & TOPB) == want;
        } while (!__all_sync(0xffffffffu, ok));
        if (lane < nwd) out[lane] = v0 & ~TOPB;
        if (lane + 32 < nwd) out[lane + 32] = v1 & ~TOPB;
    };
#endif
#ifdef CX_SEL_COOP_COUNTER
    auto bump = [&](int which) {  // after warp 0's slot writes
        __syncwarp();
        if (lane == 0) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");  // the warp's writes (observed via the sync)
            asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(p.cnt + 2 * g + which) : "memory");
        }
    };
    auto gather = [&](int which, int round_, uint32_t bytes) {
        if (tid != 0) return;
        const unsigned target = C * (unsigned)(round_ + 1);  // one slot per CTA
        const unsigned* c = p.cnt + 2 * g + which;
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
        } while ((int)(v - target) < 0);
        asm volatile("fence.proxy.async.global;" ::: "memory");  // generic writes -> the bulk copy
        const int par = round_ & 1;
        mbar_arrive_expect(&mbar[which], bytes);
        if (which == 0) {
            bulk_g2s(mm, p.x1g + ((size_t)(2 * g + par) * C) * 4, C * 32u, &mbar[0]);
        } else {
            bulk_g2s(hdr, p.x2h + (size_t)(2 * g + par) * C, C * (uint32_t)sizeof(Hdr), &mbar[1]);
            bulk_g2s(bc, p.x2c + (size_t)(2 * g + par) * C * D, C * D * (uint32_t)sizeof(float), &mbar[1]);
        }
    };
#endif

    const double lam = p.lambda;
    const double one_m_lam = __dsub_rn(1.0, lam);
    int64_t* pick_rows = p.pick_rows + (int64_t)g * p.take;
    double* pick_scores = p.pick_scores + (int64_t)g * p.take;
    uint32_t ph1 = 0, ph2 = 0, ph3 = 0, ph4 = 0;
    const float* bw = nullptr;  // the previous round's winner coordinates (in bc)
    float nbw = 0.f;
    const uint32_t idesc = idesc_f16_f32(TILE, 8);
    // MMA operands that never change: B descriptors per k-step, the A descriptor of shared tile 0,
    // the first TMEM column of the row tiles
    // B descriptor of operand q, k-step kk: bdesc0 + ((q * 1024 + kk * 256) >> 4) (address field)
    const uint64_t bdesc0 = sdesc(su32(bop), 128, 128);
    const uint64_t adesc0 = sdesc(su32(tiles), (TILE / 8) * 128, 128);
    const uint32_t tm_col = (uint32_t)tm_rows_col(p.n_tiles);

    for (int round = 0; round < p.take; ++round) {
        XSTAMP(0);
        // ======== U: distance update against the previous pick ========
        if (round > 0) {
            const bool assign = (round == 1);  // the first pick REPLACES the centroid distances
            const bool use_tc = !assign && p.filter;
            if (use_tc) {
                // B = [b_hi; b_lo; 0 ...] (fp16, K-major core matrices), then one thread issues
                // the filter GEMV over every tile: D[:, 0] = x~ . b_hi, D[:, 1] = x~ . b_lo
                if (tid < D) {
                    const float bcv = bw[tid];
                    const __half hi = __float2half_rn(bcv);
                    const __half lo = __float2half_rn(bcv - __half2float(hi));
#pragma unroll
                    for (int q = 0; q < DPACK; ++q) {
                        *reinterpret_cast<__half*>(bop + q * 8 * D * 2 + cm_off(2 * q % 8, tid, 8)) = hi;
                        *reinterpret_cast<__half*>(bop + q * 8 * D * 2 + cm_off((2 * q + 1) % 8, tid, 8)) = lo;
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                }
                __syncthreads();  // the B operand is written
                // The filter GEMV: lane 0 of warp w issues D block w's tiles 4w .. 4w + 3 in order
                // (k-step major per tile; the block's first MMA overwrites, the rest accumulate)
                // and commits: the mbarrier counts one arrival per issuing warp.
                if (wid < n_dblocks(p.n_tiles)) {  // warp-uniform: blocks wid, wid + NW, ...
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    for (int blk = wid; blk < n_dblocks(p.n_tiles); blk += NW) {
                    const uint32_t dt = tbase + (uint32_t)(DC * blk);
#pragma unroll
                    for (int q = 0; q < DPACK; ++q) {
                        const int j = DPACK * blk + q;
                        if (j >= p.n_tiles) break;
                        const uint64_t bq = bdesc0 + (uint64_t)((q * 8 * D * 2) >> 4);
                        if (j >= p.n_smem) {
                            const uint32_t at = tbase + (uint32_t)(tm_col + 32 * (j - p.n_smem));
#pragma unroll
                            for (int kk = 0; kk < D / 16; ++kk)
                                mma_ts_elect(dt, at + 8 * kk, bq + (uint64_t)((kk * 2 * 128) >> 4), idesc, q | kk);
                        } else {
                            const uint64_t ad = adesc0 + (uint64_t)((j * TILE_BYTES) >> 4);
#pragma unroll
                            for (int kk = 0; kk < D / 16; ++kk)
                                mma_ss_elect(dt, ad + (uint64_t)((kk * 2 * (TILE / 8) * 128) >> 4),
                                             bq + (uint64_t)((kk * 2 * 128) >> 4), idesc, q | kk);
                        }
                    }
                    }
                    mma_commit_elect(&mbar[2]);
                }
                mbar_wait(&mbar[2], ph3);
                ph3 ^= 1u;
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            }
            XSTAMP(1);
            float dot[RPT];
            if (use_tc) {
                uint32_t dh[RPT], dl[RPT];
#pragma unroll
                for (int k = 0; k < RPT; ++k) {
                    const int j = quad + (NW / 4) * k;
                    dh[k] = dl[k] = 0u;
                    if (j < p.n_tiles)
                        tmem_ld2(tbase + ((uint32_t)(32 * sub) << 16) + (uint32_t)(DC * (j / DPACK) + 2 * (j % DPACK)), dh[k],
                                 dl[k]);
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int k = 0; k < RPT; ++k) dot[k] = __uint_as_float(dh[k]) + __uint_as_float(dl[k]);
            }
            // rows the bound cannot rule out are evaluated exactly in fp64 from their fp32 row
            // in global memory (L2).  Rounds >= 2 (~3% of rows): a block-wide queue, one
            // evaluator thread per queued row, so all the row reads are one round trip.  Round 1
            // (every row, it replaces the centroid distances): each owner evaluates its rows.
            uint32_t need = 0;
#pragma unroll
            for (int k = 0; k < RPT; ++k)
                if ((remm >> k & 1u) && (!use_tc || !(tc_lower_bound(nx[k], nbw, dot[k]) > th[k]))) need |= 1u << k;
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");  // D read before the next MMA
            int slot[RPT];
#pragma unroll
            for (int k = 0; k < RPT; ++k) {
                slot[k] = -1;
                if (!assign && (need >> k & 1u)) {
                    const int sl = atomicAdd(qn, 1);
                    if (sl < NT) {
                        slot[k] = sl;
                        const int li = (quad + (NW / 4) * k) * TILE + 32 * sub + lane;
                        qrow[sl] = li;
                        need &= ~(1u << k);
#ifndef CX_SEL_NO_QPREFETCH
                        // the evaluator thread reads this row after the block barrier: start
                        // its two 128-B lines towards L1 now (the L2 / HBM latency overlaps
                        // the rest of the bound pass and the barrier)
                        {
                            const float* rp = gX + (int64_t)li * p.rstride;
                            asm volatile("prefetch.global.L1 [%0];\n\tprefetch.global.L1 [%1];" ::"l"(rp), "l"(rp + 32));
                        }
#endif
                        if (sl < p.n_stage) {  // the row starts moving now (TMA), not after the barrier
                            mbar_expect_tx(&mbar[4], D * sizeof(float));
                            bulk_g2s(stage + sl * D, gX + (int64_t)li * p.rstride, D * sizeof(float), &mbar[4]);
                        }
                    }
                }
            }
            while (__any_sync(0xffffffffu, need != 0)) {  // round 1, or a queue overflow
                const int k = need ? __ffs(need) - 1 : 0;
                const int li = (quad + (NW / 4) * k) * TILE + 32 * sub + lane;
                const float4* src = reinterpret_cast<const float4*>(gX + (int64_t)li * p.rstride);
                float4 x4[D / 4];
#pragma unroll
                for (int c4 = 0; c4 < D / 4; ++c4) x4[c4] = need ? __ldg(src + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
                const double d2 = exact_sq([&](int c4) { return x4[c4]; }, bw);
                const double d = __dsqrt_rn(d2);
#pragma unroll
                for (int kk = 0; kk < RPT; ++kk) {
                    if (need && kk == k && (assign || d < m[kk])) {
                        m[kk] = d;
                        th[kk] = __double2float_ru(d2);
                    }
                }
                need &= need - 1;
            }
            __syncthreads();
            XSTAMP(2);
            const int nq = min(*qn, NT);
            if (!assign) {
                if (tid == 0) mbar_arrive(&mbar[4]);  // every expect_tx is in: the phase ends with the copies
                if (tid < nq) {
                    double d2;
                    if (tid < p.n_stage) {
                        mbar_wait(&mbar[4], ph4);
                        const float4* st = reinterpret_cast<const float4*>(stage + tid * D);
                        d2 = exact_sq([&](int c4) { return st[c4]; }, bw);
                    } else {
                        const float4* src = reinterpret_cast<const float4*>(gX + (int64_t)qrow[tid] * p.rstride);
                        float4 x4[D / 4];
#pragma unroll
                        for (int c4 = 0; c4 < D / 4; ++c4) x4[c4] = __ldg(src + c4);
                        d2 = exact_sq([&](int c4) { return x4[c4]; }, bw);
                    }
                    qres[2 * tid] = d2;
                    qres[2 * tid + 1] = __dsqrt_rn(d2);
                }
                ph4 ^= 1u;
            }
            __syncthreads();
            XSTAMP(3);
#ifdef CX_EXPERIMENTS
            if (p.trace && tid == 0 && rank == 0 && g == 0 && round < 4096) p.trace[round * 16 + 8] = *qn;
#endif
            if (tid == 0) *qn = 0;  // next use is after >= 2 more barriers
#pragma unroll
            for (int k = 0; k < RPT; ++k) {
                if (slot[k] < 0) continue;
                const double d2 = qres[2 * slot[k]], d = qres[2 * slot[k] + 1];
                if (d < m[k]) {  // std::min (round 1 never queues)
                    m[k] = d;
                    th[k] = __double2float_ru(d2);
                }
            }
        }

        // ======== X1: cluster-wide min/max over remaining rows ========
        double amin, amax, cmin, cmax;
        {
            // per-thread min / max in fp64 (one DMNMX each; the values are finite and >= 0, so the
            // fp64 order is the order of their bit patterns the warp reductions use)
            double f0 = INFINITY, f1 = 0.0, f2 = INFINITY, f3 = 0.0;
#pragma unroll
            for (int k = 0; k < RPT; ++k) {
                const bool r = remm >> k & 1u;
                f0 = fmin(f0, r ? a[k] : INFINITY);
                f1 = fmax(f1, r ? a[k] : 0.0);
                f2 = fmin(f2, r ? m[k] : INFINITY);
                f3 = fmax(f3, r ? m[k] : 0.0);
            }
            unsigned long long b0 = dbits(f0), b1 = dbits(f1), b2_ = dbits(f2), b3 = dbits(f3);
            b0 = wmin64(b0);
            b1 = wmax64(b1);
            b2_ = wmin64(b2_);
            b3 = wmax64(b3);
            // every warp pushes its partial straight to every CTA of the cluster (no block-level
            // reduction first): C x NW slots of 32 B, one mbarrier
            if (CL) {
                if (lane < (int)C) {
                    const uint32_t dst = mapa(su32(mm + ((int)rank * NW + wid) * 4), lane);
                    const uint32_t mb = mapa(su32(&mbar[0]), lane);
                    st_async_v2(dst, b0, b1, mb);
                    st_async_v2(dst + 16, b2_, b3, mb);
                }
            } else {
                // cooperative: the CTA's warps combine first (one slot and one counter add per
                // CTA: 16x fewer global atomics on the group's counter)
                if (lane == 0) {
                    loc1[4 * wid] = b0; loc1[4 * wid + 1] = b1; loc1[4 * wid + 2] = b2_; loc1[4 * wid + 3] = b3;
                }
                __syncthreads();
                if (wid == 0) {
                    const unsigned long long c0 = wmin64(lane < NW ? loc1[4 * lane] : BITS_INF);
                    const unsigned long long c1 = wmax64(lane < NW ? loc1[4 * lane + 1] : 0ull);
                    const unsigned long long c2 = wmin64(lane < NW ? loc1[4 * lane + 2] : BITS_INF);
                    const unsigned long long c3 = wmax64(lane < NW ? loc1[4 * lane + 3] : 0ull);
#ifndef CX_SEL_COOP_COUNTER
                    unsigned long long* sl = p.x1g + (size_t)(2 * g + (round & 1)) * C * 4;
                    if (lane < 4) {
                        const unsigned long long v = lane == 0 ? c0 : lane == 1 ? c1 : lane == 2 ? c2 : c3;
                        st_word(sl + rank * 4 + lane, v | stamp_of(round));
                    }
                    poll_slots(sl, round, reinterpret_cast<unsigned long long*>(mm));
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&mbar[0]);  // mm is written: the other warps may read it
#else
                    if (lane == 0) {
                        unsigned long long* d = p.x1g + ((size_t)(2 * g + (round & 1)) * C + rank) * 4;
                        reinterpret_cast<ulonglong2*>(d)[0] = make_ulonglong2(c0, c1);
                        reinterpret_cast<ulonglong2*>(d)[1] = make_ulonglong2(c2, c3);
                    }
                    bump(0);
                    gather(0, round, C * 32u);
#endif
                }
            }
            XSTAMP(9);
            mbar_wait(&mbar[0], ph1);
            ph1 ^= 1u;
            XSTAMP(4);
            if (CL && tid == 0 && round + 1 < p.take) mbar_arrive_expect(&mbar[0], tx1);
            f0 = INFINITY; f1 = 0.0; f2 = INFINITY; f3 = 0.0;
            for (int e = lane; e < (int)C * (CL ? NW : 1); e += 32) {
                const double2 lo = reinterpret_cast<const double2*>(mm)[2 * e];
                const double2 hi = reinterpret_cast<const double2*>(mm)[2 * e + 1];
                f0 = fmin(f0, lo.x);
                f1 = fmax(f1, lo.y);
                f2 = fmin(f2, hi.x);
                f3 = fmax(f3, hi.y);
            }
            b0 = dbits(f0); b1 = dbits(f1); b2_ = dbits(f2); b3 = dbits(f3);
            // a warp with no remaining rows pushed (inf, 0, inf, 0): neutral
            amin = bitsd(wmin64(b0));
            amax = bitsd(wmax64(b1));
            cmin = bitsd(wmin64(b2_));
            cmax = bitsd(wmax64(b3));
        }

        // ======== H: hybrid argmax (synapse.cpp:247-260), per WARP ========
        // Every warp ranks its rows with the reciprocal form, fetches the coordinates of its
        // approximate best row right away (L2, overlapping the exact step), scores the rows
        // within GAP_WINDOW of its approximate maximum with the reference's exact divisions,
        // and takes its exact (score desc, row asc) argmax with shuffles.  X2 then carries
        // every warp's candidate to every CTA: no block-level barrier in H.
        XSTAMP(10);
        const bool a_span = amax > amin, c_span = cmax > cmin;
        const double ar = __dsub_rn(amax, amin), cr = __dsub_rn(cmax, cmin);
        const double iar = a_span ? __drcp_rn(ar) : 0.0, icr = c_span ? __drcp_rn(cr) : 0.0;
        double happ[RPT];
        unsigned long long hkey = 0ull;  // this lane's approximate best (bits; h >= 0)
        int kmax = -1;
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
            happ[k] = -1.0;
            if (!(remm >> k & 1u)) continue;
            const double na = __dmul_rn(__dsub_rn(a[k], amin), iar);
            const double nc = __dmul_rn(__dsub_rn(m[k], cmin), icr);
            happ[k] = __dadd_rn(__dmul_rn(lam, nc), __dmul_rn(one_m_lam, na));
            if (kmax < 0 || dbits(happ[k]) > hkey) { hkey = dbits(happ[k]); kmax = k; }
        }
        // the warp's approximate best -> its coordinates start loading (a prefetch: any row of
        // the approximate maximum will do)
        const unsigned long long wkey = wmax64(kmax >= 0 ? hkey : 0ull);
        const uint32_t atmax = __ballot_sync(0xffffffffu, kmax >= 0 && hkey == wkey);
        const int wl = atmax ? __ffs(atmax) - 1 : 0;
        const int spec_k = __shfl_sync(0xffffffffu, kmax, wl);
        const int spec_li = atmax ? (quad + (NW / 4) * spec_k) * TILE + 32 * sub + wl : -1;
        float4 spec4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (atmax && lane < D / 4)
            spec4 = __ldg(reinterpret_cast<const float4*>(gX + (int64_t)spec_li * p.rstride) + lane);
        const bool approx_ok = (!a_span || ar >= 1e-290) && (!c_span || cr >= 1e-290);
        const double cut = approx_ok ? bitsd(wkey) - GAP_WINDOW : -INFINITY;
        XSTAMP(11);
        // exact hybrid of the rows within the window; per lane: best (score desc, row asc)
        // and runner-up
        unsigned long long bkey = 0ull, rkey = 0ull;
        bool has_b = false, has_r = false;
        int brow = INT_MAX;
        float bnx = 0.f;
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
            if (!(remm >> k & 1u) || happ[k] < cut) continue;
            const double na = a_span ? __ddiv_rn(__dsub_rn(a[k], amin), ar) : 0.0;
            const double nc = c_span ? __ddiv_rn(__dsub_rn(m[k], cmin), cr) : 0.0;
            const unsigned long long hk = dbits(__dadd_rn(__dmul_rn(lam, nc), __dmul_rn(one_m_lam, na)));
            const int li = (quad + (NW / 4) * k) * TILE + 32 * sub + lane;
            if (!has_b || hk > bkey) {  // rows ascend with k: on a tie the earlier (lower) row stays
                if (has_b) { rkey = max(rkey, bkey); has_r = true; }
                bkey = hk; brow = li; bnx = nx[k]; has_b = true;
            } else {
                rkey = max(rkey, hk);
                has_r = true;
            }
        }
        XSTAMP(12);
        // the warp's exact winner: max score, then the lowest row among equal scores
        const unsigned long long wbest = wmax64(has_b ? bkey : 0ull);
        const bool cand_b = has_b && bkey == wbest;
        const int wrow = __reduce_min_sync(0xffffffffu, cand_b ? (unsigned)brow : 0xffffffffu);
        const bool any_b = __ballot_sync(0xffffffffu, has_b) != 0u;
        const bool is_w = cand_b && brow == wrow;
        const uint32_t wmask = __ballot_sync(0xffffffffu, is_w);
        const float wnx = __shfl_sync(0xffffffffu, bnx, wmask ? __ffs(wmask) - 1 : 0);
        // runner-up: other lanes' best and every lane's runner-up (a tie with the winner included)
        const bool has_r2 = has_r || (has_b && !is_w);
        const unsigned long long r2 = wmax64(has_r2 ? (is_w ? rkey : max(rkey, bkey)) : 0ull);
        const bool any_r = __ballot_sync(0xffffffffu, has_r2) != 0u;
        // the exact winner is almost always the approximate one: else load its row now
        if (any_b && wrow != spec_li && lane < D / 4)
            spec4 = __ldg(reinterpret_cast<const float4*>(gX + (int64_t)wrow * p.rstride) + lane);
        if (!any_b) spec4 = make_float4(0.f, 0.f, 0.f, 0.f);
        const double bsc = any_b ? bitsd(wbest) : -1.0;
        const double b2 = any_r ? bitsd(r2) : -1.0;
        const int brow_w = any_b ? wrow : INT_MAX;
        const float bnx_w = wnx;

        XSTAMP(5);
        // ======== X2: every warp's (score, row, |b|^2, runner-up, coordinates) -> every CTA ========
        {
            const int slot = (int)rank * NW + wid;
            const double sc = bsc;
            const long long rw = brow_w != INT_MAX ? r0 + brow_w : LLONG_MAX;
            if (CL) {
                for (int dst = 0; dst < (int)C; ++dst) {
                    const uint32_t mb = mapa(su32(&mbar[1]), dst);
                    if (lane == 0) {
                        const uint32_t hd = mapa(su32(hdr + slot), dst);
                        st_async_v2(hd, __double_as_longlong(sc), (uint64_t)rw, mb);
                        st_async_v2(hd + 16, __double_as_longlong((double)bnx_w), __double_as_longlong(b2), mb);
                    }
                    if (lane < D / 4) st_async_v4(mapa(su32(bc + slot * D + 4 * lane), dst), spec4, mb);
                }
            } else {
                // cooperative: the CTA's best candidate first (score desc, row asc; its runner-up
                // is the best of the other warps or the winning warp's own runner-up)
                if (lane == 0) {
                    Hdr h;
                    h.score = sc; h.row = rw; h.nb = (double)bnx_w; h.second = b2;
                    locH[wid] = h;
                }
                if (lane < D / 4) reinterpret_cast<float4*>(locC + wid * D)[lane] = spec4;
                __syncthreads();
                if (wid == 0) {
                    const bool has = lane < NW && locH[lane].score >= 0.0;
                    const unsigned long long sb = has ? dbits(locH[lane].score) : 0ull;
                    const unsigned long long best = wmax64(sb);
                    const bool cs = has && sb == best;
                    const unsigned rmin = __reduce_min_sync(0xffffffffu, cs ? (unsigned)locH[lane].row : 0xffffffffu);
                    const bool iw = cs && (unsigned)locH[lane].row == rmin;
                    const uint32_t wm = __ballot_sync(0xffffffffu, iw);
                    const bool any = __ballot_sync(0xffffffffu, has) != 0u;
                    const int wsl = wm ? __ffs(wm) - 1 : 0;
                    const bool hs = lane < NW && locH[lane].second >= 0.0;
                    const bool hr = hs || (has && !iw);
                    const unsigned long long rb =
                        hr ? (iw ? dbits(locH[lane].second)
                                 : max(has ? sb : 0ull, hs ? dbits(locH[lane].second) : 0ull))
                           : 0ull;
                    const unsigned long long r2b = wmax64(rb);
                    const bool any2 = __ballot_sync(0xffffffffu, hr) != 0u;
#ifndef CX_SEL_COOP_COUNTER
                    // header words: score / runner-up (>= 0, or SENT for -1), row, |b|^2; the
                    // coordinates are not exchanged: every CTA reads the C candidates' rows from
                    // the cloud itself (read-only, L2) once the headers are in
                    unsigned long long* sl = reinterpret_cast<unsigned long long*>(p.x2h + (size_t)(2 * g + (round & 1)) * C);
                    if (lane < 4) {
                        const double hs = any ? locH[wsl].score : -1.0;
                        const double h2 = any2 ? bitsd(r2b) : -1.0;
                        unsigned long long v;
                        if (lane == 0) v = hs < 0.0 ? SENT : dbits(hs);
                        else if (lane == 1) v = (unsigned long long)(any ? locH[wsl].row : LLONG_MAX);
                        else if (lane == 2) v = dbits(locH[wsl].nb);
                        else v = h2 < 0.0 ? SENT : dbits(h2);
                        st_word(sl + rank * 4 + lane, v | stamp_of(round));
                    }
                    unsigned long long* hw = reinterpret_cast<unsigned long long*>(hdr);
                    poll_slots(sl, round, hw);
                    __syncwarp();
                    if (lane < (int)C) {  // decode the sentinels
                        if (hw[4 * lane] == SENT) hdr[lane].score = -1.0;
                        if (hw[4 * lane + 3] == SENT) hdr[lane].second = -1.0;
                    }
                    __syncwarp();
                    // the candidates' coordinates: this CTA's own from locC, the others' rows from
                    // the cloud (C x 16 float4, two per lane up to C = 4)
                    for (int e4 = lane; e4 < (int)C * (D / 4); e4 += 32) {
                        const int e = e4 / (D / 4), c4 = e4 % (D / 4);
                        const long long rw = hdr[e].row;
                        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                        if (e == (int)rank) v = reinterpret_cast<const float4*>(locC + wsl * D)[c4];
                        else if (rw != LLONG_MAX)
                            v = __ldg(reinterpret_cast<const float4*>(p.X + g * p.gstride + rw * p.rstride) + c4);
                        reinterpret_cast<float4*>(bc + e * D)[c4] = v;
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&mbar[1]);
#else
                    const size_t base = (size_t)(2 * g + (round & 1)) * C + rank;
                    if (lane == 0) {
                        Hdr h;
                        h.score = any ? locH[wsl].score : -1.0;
                        h.row = any ? locH[wsl].row : LLONG_MAX;
                        h.nb = locH[wsl].nb;
                        h.second = any2 ? bitsd(r2b) : -1.0;
                        p.x2h[base] = h;
                    }
                    if (lane < D / 4)
                        reinterpret_cast<float4*>(p.x2c + base * D)[lane] = reinterpret_cast<const float4*>(locC + wsl * D)[lane];
                    bump(1);
                    gather(1, round, C * (uint32_t)(sizeof(Hdr) + D * sizeof(float)));
#endif
                }
            }
        }
        mbar_wait(&mbar[1], ph2);
        ph2 ^= 1u;
        XSTAMP(6);
        if (CL && tid == 0 && round + 1 < p.take) mbar_arrive_expect(&mbar[1], tx2);
        // the cluster winner (score desc, row asc) over all C x NW candidates, and the runner-up
        double bs, rs2;
        long long br;
        int w;
        {
            unsigned long long ls = 0ull, l2 = 0ull;  // lane: best score bits, runner-up bits
            bool lb = false, lr = false;
            long long lrow = LLONG_MAX;
            int le = 0;
            for (int e = lane; e < (int)C * (CL ? NW : 1); e += 32) {
                const double es = hdr[e].score, e2 = hdr[e].second;
                const long long er = hdr[e].row;
                if (e2 >= 0.0) { l2 = max(l2, dbits(e2)); lr = true; }
                if (es < 0.0) continue;  // a warp without rows
                const unsigned long long eb = dbits(es);
                if (!lb || eb > ls || (eb == ls && er < lrow)) {
                    if (lb) { l2 = max(l2, ls); lr = true; }
                    ls = eb; lrow = er; le = e; lb = true;
                } else {
                    l2 = max(l2, eb);
                    lr = true;
                }
            }
            const unsigned long long gs = wmax64(lb ? ls : 0ull);
            const bool cs = lb && ls == gs;
            // rows are < 2^31 here (a group's rows): the low word orders them
            const unsigned grow = __reduce_min_sync(0xffffffffu, cs ? (unsigned)lrow : 0xffffffffu);
            const bool iw = cs && (unsigned)lrow == grow;
            const uint32_t wm = __ballot_sync(0xffffffffu, iw);
            const int wlane = wm ? __ffs(wm) - 1 : 0;
            const bool hr = lr || (lb && !iw);
            const unsigned long long g2 = wmax64(hr ? (iw ? l2 : max(l2, ls)) : 0ull);
            const bool any = __ballot_sync(0xffffffffu, lb) != 0u;
            const bool any2 = __ballot_sync(0xffffffffu, hr) != 0u;
            bs = any ? bitsd(gs) : -1.0;
            br = any ? (long long)grow : LLONG_MAX;
            w = __shfl_sync(0xffffffffu, le, wlane);
            rs2 = any2 ? bitsd(g2) : -1.0;
        }
        // gap monitor: a row outside every warp's window scores < bs - GAP_WINDOW (+ ~1e-15)
        if (tid == 0 && rank == 0 && rs2 >= 0.0)
            *min_gap = (unsigned long long)__double_as_longlong(
                dmin_std(__longlong_as_double((long long)*min_gap), __dsub_rn(bs, rs2)));
        bw = bc + w * D;
        nbw = (float)hdr[w].nb;
        if (br >= r0 && br < r0 + nrows) {
            const int li = (int)(br - r0);
            const int j = li / TILE, r = li % TILE;
            if (wid == ((j % (NW / 4)) << 2) + (r >> 5) && lane == (r & 31)) remm &= ~(1u << (j / (NW / 4)));
        }
        if (tid == 0 && rank == 0) {
            pick_rows[round] = br;
            pick_scores[round] = bs;
        }
        // every warp has read this round's hdr / bc before any CTA can push the next round's
        // (a peer pushes only after ITS X1 wait, which needs this CTA's next X1 push)
    }

    __syncthreads();
    if (rank == 0 && tid == 0 && p.gaps) p.gaps[g] = dmin_std(__longlong_as_double((long long)*min_gap), GAP_WINDOW);
    if (rank == 0) {  // sort the picks ascending by row (synapse.cpp:276-277)
        int64_t* out_rows = p.out_rows + (int64_t)g * p.take;
        double* out_scores = p.out_scores + (int64_t)g * p.take;
        for (int s = tid; s < p.take; s += NT) {
            const int64_t r = pick_rows[s];
            int pos = 0;
            for (int t = 0; t < p.take; ++t) pos += pick_rows[t] < r;
            out_rows[pos] = r;
            out_scores[pos] = pick_scores[s];
        }
        if (p.syn_k || p.syn_v) {  // the fused gather: one 16-B chunk per item, 4 loads in flight per thread
            __syncthreads();       // the sorted rows are in out_rows
            constexpr int CH = D / 4;
            const int per = p.take * CH, items = per * ((p.syn_k ? 1 : 0) + (p.syn_v ? 1 : 0));
            for (int i0 = tid; i0 < items; i0 += 4 * NT) {
                float4 v[4];
                float4* dst[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int it = i0 + u * NT;
                    dst[u] = nullptr;
                    if (it < items) {
                        const int kv = it / per, sc = (it % per) / CH, c = it % CH;
                        const bool isv = !p.syn_k || kv == 1;
                        const float* src = (isv ? p.V : p.X) + g * p.gstride + out_rows[sc] * p.rstride;
                        v[u] = __ldg(reinterpret_cast<const float4*>(src) + c);
                        dst[u] = reinterpret_cast<float4*>((isv ? p.syn_v : p.syn_k) + g * p.syn_gs + (int64_t)sc * D) + c;
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (dst[u]) *dst[u] = v[u];
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (CL) cg::this_cluster().sync();  // no CTA exits while a peer may still push into it
    else __syncthreads();
    if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
    // launched as a programmatic dependent (a split plan's cooperative part): complete only
    // after the cluster grid has (a no-op for a normally launched grid)
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

using SelxKern = void (*)(SelxParams);
template <bool CL>
SelxKern selx_kernel_for(int rpt) {
    switch (rpt) {
        case 1: return selx_kernel<1, CL>;
        case 2: return selx_kernel<2, CL>;
        case 3: return selx_kernel<3, CL>;
        case 4: return selx_kernel<4, CL>;
        case 5: return selx_kernel<5, CL>;
        default: return selx_kernel<6, CL>;
    }
}
SelxKern selx_kernel_for(int rpt, bool cl) { return cl ? selx_kernel_for<true>(rpt) : selx_kernel_for<false>(rpt); }

struct SelxCfg {
    int C = 0, S = 0, n_tiles = 0, n_smem = 0, rpt = 0, n_stage = 0;
    bool cluster = true;  // false: cooperative launch, exchanges through global memory
    int per_wave = 0;     // groups resident at once
    size_t smem = 0;
};

// rows per CTA s -> tiles, shared-memory tiles, TMEM tiles; false if s does not fit
bool selx_shape(int s, size_t budget, SelxCfg* c) {
    const int nt = (s + TILE - 1) / TILE;
    if (nt > MAXT) return false;
    const size_t base = selx_layout(0, c->C, 0).total;
    const int smem_max = (int)((budget - base) / TILE_BYTES);
    // rows in TMEM first (TS-form MMAs issue faster than SS, measured), the rest in shared memory
    const int nt_tm = std::min(nt, (512 - tm_rows_col(nt)) / 32);
    const int ns = nt - nt_tm;
    if (ns > smem_max) return false;
    c->S = s;
    c->n_tiles = nt;
    c->n_smem = ns;
    c->rpt = (nt + NW / 4 - 1) / (NW / 4);
    c->n_stage = 0;  // (TMA staging of the exact rows measured slower than direct loads)
    // at least ~116 KB so that one CTA owns an SM (and its 512 TMEM columns)
    c->smem = std::max(selx_layout(ns, c->C, c->n_stage).total, (size_t)116 * 1024);
    return true;
}

int sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    }
    return n;
}

// co-resident groups: clusters from the occupancy API; cooperative: blocks per SM x SMs / C
int selx_active(const SelxCfg& c) {
    static std::mutex mu;
    static std::map<std::tuple<int, int, size_t, bool>, int> cache;
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(c.C, c.rpt, c.smem, c.cluster);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    SelxKern kern = selx_kernel_for(c.rpt, c.cluster);
    int n = 0;
    try {
        kernel_smem(kern, c.smem, c.cluster && c.C > 8);
        if (c.cluster) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)c.C, 1, 1);
            cfg.blockDim = dim3(NT, 1, 1);
            cfg.dynamicSmemBytes = c.smem;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = (unsigned)c.C;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) n = 0;
        } else {
            int per_sm = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, c.smem) != cudaSuccess) per_sm = 0;
            n = per_sm * sm_count() / c.C;
        }
    } catch (const Failure&) {
        n = 0;
    }
    cudaGetLastError();
    cache[key] = n;
    return n;
}

}  // namespace

// Cost model (us per round, fitted below): a fixed part, a per-row part and a per-CTA part
// (exchange fan-in) for each exchange mode; times the waves = ceil(G / co-resident groups).
// The first model (fixed + per-row only) picked clusters of 16 for 6 groups -- cfg2 sharded
// over 8 GPUs -- at 2.02 ms where clusters of 6 take 1.32 ms.
//
// A SPLIT plan runs two launches side by side in one wave: as many groups as are
// co-resident as thread-block clusters (DSMEM exchanges), and the rest as a cooperative
// launch on the SMs the clusters leave free (CTAs anywhere, global-memory exchanges).
// cfg2 (48 groups of 8192 rows): a cluster of 3 CTAs holds a group on chip (22 tiles) and
// 45 clusters of 3 are co-resident (GPC granularity), leaving 13 SMs: the other 3 groups run
// as cooperative groups of 4 CTAs.  Measured per round: clusters of 3 17.5K cycles,
// cooperative 3 CTAs 21.6K (the single-wave alternative), cooperative 4 CTAs ~ the same as
// clusters of 3 (fewer rows per CTA offset the slower exchanges).
struct SelxPlan {
    SelxCfg a;           // groups [0, na): clusters (or the single plan)
    SelxCfg b;           // groups [na, G): cooperative, concurrently (split plans only)
    int na = 0;
    bool split = false;
};

static bool selx_plan(int G, int64_t L, const Options& o, SelxPlan* out) {
    static int max_optin = -1;
    if (max_optin < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
            max_optin = 232448;
    }
    const size_t budget = (size_t)max_optin - 1024;
    // us per round, fitted to B200 measurements (cfg2 rows, k = 164; tools/sel_sweep.sh):
    // clusters C = 4 / 5 / 6 / 8 / 12 / 16: 7.80 / 7.98 / 7.63 / 8.23 / 9.74 / 11.86 us, stamped
    // cooperative C = 4 / 6 / 8: 8.88 / 8.19 / 7.96 us -- a per-row part (the bound and ranking
    // passes) plus a per-CTA part (exchange fan-in), smaller for the cooperative exchanges
    auto per_round = [](const SelxCfg& c) {
        return c.cluster ? 1.50 + 0.00195 * c.S + 0.58 * c.C : 3.83 + 0.00195 * c.S + 0.27 * c.C;
    };
    // every (mode, C) that fits, with its co-residency
    std::vector<SelxCfg> cand;
    for (int mode = 0; mode < 2; ++mode) {
        const bool cl = mode == 0;
        for (int c = 1; c <= MAXC; ++c) {
            if (o.select_cluster > 0 && c != o.select_cluster && o.select_exchange != 3) continue;
            SelxCfg cfg;
            cfg.C = c;
            cfg.cluster = cl;
            if (!selx_shape((int)((L + c - 1) / c), budget, &cfg)) continue;
            cfg.per_wave = selx_active(cfg);
            if (cfg.per_wave > 0) cand.push_back(cfg);
        }
    }
    double best = 1e300;
    bool found = false;
    if (o.select_exchange != 3) {
        for (const SelxCfg& cfg : cand) {
            if (o.select_exchange == 1 && !cfg.cluster) continue;  // pinned: clusters
            if (o.select_exchange == 2 && cfg.cluster) continue;   // pinned: cooperative
            const double cost = (double)((G + cfg.per_wave - 1) / cfg.per_wave) * per_round(cfg);
            if (cost < best * (1.0 - 1e-9)) {
                best = cost;
                out->a = cfg;
                out->na = G;
                out->split = false;
                found = true;
            }
        }
    }
    // split plans: auto (no pinned exchange / cluster size) or pinned (select_exchange = 3)
    if (o.select_exchange == 3 || (o.select_exchange == 0 && o.select_cluster == 0)) {
        const int sms = sm_count();
        for (const SelxCfg& ca : cand) {
            // auto: only when the clusters alone would need a second wave; pinned (tests): any
            // G >= 2 splits, at most G - 1 groups as clusters
            if (!ca.cluster || G < 2 || (o.select_exchange != 3 && ca.per_wave >= G)) continue;
            if (o.select_exchange == 3 && o.select_cluster > 0 && ca.C != o.select_cluster) continue;
            const int na = std::min(ca.per_wave, G - 1), rest = G - na, free_sms = sms - na * ca.C;
            for (const SelxCfg& cb : cand) {
                if (cb.cluster || rest * cb.C > free_sms || cb.per_wave < rest) continue;
                const double cost = std::max(per_round(ca), per_round(cb));
                if (cost < best * (1.0 - 1e-9)) {
                    best = cost;
                    out->a = ca;
                    out->b = cb;
                    out->na = na;
                    out->split = true;
                    found = true;
                }
            }
        }
    }
    return found;
}

size_t select_tc_scratch(int G) {
    // cooperative-mode exchange buffers + counters, for any C <= 16
    return (size_t)G * 2 * MAXC * NW * (4 * sizeof(unsigned long long) + sizeof(Hdr) + D * sizeof(float)) +
           (size_t)G * 2 * sizeof(unsigned) + 1024;
}

bool select_tc_launch(const GroupView& g, const Options& o, const double* attn, const double* cen, int take,
                      double lambda, unsigned flags, int64_t* pick_rows, double* pick_scores, int64_t* rows,
                      double* scores, double* gaps, void* scratch, cudaStream_t s, const SynGather* gat,
                      bool* gathered) {
    if (gathered) *gathered = false;
    if (g.dim != D || (g.rstride & 3) != 0 || (g.gstride & 3) != 0 || (reinterpret_cast<uintptr_t>(g.X) & 15) != 0 ||
        g.L < 1)
        return false;
    SelxPlan plan;
    if (!selx_plan(g.G, g.L, o, &plan)) return false;
    SelxParams prm;
    prm.X = g.X;
    prm.gstride = g.gstride;
    prm.rstride = g.rstride;
    prm.L = g.L;
    prm.attn = attn;
    prm.cen = cen;
    prm.take = take;
    prm.lambda = lambda;
    prm.filter = (flags & CX_SELECT_EXACT_ONLY) ? 0 : 1;
    prm.pick_rows = pick_rows;
    prm.pick_scores = pick_scores;
    prm.out_rows = rows;
    prm.out_scores = scores;
    prm.gaps = gaps;
    prm.trace = nullptr;
    prm.x1g = nullptr;
    prm.x2h = nullptr;
    prm.x2c = nullptr;
    prm.cnt = nullptr;
    prm.V = nullptr;
    prm.syn_k = nullptr;
    prm.syn_v = nullptr;
    prm.syn_gs = 0;
    {  // the gather goes into the kernel when every access is a 16-B chunk
        auto a16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
        if (gat && (gat->syn_k || (gat->syn_v && gat->values)) && (gat->syn_gs & 3) == 0 &&
            (!gat->syn_k || a16(gat->syn_k)) && (!gat->syn_v || !gat->values || (a16(gat->syn_v) && a16(gat->values)))) {
            prm.syn_k = gat->syn_k;
            if (gat->syn_v && gat->values) {
                prm.V = gat->values;
                prm.syn_v = gat->syn_v;
            }
            prm.syn_gs = gat->syn_gs;
            if (gathered) *gathered = true;
        }
    }
#ifdef CX_EXPERIMENTS
    const char* tr = getenv("CX_SEL_TRACE");
    if (tr && tr[0] == '1') CX_CUDA(cudaMallocManaged(&prm.trace, sizeof(long long) * 16 * 4096));
#endif
    // cooperative exchange buffers + counters for ng groups of C CTAs, carved from scr
    auto coop_scratch = [](void* scr, int ng, int C, SelxParams* pw) {
        char* sc = reinterpret_cast<char*>(((uintptr_t)scr + 255) & ~(uintptr_t)255);
        const size_t slots = (size_t)ng * 2 * C * NW;
        pw->x1g = reinterpret_cast<unsigned long long*>(sc);
        sc += slots * 4 * sizeof(unsigned long long);
        pw->x2h = reinterpret_cast<Hdr*>(sc);
        sc += slots * sizeof(Hdr);
        pw->x2c = reinterpret_cast<float*>(sc);
        sc += slots * D * sizeof(float);
        pw->cnt = reinterpret_cast<unsigned*>(sc);
    };
    // per launch: the exchange counters (counter protocol) or the stamped slots (zero = no
    // round's stamp yet) of ng groups of C CTAs
    auto coop_clear = [](const SelxParams& pw, int ng, int C, cudaStream_t st) {
        CX_CUDA(cudaMemsetAsync(pw.cnt, 0, sizeof(unsigned) * 2 * ng, st));
        CX_CUDA(cudaMemsetAsync(pw.x1g, 0, sizeof(unsigned long long) * 4 * 2 * (size_t)ng * C, st));
        CX_CUDA(cudaMemsetAsync(pw.x2h, 0, sizeof(Hdr) * 2 * (size_t)ng * C, st));
    };
    // one part of the plan: groups [gb, ge) with configuration cfg on stream st
    auto launch_part = [&](const SelxCfg& cfg, int gb, int ge, cudaStream_t st, void* scr, bool dependent) {
        SelxParams pp = prm;
        pp.S = cfg.S;
        pp.n_tiles = cfg.n_tiles;
        pp.n_smem = cfg.n_smem;
        pp.n_stage = cfg.n_stage;
        pp.C = cfg.C;
        SelxKern kern = selx_kernel_for(cfg.rpt, cfg.cluster);
        kernel_smem(kern, cfg.smem, cfg.cluster && cfg.C > 8);
        // the groups in waves of per_wave (cooperative launches must fit on the GPU at once;
        // cluster launches are a single grid, the hardware forms the waves)
        const int wave = cfg.cluster ? ge - gb : cfg.per_wave;
        for (int g0 = gb; g0 < ge; g0 += wave) {
            const int ng = std::min(wave, ge - g0);
            SelxParams pw = pp;
            pw.X = g.X + (int64_t)g0 * g.gstride;
            pw.attn = attn + (int64_t)g0 * g.L;
            pw.cen = cen + (int64_t)g0 * D;
            pw.pick_rows = pick_rows + (int64_t)g0 * take;
            pw.pick_scores = pick_scores + (int64_t)g0 * take;
            pw.out_rows = rows + (int64_t)g0 * take;
            pw.out_scores = scores + (int64_t)g0 * take;
            pw.gaps = gaps ? gaps + g0 : nullptr;
            if (pw.V) pw.V += (int64_t)g0 * g.gstride;
            if (pw.syn_k) pw.syn_k += (int64_t)g0 * pw.syn_gs;
            if (pw.syn_v) pw.syn_v += (int64_t)g0 * pw.syn_gs;
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3((unsigned)cfg.C, (unsigned)ng, 1);
            lc.blockDim = dim3(NT, 1, 1);
            lc.dynamicSmemBytes = cfg.smem;
            lc.stream = st;
            cudaLaunchAttribute attr[2];
            if (cfg.cluster) {
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = (unsigned)cfg.C;
                attr[0].val.clusterDim.y = 1;
                attr[0].val.clusterDim.z = 1;
            } else {
                coop_scratch(scr, ng, cfg.C, &pw);
                // (a dependent part's counters were cleared before its primary: a memset
                // between the two launches would serialise them)
                if (!dependent) coop_clear(pw, ng, cfg.C, st);
                // a dependent part is a plain grid: a cooperative launch ignores programmatic
                // serialisation (measured: it ran after the cluster grid).  Its ng * C CTAs fit
                // in the SMs the clusters leave free; were one not resident, its group would
                // only wait for the cluster grid to retire (that grid never waits on them)
                attr[0].id = cudaLaunchAttributeCooperative;
                attr[0].val.cooperative = dependent ? 0 : 1;
            }
            int na = 1;
            if (dependent) {
                attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                attr[na].val.programmaticStreamSerializationAllowed = 1;
                ++na;
            }
            lc.attrs = attr;
            lc.numAttrs = na;
            CX_CUDA(cudaLaunchKernelEx(&lc, kern, pw));
            count_launch();
        }
    };
    if (!plan.split) {
        launch_part(plan.a, 0, g.G, s, scratch, false);
    } else {
        // both parts on s: the cooperative part is a programmatic dependent launch, released
        // once EVERY cluster CTA is resident (each executes griddepcontrol.launch_dependents
        // first), so the clusters take whole GPCs and the cooperative CTAs fill the SMs they
        // leave; it waits for the cluster grid (griddepcontrol.wait) before it exits, so the
        // next launch on s sees both parts complete
        SelxParams pb = prm;
        coop_scratch(scratch, g.G - plan.na, plan.b.C, &pb);
        coop_clear(pb, g.G - plan.na, plan.b.C, s);
        launch_part(plan.a, 0, plan.na, s, scratch, false);
        launch_part(plan.b, plan.na, g.G, s, scratch, true);
    }
#ifdef CX_EXPERIMENTS
    const SelxCfg& cfg = plan.a;  // (a split plan traces group 0 of both parts into one buffer)
    if (prm.trace) {  // average cycles per phase over rounds 2 .. take-2
        CX_CUDA(cudaStreamSynchronize(s));
        double acc[10] = {0}, hacc[3] = {0};
        int n = 0;
        for (int r = 2; r < std::min(take, 4096) - 1; ++r, ++n) {
            const long long* t = prm.trace + r * 16;
            acc[0] += (double)(t[1] - t[0]);  // B operand + MMA
            acc[1] += (double)(t[2] - t[1]);  // bound + queue + staging
            acc[2] += (double)(t[3] - t[2]);  // exact
            acc[3] += (double)(t[9] - t[3]);  // X1 local
            acc[4] += (double)(t[4] - t[9]);  // X1 wait
            acc[5] += (double)(t[5] - t[4]);  // H
            acc[6] += (double)(t[6] - t[5]);  // X2
            acc[7] += (double)(prm.trace[(r + 1) * 16] - t[0]);
            acc[8] += (double)t[8];
            acc[9] += (double)(t[10] - t[4]);   // H: X1 values -> min/max
            hacc[0] += (double)(t[11] - t[10]); // H: approximate ranking + winner-row prefetch issue
            hacc[1] += (double)(t[12] - t[11]); // H: exact window
            hacc[2] += (double)(t[5] - t[12]);  // H: warp winner / runner-up
        }
        if (n > 0)
            fprintf(stderr, "select_tc %s C=%d (co-resident %d) S=%d tiles=%d (smem %d) cycles/round: mma=%.0f bound+queue=%.0f exact=%.0f "
                            "X1loc=%.0f X1wait=%.0f H=%.0f X2=%.0f total=%.0f queued=%.1f\n",
                    cfg.cluster ? "cluster" : "cooperative", cfg.C, cfg.per_wave, cfg.S, cfg.n_tiles, cfg.n_smem, acc[0] / n, acc[1] / n, acc[2] / n, acc[3] / n, acc[4] / n,
                    acc[5] / n, acc[6] / n, acc[7] / n, acc[8] / n);
            fprintf(stderr, "  H split: minmax=%.0f rank=%.0f exact=%.0f winner=%.0f\n", acc[9] / n, hacc[0] / n,
                    hacc[1] / n, hacc[2] / n);
        cudaFree(prm.trace);
    }
#endif
    return true;
}

int select_tc_wave(int64_t L, int G) {
    SelxPlan plan;
    Options o;
    return selx_plan(G, L, o, &plan) ? (plan.split ? G : plan.a.per_wave) : 0;
}

}  // namespace cx

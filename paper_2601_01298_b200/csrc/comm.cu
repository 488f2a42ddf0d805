// comm.cu -- multi-GPU sharding of the hot path behind the C-ABI.
//
// Selection groups (layer, KV head) are independent: rank r of R owns the
// balanced contiguous block shard(G, r, R) and runs the whole greedy loop
// locally, with no collective while it runs.  The path's ONE exchange step
// follows: every rank packs its groups' synapse (rows, scores, landmark K, V)
// into fixed-size per-group records, pads its block to ceil(G / R) records,
// and a single ncclAllGather over NVLink / NVSwitch gives every GPU all G
// records, which one kernel unpacks into the [G][take] / [G][take][d] arrays
// the decode kernels read.  Accepted thoughts produced on a non-river GPU travel
// to the river GPU as one ncclSend / ncclRecv pair of the KvBlock
// (scheduler.cpp:139-156 drain_injections consumes them there).
//
// NCCL is loaded at first use with dlopen("libnccl.so.2"), so the library loads
// (and every single-GPU entry point works) on hosts without NCCL; in a process
// that already loaded NCCL (e.g. through torch) the same copy is reused.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <memory>

#include "cx_internal.cuh"

struct cx_comm {
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1, device = 0;
    char* buf = nullptr;  // [send block | receive buffer], grow-only
    size_t cap = 0;
};

namespace cx {
namespace {

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*getVersion)(int*) = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
    bool ok = false;
};

Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            n.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (n.h) break;
        }
        if (!n.h) return;
        auto sym = [](const char* s) { return dlsym(n.h, s); };
        n.getVersion = reinterpret_cast<decltype(n.getVersion)>(sym("ncclGetVersion"));
        n.getUniqueId = reinterpret_cast<decltype(n.getUniqueId)>(sym("ncclGetUniqueId"));
        n.commInitRank = reinterpret_cast<decltype(n.commInitRank)>(sym("ncclCommInitRank"));
        n.commInitAll = reinterpret_cast<decltype(n.commInitAll)>(sym("ncclCommInitAll"));
        n.commDestroy = reinterpret_cast<decltype(n.commDestroy)>(sym("ncclCommDestroy"));
        n.allGather = reinterpret_cast<decltype(n.allGather)>(sym("ncclAllGather"));
        n.send = reinterpret_cast<decltype(n.send)>(sym("ncclSend"));
        n.recv = reinterpret_cast<decltype(n.recv)>(sym("ncclRecv"));
        n.groupStart = reinterpret_cast<decltype(n.groupStart)>(sym("ncclGroupStart"));
        n.groupEnd = reinterpret_cast<decltype(n.groupEnd)>(sym("ncclGroupEnd"));
        n.errorString = reinterpret_cast<decltype(n.errorString)>(sym("ncclGetErrorString"));
        n.ok = n.getVersion && n.getUniqueId && n.commInitRank && n.commInitAll && n.commDestroy && n.allGather &&
               n.send && n.recv && n.groupStart && n.groupEnd && n.errorString;
    });
    if (!n.ok) fail(CX_DEVICE_ERROR, "NCCL (libnccl.so.2) could not be loaded");
    return n;
}

#define CX_NCCL(call)                                                                                  \
    do {                                                                                               \
        ncclResult_t cx_r_ = (call);                                                                   \
        if (cx_r_ != ncclSuccess) fail(CX_DEVICE_ERROR, std::string(#call) + ": " + nccl().errorString(cx_r_)); \
    } while (0)

// balanced contiguous block of n items for rank r of R (parallel.py shard_range)
__host__ __device__ inline void shard(int n, int r, int R, int* b, int* e) {
    const int base = n / R, extra = n % R;
    *b = r * base + (r < extra ? r : extra);
    *e = *b + base + (r < extra ? 1 : 0);
}

// per-group record: rows int64[take] | scores f64[take] | keys f32[take][dim] | values f32[take][dim]
__host__ __device__ inline size_t record_bytes(int take, int dim) {
    const size_t b = (size_t)take * 16 + (size_t)take * dim * 8;
    return (b + 255) & ~(size_t)255;
}

// pack groups [g0, g0 + n) of the [G] arrays into n consecutive records (16-byte units)
__global__ void synapse_pack_kernel(const int64_t* rows, const double* scores, const float* sk, const float* sv,
                                    int g0, int take, int dim, size_t rec, unsigned char* dst) {
    const int gi = blockIdx.y, g = g0 + gi;
    const size_t nrow = (size_t)take * 2, nkv = (size_t)take * dim / 4;  // 8-byte and 16-byte units
    unsigned char* r = dst + (size_t)gi * rec;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nrow + 2 * nkv; i += (size_t)gridDim.x * blockDim.x) {
        if (i < (size_t)take)
            reinterpret_cast<int64_t*>(r)[i] = rows[(size_t)g * take + i];
        else if (i < nrow)
            reinterpret_cast<double*>(r)[i] = scores[(size_t)g * take + (i - take)];
        else {
            const size_t j = i - nrow;
            const float4* src = reinterpret_cast<const float4*>(j < nkv ? sk : sv) + (size_t)g * nkv + (j < nkv ? j : j - nkv);
            reinterpret_cast<float4*>(r + nrow * 8)[j] = *src;
        }
    }
}

// records of all R padded blocks -> the [G] arrays (group g = record (r, g - begin(r)))
__global__ void synapse_unpack_kernel(const unsigned char* src, int G, int R, int per_rank, int take, int dim,
                                      size_t rec, int64_t* rows, double* scores, float* sk, float* sv) {
    const int g = blockIdx.y;
    int r = 0, b = 0, e = 0;
    for (; r < R; ++r) {
        shard(G, r, R, &b, &e);
        if (g < e) break;
    }
    const unsigned char* s = src + ((size_t)r * per_rank + (g - b)) * rec;
    const size_t nrow = (size_t)take * 2, nkv = (size_t)take * dim / 4;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nrow + 2 * nkv; i += (size_t)gridDim.x * blockDim.x) {
        if (i < (size_t)take)
            rows[(size_t)g * take + i] = reinterpret_cast<const int64_t*>(s)[i];
        else if (i < nrow)
            scores[(size_t)g * take + (i - take)] = reinterpret_cast<const double*>(s)[i];
        else {
            const size_t j = i - nrow;
            float4* dst = reinterpret_cast<float4*>(j < nkv ? sk : sv) + (size_t)g * nkv + (j < nkv ? j : j - nkv);
            *dst = reinterpret_cast<const float4*>(s + nrow * 8)[j];
        }
    }
}

void pack(const int64_t* rows, const double* scores, const float* sk, const float* sv, int g0, int n, int take,
          int dim, unsigned char* dst, cudaStream_t s) {
    if (n <= 0) return;
    synapse_pack_kernel<<<dim3(4, (unsigned)n), 256, 0, s>>>(rows, scores, sk, sv, g0, take, dim,
                                                              record_bytes(take, dim), dst);
    check_launch("synapse_pack_kernel");
}

void unpack(const unsigned char* src, int G, int R, int take, int dim, int64_t* rows, double* scores, float* sk,
            float* sv, cudaStream_t s) {
    if (G <= 0) return;
    synapse_unpack_kernel<<<dim3(4, (unsigned)G), 256, 0, s>>>(src, G, R, (G + R - 1) / R, take, dim,
                                                                record_bytes(take, dim), rows, scores, sk, sv);
    check_launch("synapse_unpack_kernel");
}

void check_dim(int dim) {
    if (dim < 4 || dim % 4 != 0) fail(CX_PRECONDITION_ERROR, "synapse records need dim % 4 == 0");
}

}  // namespace
}  // namespace cx

using namespace cx;

extern "C" int cx_nccl_version(void) {
    int v = 0;
    try {
        if (nccl().getVersion(&v) != ncclSuccess) v = 0;
    } catch (...) {
        v = 0;
    }
    return v;
}

extern "C" cx_status cx_comm_unique_id(void* id) {
    return guard(__func__, [&] {
        if (!id) fail(CX_INVALID_ARGUMENT, "null id");
        ncclUniqueId u;
        CX_NCCL(nccl().getUniqueId(&u));
        memcpy(id, &u, sizeof(u));
    });
}

extern "C" cx_status cx_comm_init_rank(int nranks, const void* id, int rank, int device, cx_comm** out) {
    return guard(__func__, [&] {
        if (!id || !out) fail(CX_INVALID_ARGUMENT, "null id/out");
        if (nranks < 1 || rank < 0 || rank >= nranks) fail(CX_INVALID_ARGUMENT, "bad rank / nranks");
        ncclUniqueId u;
        memcpy(&u, id, sizeof(u));
        CX_CUDA(cudaSetDevice(device));
        auto c = std::make_unique<cx_comm>();
        CX_NCCL(nccl().commInitRank(&c->comm, nranks, u, rank));
        c->rank = rank;
        c->nranks = nranks;
        c->device = device;
        *out = c.release();
    });
}

extern "C" cx_status cx_comm_init_all(int ndev, const int* devices, cx_comm** out) {
    return guard(__func__, [&] {
        if (ndev < 1 || !devices || !out) fail(CX_INVALID_ARGUMENT, "bad device list");
        std::vector<ncclComm_t> comms((size_t)ndev);
        CX_NCCL(nccl().commInitAll(comms.data(), ndev, devices));
        for (int i = 0; i < ndev; ++i) {
            auto* c = new cx_comm();
            c->comm = comms[(size_t)i];
            c->rank = i;
            c->nranks = ndev;
            c->device = devices[i];
            out[i] = c;
        }
    });
}

extern "C" cx_status cx_comm_destroy(cx_comm* c) {
    return guard(__func__, [&] {
        if (!c) return;
        if (c->buf) cudaFree(c->buf);
        if (c->comm) nccl().commDestroy(c->comm);
        delete c;
    });
}

extern "C" cx_status cx_comm_info(const cx_comm* c, int* rank, int* nranks, int* device) {
    return guard(__func__, [&] {
        if (!c) fail(CX_INVALID_ARGUMENT, "null comm");
        if (rank) *rank = c->rank;
        if (nranks) *nranks = c->nranks;
        if (device) *device = c->device;
    });
}

extern "C" cx_status cx_comm_group_start(void) { return guard(__func__, [&] { CX_NCCL(nccl().groupStart()); }); }
extern "C" cx_status cx_comm_group_end(void) { return guard(__func__, [&] { CX_NCCL(nccl().groupEnd()); }); }

extern "C" size_t cx_synapse_record_bytes(int take, int dim) { return record_bytes(take, dim); }

extern "C" cx_status cx_synapse_pack_dev(const int64_t* rows, const double* scores, const float* syn_keys,
                                         const float* syn_values, int g_begin, int n_groups, int take, int dim,
                                         void* dst, void* stream) {
    return guard(__func__, [&] {
        if (n_groups < 0 || take < 0 || g_begin < 0) fail(CX_INVALID_ARGUMENT, "negative size");
        if (n_groups == 0 || take == 0) return;
        check_dim(dim);
        if (!rows || !scores || !syn_keys || !syn_values || !dst) fail(CX_INVALID_ARGUMENT, "null pointer");
        pack(rows, scores, syn_keys, syn_values, g_begin, n_groups, take, dim, (unsigned char*)dst, (cudaStream_t)stream);
    });
}

extern "C" cx_status cx_synapse_unpack_dev(const void* src, int n_groups, int nranks, int take, int dim,
                                           int64_t* rows, double* scores, float* syn_keys, float* syn_values,
                                           void* stream) {
    return guard(__func__, [&] {
        if (n_groups < 0 || take < 0 || nranks < 1) fail(CX_INVALID_ARGUMENT, "bad size");
        if (n_groups == 0 || take == 0) return;
        check_dim(dim);
        if (!src || !rows || !scores || !syn_keys || !syn_values) fail(CX_INVALID_ARGUMENT, "null pointer");
        unpack((const unsigned char*)src, n_groups, nranks, take, dim, rows, scores, syn_keys, syn_values,
               (cudaStream_t)stream);
    });
}

// Host twins of pack / unpack (same record layout; for host-buffer outputs such as
// cx_compress_grouped_host's, exchanged over a host transport).
extern "C" cx_status cx_synapse_pack_host(const int64_t* rows, const double* scores, const float* syn_keys,
                                          const float* syn_values, int g_begin, int n_groups, int take, int dim,
                                          void* dst) {
    return guard(__func__, [&] {
        if (n_groups < 0 || take < 0 || g_begin < 0) fail(CX_INVALID_ARGUMENT, "negative size");
        if (n_groups == 0 || take == 0) return;
        check_dim(dim);
        if (!rows || !scores || !syn_keys || !syn_values || !dst) fail(CX_INVALID_ARGUMENT, "null pointer");
        const size_t rec = record_bytes(take, dim), kv = (size_t)take * dim;
        for (int gi = 0; gi < n_groups; ++gi) {
            const size_t g = (size_t)g_begin + gi;
            unsigned char* r = (unsigned char*)dst + (size_t)gi * rec;
            memcpy(r, rows + g * take, sizeof(int64_t) * take);
            memcpy(r + 8 * (size_t)take, scores + g * take, sizeof(double) * take);
            memcpy(r + 16 * (size_t)take, syn_keys + g * kv, sizeof(float) * kv);
            memcpy(r + 16 * (size_t)take + 4 * kv, syn_values + g * kv, sizeof(float) * kv);
            memset(r + 16 * (size_t)take + 8 * kv, 0, rec - (16 * (size_t)take + 8 * kv));
        }
    });
}

extern "C" cx_status cx_synapse_unpack_host(const void* src, int n_groups, int nranks, int take, int dim,
                                            int64_t* rows, double* scores, float* syn_keys, float* syn_values) {
    return guard(__func__, [&] {
        if (n_groups < 0 || take < 0 || nranks < 1) fail(CX_INVALID_ARGUMENT, "bad size");
        if (n_groups == 0 || take == 0) return;
        check_dim(dim);
        if (!src || !rows || !scores || !syn_keys || !syn_values) fail(CX_INVALID_ARGUMENT, "null pointer");
        const size_t rec = record_bytes(take, dim), kv = (size_t)take * dim;
        const int per = (n_groups + nranks - 1) / nranks;
        for (int r = 0; r < nranks; ++r) {
            int b = 0, e = 0;
            shard(n_groups, r, nranks, &b, &e);
            for (int g = b; g < e; ++g) {
                const unsigned char* p = (const unsigned char*)src + ((size_t)r * per + (g - b)) * rec;
                memcpy(rows + (size_t)g * take, p, sizeof(int64_t) * take);
                memcpy(scores + (size_t)g * take, p + 8 * (size_t)take, sizeof(double) * take);
                memcpy(syn_keys + (size_t)g * kv, p + 16 * (size_t)take, sizeof(float) * kv);
                memcpy(syn_values + (size_t)g * kv, p + 16 * (size_t)take + 4 * kv, sizeof(float) * kv);
            }
        }
    });
}

// The sharded compression: this rank's groups, then the one all-gather.
extern "C" cx_status cx_compress_sharded_dev(cx_ctx* ctx, cx_comm* comm, const cx_groups* local, const float* values,
                                             int n_groups_total, int k, double lambda, unsigned flags,
                                             int64_t* out_rows, double* out_scores, float* syn_keys,
                                             float* syn_values, void* stream) {
    return guard(__func__, [&] {
        if (k < 1) fail(CX_CONFIG_ERROR, "select_landmarks: k must be >= 1");
        if (lambda < 0.0 || lambda > 1.0) fail(CX_CONFIG_ERROR, "select_landmarks: lambda must be in [0,1]");
        if (!ctx || !comm || !local) fail(CX_INVALID_ARGUMENT, "null ctx/comm/groups");
        int b = 0, e = 0;
        shard(n_groups_total, comm->rank, comm->nranks, &b, &e);
        if (local->n_groups != e - b)
            fail(CX_PRECONDITION_ERROR, "compress_sharded: local groups != this rank's shard of n_groups_total");
        if (!out_rows || !out_scores || !syn_keys || !syn_values || !values)
            fail(CX_INVALID_ARGUMENT, "null outputs");
        check_dim(local->dim);
        const int take = (int)std::min<int64_t>(k, local->count);
        const int dim = local->dim;
        cudaStream_t s = (cudaStream_t)stream;
        // this rank's groups straight into their slots of the [G] outputs
        if (e > b) {
            const cx_status st = cx_compress_grouped_dev(ctx, local, values, k, lambda, flags, out_rows + (size_t)b * take,
                                                         out_scores + (size_t)b * take, syn_keys + (size_t)b * take * dim,
                                                         syn_values + (size_t)b * take * dim, stream);
            if (st != CX_OK) fail(st, cx_last_error());
        }
        // (one rank: the all-gather below is an identity copy, kept so every world size runs one path)
        const int per = (n_groups_total + comm->nranks - 1) / comm->nranks;
        const size_t rec = record_bytes(take, dim), blk = rec * per;
        const size_t need = blk * (1 + (size_t)comm->nranks);
        if (need > comm->cap) {
            if (comm->buf) {
                CX_CUDA(cudaStreamSynchronize(s));
                cudaFree(comm->buf);
            }
            comm->buf = nullptr;
            comm->cap = 0;
            CX_CUDA(cudaMalloc(&comm->buf, need));
            comm->cap = need;
        }
        unsigned char* send = reinterpret_cast<unsigned char*>(comm->buf);
        unsigned char* recv = send + blk;
        pack(out_rows, out_scores, syn_keys, syn_values, b, e - b, take, dim, send, s);
        CX_NCCL(nccl().allGather(send, recv, blk, ncclUint8, comm->comm, s));
        unpack(recv, n_groups_total, comm->nranks, take, dim, out_rows, out_scores, syn_keys, syn_values, s);
    });
}

// Accepted-thought transfer to the river GPU: a KvBlock
// [n_layers][T][d_model] keys + values as one ncclSend / ncclRecv pair.
extern "C" cx_status cx_thought_send_dev(cx_comm* comm, const float* keys, const float* values, int64_t token_count,
                                         int n_layers, int d_model, int river_rank, void* stream) {
    return guard(__func__, [&] {
        if (!comm || !keys || !values) fail(CX_INVALID_ARGUMENT, "null comm/block");
        if (token_count < 1) fail(CX_PRECONDITION_ERROR, "inject: empty block");
        if (river_rank < 0 || river_rank >= comm->nranks || river_rank == comm->rank)
            fail(CX_INVALID_ARGUMENT, "thought_send: bad river rank");
        const size_t n = (size_t)token_count * n_layers * d_model;
        CX_NCCL(nccl().groupStart());
        CX_NCCL(nccl().send(keys, n, ncclFloat32, river_rank, comm->comm, (cudaStream_t)stream));
        CX_NCCL(nccl().send(values, n, ncclFloat32, river_rank, comm->comm, (cudaStream_t)stream));
        CX_NCCL(nccl().groupEnd());
    });
}

extern "C" cx_status cx_thought_recv_dev(cx_comm* comm, float* keys, float* values, int64_t token_count, int n_layers,
                                         int d_model, int src_rank, void* stream) {
    return guard(__func__, [&] {
        if (!comm || !keys || !values) fail(CX_INVALID_ARGUMENT, "null comm/block");
        if (token_count < 1) fail(CX_PRECONDITION_ERROR, "inject: empty block");
        if (src_rank < 0 || src_rank >= comm->nranks || src_rank == comm->rank)
            fail(CX_INVALID_ARGUMENT, "thought_recv: bad source rank");
        const size_t n = (size_t)token_count * n_layers * d_model;
        CX_NCCL(nccl().groupStart());
        CX_NCCL(nccl().recv(keys, n, ncclFloat32, src_rank, comm->comm, (cudaStream_t)stream));
        CX_NCCL(nccl().recv(values, n, ncclFloat32, src_rank, comm->comm, (cudaStream_t)stream));
        CX_NCCL(nccl().groupEnd());
    });
}

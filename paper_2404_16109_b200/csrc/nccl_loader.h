// Multi-GPU plumbing: NCCL loaded at run time with dlopen("libnccl.so.2") so the
// library has no link-time NCCL dependency; when torch is imported first its bundled NCCL (2.28) is the
// one already mapped in the process and dlopen returns it.
//
// Collectives of one proof:
//   prepare: ncclAllReduce(u32, sum) of m (N entries) + ncclAllReduce(u64, min) of the error words, both on
//            the device (no host round trip);
//   prove:   ONE ncclAllGather of this rank's per-round sums {H0, H1, Hinf, a0, a1} for all local
//            rounds (Fr cannot be added by NCCL; the device sums the gathered rows mod r in k_derive),
//            ONE ncclAllGather of the rank's fully folded (A, S) for the last log2 P rounds, which every
//            rank then runs identically (replicated tail), + a device-side min of the error words.
//   Fiat-Shamir prove: one small ncclAllGather per local round (r_k depends on g_k, so each round's sums must be
//            global before r_k is derived), identically on every rank.
// The per-round sums are exchanged after the local rounds rather than between them: with the challenges
// passed in explicitly (north star) no local round depends on an earlier round's sums, so the P-way
// exchange of all rounds costs one collective.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <condition_variable>
#include <mutex>

#include <nccl.h>

namespace {

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    if (!api.h) {
        api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!api.h) return api;
        api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(api.h, "ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))dlsym(api.h, "ncclCommInitRank");
        api.CommDestroy = (decltype(api.CommDestroy))dlsym(api.h, "ncclCommDestroy");
        api.AllReduce = (decltype(api.AllReduce))dlsym(api.h, "ncclAllReduce");
        api.AllGather = (decltype(api.AllGather))dlsym(api.h, "ncclAllGather");
        api.GetErrorString = (decltype(api.GetErrorString))dlsym(api.h, "ncclGetErrorString");
    }
    return api;
}

int nccl_fail(zkl_ctx* ctx, ncclResult_t r, const char* what) {
    if (ctx) snprintf(ctx->last_error, sizeof(ctx->last_error), "%s: %s", what,
                      nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl");
    return ZKL_E_NCCL;
}

#define NCCL_TRY(ctx, call)                                    \
    do {                                                       \
        ncclResult_t r_ = (call);                              \
        if (r_ != ncclSuccess) return nccl_fail(ctx, r_, #call); \
    } while (0)

int zkl_nccl_get_unique_id(uint8_t id[128]) {
    NcclApi& a = nccl();
    if (!a.GetUniqueId) return ZKL_E_NCCL;
    ncclUniqueId u;
    if (a.GetUniqueId(&u) != ncclSuccess) return ZKL_E_NCCL;
    memcpy(id, u.internal, 128);
    return ZKL_OK;
}

int zkl_nccl_init(zkl_ctx* ctx, const uint8_t id[128], int rank, int nranks) {
    NcclApi& a = nccl();
    if (!a.CommInitRank) {
        snprintf(ctx->last_error, sizeof(ctx->last_error), "libnccl.so.2 not loadable: %s", dlerror());
        return ZKL_E_NCCL;
    }
    ncclUniqueId u;
    memcpy(u.internal, id, 128);
    ncclComm_t comm;
    NCCL_TRY(ctx, a.CommInitRank(&comm, nranks, u, rank));
    ctx->nccl_comm = comm;
    return ZKL_OK;
}

void zkl_nccl_destroy(zkl_ctx* ctx) {
    if (ctx->nccl_comm && nccl().CommDestroy) nccl().CommDestroy((ncclComm_t)ctx->nccl_comm);
    ctx->nccl_comm = nullptr;
}

// gathered (A, S) pairs (AoS fr, rank-major) -> SoA [A planes (8 x P)] [S planes (8 x P)]
__global__ void k_pairs_to_soa(const zkl::fr* __restrict__ g, int P, uint32_t* soa) {
    const int p = threadIdx.x;
    if (p >= P) return;
    for (int l = 0; l < 8; ++l) {
        soa[l * P + p] = g[2 * p].v[l];
        soa[8 * P + l * P + p] = g[2 * p + 1].v[l];
    }
}

// All-gather this rank's round sums (dl x 5 fr) into gath[P][dl][5] and the folded (A, S) into the
// SoA pair buffer gfin (2 x 8 x P words), via a scratch area right after gfin.
int nccl_exchange(zkl_ctx* ctx, int dl, const zkl::fr* rank_sums, zkl::fr* gath, const zkl::fr* fin,
                  zkl::fr* gfin) {
    NcclApi& a = nccl();
    ncclComm_t comm = (ncclComm_t)ctx->nccl_comm;
    const size_t words = (size_t)dl * zkl::kSlots * 8;
    if (dl > 0) NCCL_TRY(ctx, a.AllGather(rank_sums, gath, words, ncclUint32, comm, ctx->stream));
    // gather the 2 fr (16 words) per rank into the tail of gath (reserved: P x kMaxRounds x kSlots fr)
    zkl::fr* g2 = gath + (size_t)ctx->nranks * dl * zkl::kSlots;
    NCCL_TRY(ctx, a.AllGather(fin, g2, 16, ncclUint32, comm, ctx->stream));
    k_pairs_to_soa<<<1, 32, 0, ctx->stream>>>(g2, ctx->nranks, reinterpret_cast<uint32_t*>(gfin));
    ctx->launches++;
    return cudaGetLastError() == cudaSuccess ? ZKL_OK : ZKL_E_CUDA;
}

int nccl_allreduce_u32(zkl_ctx* ctx, uint32_t* buf, uint64_t n) {
    NCCL_TRY(ctx, nccl().AllReduce(buf, buf, n, ncclUint32, ncclSum, (ncclComm_t)ctx->nccl_comm, ctx->stream));
    return ZKL_OK;
}

// element-wise min over ranks of n device u64 words, in place on the ctx stream (error indices: no host round trip)
int nccl_allreduce_min_u64_dev(zkl_ctx* ctx, unsigned long long* d, int n) {
    NCCL_TRY(ctx, nccl().AllReduce(d, d, (size_t)n, ncclUint64, ncclMin, (ncclComm_t)ctx->nccl_comm, ctx->stream));
    return ZKL_OK;
}

// min over ranks of a host u64 (uses the pinned host page + a device word)
int nccl_min_u64(zkl_ctx* ctx, unsigned long long* v) {
    unsigned long long* d = reinterpret_cast<unsigned long long*>(ctx->dscratch + 16);
    unsigned long long* h = reinterpret_cast<unsigned long long*>((uint8_t*)ctx->host_out + 61000);
    *h = *v;
    cudaMemcpyAsync(d, h, sizeof(*d), cudaMemcpyHostToDevice, ctx->stream);
    NCCL_TRY(ctx, nccl().AllReduce(d, d, 1, ncclUint64, ncclMin, (ncclComm_t)ctx->nccl_comm, ctx->stream));
    cudaMemcpyAsync(h, d, sizeof(*d), cudaMemcpyDeviceToHost, ctx->stream);
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return ZKL_E_CUDA;
    *v = *h;
    return ZKL_OK;
}

// ---------------------------------------------------------------- loopback communicator
// P virtual ranks in one process (one host thread each, same device): a collective is a host barrier
// around device copies through a staging area owned by the group.  No kernel ever waits on another
// rank's kernel: every wait is a host-side barrier after a stream synchronization.  Used to run the
// P > 1 code path (partition, exchange, replicated rounds) bit-for-bit on one GPU.
int lb_barrier(zkl_group* g) {
    std::unique_lock<std::mutex> lk(g->mu);
    const uint64_t gen = g->generation;
    if (++g->arrived == g->nranks) {
        g->arrived = 0;
        ++g->generation;
        g->cv.notify_all();
    } else {
        g->cv.wait(lk, [&] { return g->generation != gen; });
    }
    return ZKL_OK;
}

// every rank contributes `bytes` at `src` (device); afterwards `dst` (device) holds all ranks' blocks, rank-major
int lb_allgather(zkl_ctx* ctx, const void* src, void* dst, size_t bytes) {
    zkl_group* g = ctx->group;
    if ((size_t)g->nranks * bytes > g->staging_bytes) return ZKL_E_OOM;
    if (cudaMemcpyAsync(g->staging + (size_t)ctx->rank * bytes, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream) !=
            cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
        return ZKL_E_CUDA;
    lb_barrier(g);
    if (cudaMemcpyAsync(dst, g->staging, (size_t)g->nranks * bytes, cudaMemcpyDeviceToDevice, ctx->stream) !=
            cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
        return ZKL_E_CUDA;
    lb_barrier(g);
    return ZKL_OK;
}

__global__ void k_sum_rows_u32(const uint32_t* __restrict__ rows, int nrows, uint64_t n, uint32_t* out) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t s = 0;
        for (int r = 0; r < nrows; ++r) s += rows[(uint64_t)r * n + j];
        out[j] = s;
    }
}

int lb_allreduce_u32(zkl_ctx* ctx, uint32_t* buf, uint64_t n) {
    zkl_group* g = ctx->group;
    const size_t bytes = n * sizeof(uint32_t);
    if ((size_t)g->nranks * bytes > g->staging_bytes) return ZKL_E_OOM;
    if (cudaMemcpyAsync(g->staging + (size_t)ctx->rank * bytes, buf, bytes, cudaMemcpyDeviceToDevice, ctx->stream) !=
            cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
        return ZKL_E_CUDA;
    lb_barrier(g);
    k_sum_rows_u32<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 1184), 256, 0, ctx->stream>>>(
        reinterpret_cast<const uint32_t*>(g->staging), g->nranks, n, buf);
    ctx->launches++;
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return ZKL_E_CUDA;
    lb_barrier(g);
    return ZKL_OK;
}

__global__ void k_min_rows_u64(const unsigned long long* __restrict__ rows, int nrows, int n, unsigned long long* out) {
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        unsigned long long v = ~0ull;
        for (int r = 0; r < nrows; ++r) v = rows[(size_t)r * n + j] < v ? rows[(size_t)r * n + j] : v;
        out[j] = v;
    }
}

int lb_allreduce_min_u64_dev(zkl_ctx* ctx, unsigned long long* d, int n) {
    zkl_group* g = ctx->group;
    const size_t bytes = (size_t)n * sizeof(unsigned long long);
    if ((size_t)g->nranks * bytes > g->staging_bytes) return ZKL_E_OOM;
    if (cudaMemcpyAsync(g->staging + (size_t)ctx->rank * bytes, d, bytes, cudaMemcpyDeviceToDevice, ctx->stream) !=
            cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
        return ZKL_E_CUDA;
    lb_barrier(g);
    k_min_rows_u64<<<1, 32, 0, ctx->stream>>>(reinterpret_cast<const unsigned long long*>(g->staging), g->nranks, n, d);
    ctx->launches++;
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return ZKL_E_CUDA;
    lb_barrier(g);
    return ZKL_OK;
}

int lb_min_u64(zkl_ctx* ctx, unsigned long long* v) {
    zkl_group* g = ctx->group;
    {
        std::lock_guard<std::mutex> lk(g->mu);
        if (g->min_arrived == 0) g->min_acc = ~0ull;
        g->min_acc = std::min(g->min_acc, *v);
        ++g->min_arrived;
    }
    lb_barrier(g);
    *v = g->min_acc;
    lb_barrier(g);
    {
        std::lock_guard<std::mutex> lk(g->mu);
        g->min_arrived = 0;
    }
    lb_barrier(g);
    return ZKL_OK;
}

int lb_exchange(zkl_ctx* ctx, int dl, const zkl::fr* rank_sums, zkl::fr* gath, const zkl::fr* fin, zkl::fr* gfin) {
    int st;
    if (dl > 0 && (st = lb_allgather(ctx, rank_sums, gath, (size_t)dl * zkl::kSlots * sizeof(zkl::fr)))) return st;
    zkl::fr* g2 = gath + (size_t)ctx->nranks * dl * zkl::kSlots;
    if ((st = lb_allgather(ctx, fin, g2, 2 * sizeof(zkl::fr)))) return st;
    k_pairs_to_soa<<<1, 32, 0, ctx->stream>>>(g2, ctx->nranks, reinterpret_cast<uint32_t*>(gfin));
    ctx->launches++;
    return cudaGetLastError() == cudaSuccess ? ZKL_OK : ZKL_E_CUDA;
}

// ---------------------------------------------------------------- dispatch
int zkl_dist_exchange(zkl_ctx* ctx, int dl, const zkl::fr* rank_sums, zkl::fr* gath, const zkl::fr* fin,
                      zkl::fr* gfin) {
    return ctx->group ? lb_exchange(ctx, dl, rank_sums, gath, fin, gfin) : nccl_exchange(ctx, dl, rank_sums, gath, fin, gfin);
}
int zkl_dist_allreduce_u32(zkl_ctx* ctx, uint32_t* buf, uint64_t n) {
    return ctx->group ? lb_allreduce_u32(ctx, buf, n) : nccl_allreduce_u32(ctx, buf, n);
}
// every rank's `bytes` (a multiple of 4) at src -> dst, rank-major, on the ctx stream
int zkl_dist_allgather(zkl_ctx* ctx, const void* src, void* dst, size_t bytes) {
    if (ctx->group) return lb_allgather(ctx, src, dst, bytes);
    NCCL_TRY(ctx, nccl().AllGather(src, dst, bytes / 4, ncclUint32, (ncclComm_t)ctx->nccl_comm, ctx->stream));
    return ZKL_OK;
}
int zkl_dist_min_u64_dev(zkl_ctx* ctx, unsigned long long* d, int n) {
    return ctx->group ? lb_allreduce_min_u64_dev(ctx, d, n) : nccl_allreduce_min_u64_dev(ctx, d, n);
}
int zkl_dist_min_u64(zkl_ctx* ctx, unsigned long long* v) {
    return ctx->group ? lb_min_u64(ctx, v) : nccl_min_u64(ctx, v);
}

}  // namespace

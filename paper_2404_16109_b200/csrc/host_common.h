// Host-side helpers shared by the library's translation units (api.cu: tlookup; mm_api.cu: matmul sumcheck;
// hx_api.cu: Hyrax).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <initializer_list>
#include <utility>

#include "common.cuh"

namespace zkl_host {
using namespace zkl;


constexpr int kSMs = 148;

inline int set_err(zkl_ctx* ctx, int st, const char* fmt, ...) {
    if (ctx) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(ctx->last_error, sizeof(ctx->last_error), fmt, ap);
        va_end(ap);
    }
    return st;
}

#define CUDA_TRY(ctx, call)                                                                         \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess) {                                                                    \
            if (e_ != cudaErrorInvalidValue && e_ != cudaErrorMemoryAllocation) (ctx)->poisoned = 1; \
            return set_err((ctx), ZKL_E_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_),       \
                           __FILE__, __LINE__);                                                     \
        }                                                                                           \
    } while (0)

// Every kernel launch goes through LAUNCH: counted, and (when profiling) bracketed by events on
// the launching stream.
#define LAUNCH(ctx, kern, grid, block, smem, stream, ...)                                           \
    do {                                                                                            \
        zkl_ctx::ProfRec* pr_ = prof_begin((ctx), #kern, (stream));                                 \
        kern<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                                   \
        (ctx)->launches++;                                                                          \
        if (pr_) cudaEventRecord(pr_->b, (stream));                                                 \
        CUDA_TRY(ctx, cudaGetLastError());                                                          \
    } while (0)

// A cooperative launch (all CTAs co-resident: the kernel synchronises its grid, csrc/coop.cuh), counted and profiled
// like LAUNCH.  One by-value argument struct.
#define LAUNCH_COOP(ctx, kern, grid, block, smem, stream, arg)                                      \
    do {                                                                                            \
        zkl_ctx::ProfRec* pr_ = prof_begin((ctx), #kern, (stream));                                 \
        void* args_[] = {(void*)&(arg)};                                                            \
        CUDA_TRY(ctx, cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(block), args_, (smem), (stream))); \
        (ctx)->launches++;                                                                          \
        if (pr_) cudaEventRecord(pr_->b, (stream));                                                 \
    } while (0)

inline zkl_ctx::ProfRec* prof_begin(zkl_ctx* ctx, const char* name, cudaStream_t st) {
    if (!ctx->profiling || ctx->nprof >= 256) return nullptr;
    zkl_ctx::ProfRec* r = &ctx->prof[ctx->nprof++];
    r->name = name;
    r->stream = st;
    cudaEventRecord(r->a, st);
    return r;
}

inline bool is_pow2(uint64_t x) { return x && !(x & (x - 1)); }
inline int ilog2(uint64_t x) { int k = 0; while ((1ull << k) < x) ++k; return k; }
inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }
inline size_t soa_bytes(uint64_t n) { return align_up(8 * 4 * std::max<uint64_t>(n, 4)); }

inline unsigned grid_for(uint64_t work, unsigned threads, unsigned cap) {
    uint64_t g = (work + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

inline unsigned grid_for(uint64_t work, unsigned threads) { return grid_for(work, threads, kSMs * 8); }

template <typename T>
inline T* at(zkl_ctx* ctx, size_t off) { return reinterpret_cast<T*>(ctx->ws + off); }

inline int check_ctx(zkl_ctx* ctx) {
    if (!ctx) return ZKL_E_ARG;
    if (ctx->poisoned) return set_err(ctx, ZKL_E_STATE, "context poisoned by an earlier CUDA fault");
    CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    return ZKL_OK;
}

inline int check_vec(zkl_ctx* ctx, const zkl_vec& v, uint64_t n, const char* name) {
    if (!v.limbs) return set_err(ctx, ZKL_E_ARG, "%s: null", name);
    if (v.n != n) return set_err(ctx, ZKL_E_SHAPE, "%s: length %llu, expected %llu", name,
                                 (unsigned long long)v.n, (unsigned long long)n);
    if (n >= 4 && ((n & 3) || ((uintptr_t)v.limbs & 15)))
        return set_err(ctx, ZKL_E_ARG, "%s: limbs must be 16-byte aligned and n a multiple of 4", name);
    return ZKL_OK;
}

// The pinned staging page (challenges of a synchronous call, alpha_f, error words at host_out + 60000/62000, matmul
// and Hyrax staging at 40000/45000) is shared by the synchronous entry points; an async prepare or prove reads its
// slots when it executes or completes (zkl_ctx_wait), so no other user of those slots may run in between.
inline int check_idle(zkl_ctx* ctx) {
    if (ctx->pend_prepare || ctx->pend_prove)
        return set_err(ctx, ZKL_E_STATE, "async work pending on this context: zkl_ctx_wait first");
    return ZKL_OK;
}

inline bool fr_ge_r_host(const zkl_fr& x) {
    static const uint32_t rl[8] = {0x00000001u, 0xffffffffu, 0xfffe5bfeu, 0x53bda402u,
                                   0x09a1d805u, 0x3339d808u, 0x299d7d48u, 0x73eda753u};
    for (int i = 7; i >= 0; --i)
        if (x.w[i] != rl[i]) return x.w[i] > rl[i];
    return true;
}

struct CopySeg {
    uint32_t* dst;
    const uint32_t* src;
    uint32_t words;
};
struct CopySegs {
    CopySeg seg[4];
    int n;
};
static __global__ void k_copy_from_host(CopySegs c) {
    for (int g = 0; g < c.n; ++g)
        for (uint32_t i = threadIdx.x; i < c.seg[g].words; i += blockDim.x) c.seg[g].dst[i] = c.seg[g].src[i];
}

inline int h2d_small(zkl_ctx* ctx, cudaStream_t s, std::initializer_list<std::pair<void*, const void*>> dsts,
              std::initializer_list<size_t> sizes) {
    CopySegs c;
    c.n = 0;
    auto sz = sizes.begin();
    for (const auto& d : dsts) {
        c.seg[c.n].dst = reinterpret_cast<uint32_t*>(d.first);
        c.seg[c.n].src = reinterpret_cast<const uint32_t*>(d.second);   // pinned (cudaMallocHost): UVA device-visible
        c.seg[c.n].words = (uint32_t)(*sz / 4);
        ++c.n;
        ++sz;
    }
    LAUNCH(ctx, k_copy_from_host, 1, 256, 0, s, c);
    return ZKL_OK;
}

inline int sync_stream(zkl_ctx* ctx) {
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) {
        ctx->poisoned = 1;
        return set_err(ctx, ZKL_E_CUDA, "asynchronous CUDA error: %s", cudaGetErrorString(e));
    }
    return ZKL_OK;
}

// ------------------------------------------------------------------ hierarchical batched inversion (a4)
// Forward passes: level 0 on `s0` (the caller's stream), the levels above and the one-block top on `s1`.
}  // namespace zkl_host

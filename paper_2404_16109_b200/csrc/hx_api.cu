// The zkl C ABI, Hyrax / Pedersen part (include/zkl.h): host orchestration.
#include <cuda_runtime.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "host_common.h"
#include "hyrax.cuh"

using namespace zkl;
using namespace zkl_host;

namespace {

struct HxPlan {
    uint64_t D, cols, rows, nslices;
    size_t o_sc, o_part, o_q, o_rho, o_out, o_v, o_er, o_ec, o_ypart, o_y, total;
};

void make_hx_plan(HxPlan& h, uint64_t D, uint64_t cols) {
    memset(&h, 0, sizeof(h));
    h.D = D; h.cols = cols; h.rows = D / cols;
    h.nslices = (cols + kHxSlice - 1) / kHxSlice;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o += align_up(bytes); return r; };
    h.o_sc = take(soa_bytes(D));
    h.o_part = take(sizeof(g1j) * h.rows * h.nslices * kHxGroups);
    h.o_q = take(sizeof(g1j) * h.rows * kHxGroups);
    h.o_rho = take(sizeof(zkl_fr) * h.rows);
    h.o_out = take(sizeof(zkl_g1) * h.rows);
    h.o_v = take(sizeof(fr) * 64);
    h.o_er = take(sizeof(fr) * h.rows);
    h.o_ec = take(sizeof(fr) * cols);
    h.o_ypart = take(sizeof(fr) * 256);
    h.o_y = take(sizeof(zkl_fr));
    h.total = o;
}

// pp = [generators G_0..G_{cols-1}, H (affine)] [their 16-entry tables, one per 32-bit scalar chunk g, of
// d 2^{32 g} G_i] [64 x 16 window table of H]
size_t hx_pp_bytes(uint64_t cols) {
    return align_up(sizeof(g1a) * (cols + 1)) + align_up(sizeof(g1a) * kHxGroups * (cols + 1) * kHxTab) +
           sizeof(g1a) * 64 * kHxTab;
}
const g1a* hx_htab(const void* pp, uint64_t cols) {
    return reinterpret_cast<const g1a*>((const uint8_t*)pp + align_up(sizeof(g1a) * (cols + 1)) +
                                        align_up(sizeof(g1a) * kHxGroups * (cols + 1) * kHxTab));
}

int hx_shape(zkl_ctx* ctx, uint64_t D, uint64_t cols) {
    if (!is_pow2(D) || !is_pow2(cols) || cols > D || cols > (1ull << 24))
        return set_err(ctx, ZKL_E_SHAPE, "Hyrax: D=%llu cols=%llu must be powers of two with cols <= D, 2^24",
                       (unsigned long long)D, (unsigned long long)cols);
    return ZKL_OK;
}

int run_hyrax_commit(zkl_ctx* ctx, const void* pp, uint64_t cols, zkl_vec S, uint64_t D, const zkl_fr* rho,
                     zkl_g1* C_host) {
    int st;
    if ((st = check_ctx(ctx))) return st;
    if ((st = check_idle(ctx))) return st;
    if (ctx->async_mode) return set_err(ctx, ZKL_E_STATE, "Hyrax: synchronous calls only");
    if (!pp || !C_host) return set_err(ctx, ZKL_E_ARG, "null argument");
    if ((st = hx_shape(ctx, D, cols))) return st;
    if ((st = check_vec(ctx, S, D, "S"))) return st;
    HxPlan h;
    make_hx_plan(h, D, cols);
    if (!ctx->ws || ctx->ws_bytes < h.total)
        return set_err(ctx, ZKL_E_OOM, "workspace %zu bytes < %zu required (zkl_hyrax_workspace_bytes)", ctx->ws_bytes,
                       h.total);
    ctx->prep_valid = 0;
    cudaStream_t s = ctx->stream;
    // pp = [generators (cols + 1, affine)] [their window tables]
    const g1a* tab = reinterpret_cast<const g1a*>((const uint8_t*)pp + align_up(sizeof(g1a) * (cols + 1)));
    uint32_t* Sc = at<uint32_t>(ctx, h.o_sc);
    g1j* part = at<g1j>(ctx, h.o_part);
    uint32_t* drho = nullptr;
    if (rho) {
        for (uint64_t j = 0; j < h.rows; ++j)
            if (fr_ge_r_host(rho[j])) return set_err(ctx, ZKL_E_NONCANONICAL, "rho_%llu is not canonical",
                                                     (unsigned long long)j);
        drho = at<uint32_t>(ctx, h.o_rho);
        CUDA_TRY(ctx, cudaMemcpyAsync(drho, rho, sizeof(zkl_fr) * h.rows, cudaMemcpyHostToDevice, s));
    }
    LAUNCH(ctx, k_hx_canon, grid_for(D, 256), 256, 0, s, S.limbs, D, Sc);
    const uint64_t nthreads = h.rows * h.nslices * kHxGroups;
    LAUNCH(ctx, k_hx_commit_partial, (unsigned)((nthreads + kHxThreads - 1) / kHxThreads), kHxThreads, 0, s, Sc, D,
           cols, tab, h.nslices, part);
    g1j* Q = at<g1j>(ctx, h.o_q);
    LAUNCH(ctx, k_hx_reduce_slices, (unsigned)(h.rows * kHxGroups), kHxRedThreads, 0, s, part, h.nslices, Q);
    zkl_g1* dout = at<zkl_g1>(ctx, h.o_out);
    LAUNCH(ctx, k_hx_commit_rows, (unsigned)((h.rows + 63) / 64), 64, 0, s, Q, h.rows, drho, hx_htab(pp, cols),
           dout);
    CUDA_TRY(ctx, cudaMemcpyAsync(C_host, dout, sizeof(zkl_g1) * h.rows, cudaMemcpyDeviceToHost, s));
    return sync_stream(ctx);
}

int run_hyrax_eval(zkl_ctx* ctx, zkl_vec S, uint64_t D, uint64_t cols, const zkl_fr* v, zkl_vec w_out,
                   zkl_fr* y_host) {
    int st;
    if ((st = check_ctx(ctx))) return st;
    if ((st = check_idle(ctx))) return st;
    if (ctx->async_mode) return set_err(ctx, ZKL_E_STATE, "Hyrax: synchronous calls only");
    if (!v || !y_host || !w_out.limbs) return set_err(ctx, ZKL_E_ARG, "null argument");
    if ((st = hx_shape(ctx, D, cols))) return st;
    if ((st = check_vec(ctx, S, D, "S")) || (st = check_vec(ctx, w_out, cols, "w_out"))) return st;
    HxPlan h;
    make_hx_plan(h, D, cols);
    if (!ctx->ws || ctx->ws_bytes < h.total)
        return set_err(ctx, ZKL_E_OOM, "workspace %zu bytes < %zu required (zkl_hyrax_workspace_bytes)", ctx->ws_bytes,
                       h.total);
    ctx->prep_valid = 0;
    const int d = ilog2(D), lr = ilog2(h.rows), lc = ilog2(cols);
    for (int i = 0; i < d; ++i)
        if (fr_ge_r_host(v[i])) return set_err(ctx, ZKL_E_NONCANONICAL, "v_%d is not canonical", i);
    cudaStream_t s = ctx->stream;
    zkl_fr* hs = reinterpret_cast<zkl_fr*>((uint8_t*)ctx->host_out + 40000);
    memcpy(hs, v, sizeof(zkl_fr) * d);
    zkl_fr* dstage = at<zkl_fr>(ctx, h.o_rho);
    fr* dv = at<fr>(ctx, h.o_v);
    if (d) {
        CUDA_TRY(ctx, cudaMemcpyAsync(dstage, hs, sizeof(zkl_fr) * d, cudaMemcpyHostToDevice, s));
        LAUNCH(ctx, k_hx_consts, 1, 64, 0, s, dstage, d, dv);
    }
    fr* Er = at<fr>(ctx, h.o_er);
    fr* Ec = at<fr>(ctx, h.o_ec);
    LAUNCH(ctx, k_hx_eq, grid_for(h.rows, 256), 256, 0, s, dv, lr, h.rows, Er);
    LAUNCH(ctx, k_hx_eq, grid_for(cols, 256), 256, 0, s, dv + lr, lc, cols, Ec);
    LAUNCH(ctx, k_hx_eval_w, (unsigned)((cols + 127) / 128), 128, 0, s, S.limbs, D, cols, Er, w_out.limbs);
    const unsigned nb = grid_for(cols, 256, 256);
    LAUNCH(ctx, k_hx_eval_y, nb, 256, 0, s, w_out.limbs, cols, Ec, at<fr>(ctx, h.o_ypart));
    zkl_fr* dy = at<zkl_fr>(ctx, h.o_y);
    LAUNCH(ctx, k_hx_eval_y_final, 1, 256, 0, s, at<fr>(ctx, h.o_ypart), (int)nb, dy);
    zkl_fr* hy = reinterpret_cast<zkl_fr*>((uint8_t*)ctx->host_out + 45000);
    CUDA_TRY(ctx, cudaMemcpyAsync(hy, dy, sizeof(zkl_fr), cudaMemcpyDeviceToHost, s));
    if ((st = sync_stream(ctx))) return st;
    *y_host = *hy;
    return ZKL_OK;
}

}  // namespace

extern "C" {

size_t zkl_hyrax_pp_bytes(uint64_t cols) { return is_pow2(cols) ? hx_pp_bytes(cols) : 0; }

int zkl_hyrax_setup(zkl_ctx* ctx, uint64_t cols, void* pp, size_t pp_bytes) {
    int st;
    if ((st = check_ctx(ctx))) return st;
    if (!pp) return set_err(ctx, ZKL_E_ARG, "null argument");
    if (!is_pow2(cols) || cols > (1ull << 24)) return set_err(ctx, ZKL_E_SHAPE, "cols must be a power of two <= 2^24");
    if (pp_bytes < hx_pp_bytes(cols)) return set_err(ctx, ZKL_E_OOM, "pp %zu bytes < %zu", pp_bytes, hx_pp_bytes(cols));
    cudaStream_t s = ctx->stream;
    g1a* gens = reinterpret_cast<g1a*>(pp);
    g1a* tab = reinterpret_cast<g1a*>((uint8_t*)pp + align_up(sizeof(g1a) * (cols + 1)));
    LAUNCH(ctx, k_hx_gens, (unsigned)((cols + 1 + 63) / 64), 64, 0, s, cols, gens);
    LAUNCH(ctx, k_hx_tables, (unsigned)((kHxGroups * (cols + 1) * kHxTab + 127) / 128), 128, 0, s, gens, cols + 1,
           tab);
    LAUNCH(ctx, k_hx_htables, (64 * kHxTab + 127) / 128, 128, 0, s, gens + cols, const_cast<g1a*>(hx_htab(pp, cols)));
    return sync_stream(ctx);
}

int zkl_hyrax_export_generators(zkl_ctx* ctx, const void* pp, uint64_t cols, zkl_g1* out_host) {
    int st;
    if ((st = check_ctx(ctx))) return st;
    if (!pp || !out_host) return set_err(ctx, ZKL_E_ARG, "null argument");
    if (!is_pow2(cols)) return set_err(ctx, ZKL_E_SHAPE, "cols must be a power of two");
    zkl_g1* d = nullptr;
    CUDA_TRY(ctx, cudaMallocAsync((void**)&d, sizeof(zkl_g1) * (cols + 1), ctx->stream));
    LAUNCH(ctx, k_hx_export, (unsigned)((cols + 1 + 127) / 128), 128, 0, ctx->stream, (const g1a*)pp, cols + 1, d);
    CUDA_TRY(ctx, cudaMemcpyAsync(out_host, d, sizeof(zkl_g1) * (cols + 1), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaFreeAsync(d, ctx->stream));
    return sync_stream(ctx);
}

size_t zkl_hyrax_workspace_bytes(uint64_t D, uint64_t cols) {
    if (!is_pow2(D) || !is_pow2(cols) || cols > D) return 0;
    HxPlan h;
    make_hx_plan(h, D, cols);
    return h.total;
}

int zkl_hyrax_commit(zkl_ctx* ctx, const void* pp, uint64_t cols, zkl_vec S, uint64_t D, const zkl_fr* rho,
                     zkl_g1* C_host) {
    return run_hyrax_commit(ctx, pp, cols, S, D, rho, C_host);
}

int zkl_hyrax_prove_eval(zkl_ctx* ctx, zkl_vec S, uint64_t D, uint64_t cols, const zkl_fr* v, zkl_vec w_out,
                         zkl_fr* y_host) {
    return run_hyrax_eval(ctx, S, D, cols, v, w_out, y_host);
}
}  // extern "C"

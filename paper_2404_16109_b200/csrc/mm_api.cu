// The zkl C ABI, matmul sumcheck part (include/zkl.h): host orchestration.
#include <cuda_runtime.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "host_common.h"
#include "matmul.cuh"

using namespace zkl;
using namespace zkl_host;

namespace {

struct MMPlan {
    uint64_t m, n, p;
    int lm, L, lp;
    int kc, nr;              // chunked rounds kc .. kc+nr-1 (0 = none)
    uint64_t chunk, nchunks; // chunk elements, number of chunks (= elements left for the tail)
    uint32_t gridA[kMaxRounds];   // multi-block rounds 1 .. kc-1: blocks per round
    MMRound rd[kMaxRounds];
    uint64_t parts;          // total partial rows (fr)
    uint64_t rowchunks;      // row chunks of the a-restriction
    size_t o_ch, o_eu, o_ev, o_rpart, o_a, o_b, o_f1a, o_f1b, o_f2a, o_f2b, o_ca, o_cb, o_parts, o_rd, o_fin, o_out,
        total;
};

void make_mm_plan(MMPlan& q, uint64_t m, uint64_t n, uint64_t p) {
    memset(&q, 0, sizeof(q));
    q.m = m; q.n = n; q.p = p;
    q.lm = ilog2(m); q.L = ilog2(n); q.lp = ilog2(p);
    uint64_t rows = 0;
    int k = 1;
    uint64_t len = n;
    for (; k <= q.L && len > kMMChunkMaxElems; ++k, len /= 2) {
        q.gridA[k - 1] = grid_for(len / 2, kMMThreads, kMaxBlocks);
        q.rd[k - 1] = MMRound{3 * rows, q.gridA[k - 1]};
        rows += q.gridA[k - 1];
    }
    if (k <= q.L) {
        q.kc = k;
        q.chunk = std::min<uint64_t>(kMMChunk, len);
        q.nr = ilog2(q.chunk);
        q.nchunks = len / q.chunk;
        for (int j = 0; j < q.nr; ++j) {
            q.rd[k + j - 1] = MMRound{3 * rows, (uint32_t)(q.nchunks * kMMChunkWarps)};
            rows += q.nchunks * kMMChunkWarps;
        }
        for (int kk = k + q.nr; kk <= q.L; ++kk) {
            q.rd[kk - 1] = MMRound{3 * rows, 1};
            rows += 1;
        }
    }
    q.parts = 3 * std::max<uint64_t>(rows, 1);
    q.rowchunks = (m + kMMRowChunk - 1) / kMMRowChunk;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o += align_up(bytes); return r; };
    q.o_ch = take(sizeof(fr) * (q.lm + q.lp + q.L + 1));
    q.o_eu = take(sizeof(fr) * m);
    q.o_ev = take(sizeof(fr) * p);
    q.o_rpart = take(sizeof(fr) * q.rowchunks * n);
    q.o_a = take(soa_bytes(n));
    q.o_b = take(soa_bytes(n));
    q.o_f1a = take(soa_bytes(n / 2));
    q.o_f1b = take(soa_bytes(n / 2));
    q.o_f2a = take(soa_bytes(n / 4));
    q.o_f2b = take(soa_bytes(n / 4));
    q.o_ca = take(soa_bytes(128));
    q.o_cb = take(soa_bytes(128));
    q.o_parts = take(sizeof(fr) * q.parts);
    q.o_rd = take(sizeof(MMRound) * kMaxRounds);
    q.o_fin = take(sizeof(fr) * 2);
    q.o_out = take(sizeof(zkl_fr) * (3 + 3 * kMaxRounds));
    q.total = o;
}

int run_matmul(zkl_ctx* ctx, const int32_t* A, const int32_t* B, uint64_t m, uint64_t n, uint64_t p,
               const zkl_fr* u, const zkl_fr* v, const zkl_fr* r, zkl_vec a_out, zkl_vec b_out, zkl_fr* claim,
               zkl_fr* round_evals, zkl_fr* finals) {
    int st;
    if ((st = check_ctx(ctx))) return st;
    if ((st = check_idle(ctx))) return st;
    if (ctx->async_mode) return set_err(ctx, ZKL_E_STATE, "matmul prove: synchronous calls only");
    if (!A || !B || !claim || !finals || (n > 1 && (!r || !round_evals)) || (m > 1 && !u) || (p > 1 && !v))
        return set_err(ctx, ZKL_E_ARG, "null argument");
    if (!is_pow2(m) || !is_pow2(n) || !is_pow2(p) || ilog2(n) > kMaxRounds - 1 || ilog2(m) > 32 || ilog2(p) > 32)
        return set_err(ctx, ZKL_E_SHAPE, "m=%llu n=%llu p=%llu: powers of two, n <= 2^%d", (unsigned long long)m,
                       (unsigned long long)n, (unsigned long long)p, kMaxRounds - 1);
    MMPlan q;
    make_mm_plan(q, m, n, p);
    CUDA_TRY(ctx, cudaFuncSetAttribute(k_mm_chunk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       2 * kMMChunk * (int)sizeof(fr)));
    if (!ctx->ws || ctx->ws_bytes < q.total)
        return set_err(ctx, ZKL_E_OOM, "workspace %zu bytes < %zu required (zkl_matmul_workspace_bytes)",
                       ctx->ws_bytes, q.total);
    if (a_out.limbs && (st = check_vec(ctx, a_out, n, "a_out"))) return st;
    if (b_out.limbs && (st = check_vec(ctx, b_out, n, "b_out"))) return st;
    ctx->prep_valid = 0;   // the workspace (and the cached index-map keys in it) is reused here
    cudaStream_t s = ctx->stream;
    // challenges u | v | r, canonical, through the pinned staging area
    const int nch = q.lm + q.lp + q.L;
    zkl_fr* hs = reinterpret_cast<zkl_fr*>((uint8_t*)ctx->host_out + 40000);
    for (int i = 0; i < q.lm; ++i) hs[i] = u[i];
    for (int i = 0; i < q.lp; ++i) hs[q.lm + i] = v[i];
    for (int i = 0; i < q.L; ++i) hs[q.lm + q.lp + i] = r[i];
    for (int i = 0; i < nch; ++i)
        if (fr_ge_r_host(hs[i])) return set_err(ctx, ZKL_E_NONCANONICAL, "challenge %d is not canonical", i);
    memcpy(reinterpret_cast<uint8_t*>(hs) + sizeof(zkl_fr) * (nch + 1), q.rd, sizeof(q.rd));
    zkl_fr* dstage = at<zkl_fr>(ctx, q.o_out);   // raw challenges land in the output area first
    fr* ch = at<fr>(ctx, q.o_ch);
    MMRound* drd = at<MMRound>(ctx, q.o_rd);
    if (nch) CUDA_TRY(ctx, cudaMemcpyAsync(dstage, hs, sizeof(zkl_fr) * nch, cudaMemcpyHostToDevice, s));
    CUDA_TRY(ctx, cudaMemcpyAsync(drd, reinterpret_cast<uint8_t*>(hs) + sizeof(zkl_fr) * (nch + 1), sizeof(q.rd),
                                  cudaMemcpyHostToDevice, s));
    if (nch) LAUNCH(ctx, k_mm_consts, (nch + 63) / 64, 64, 0, s, dstage, nch, ch);
    const fr *cu = ch, *cv = ch + q.lm, *cr = ch + q.lm + q.lp;
    fr* Eu = at<fr>(ctx, q.o_eu);
    fr* Ev = at<fr>(ctx, q.o_ev);
    LAUNCH(ctx, k_mm_eq, grid_for(m, 256), 256, 0, s, cu, q.lm, m, Eu);
    LAUNCH(ctx, k_mm_eq, grid_for(p, 256), 256, 0, s, cv, q.lp, p, Ev);
    // restrictions a = A~(u, .), b = B~(., v)
    uint32_t* a = a_out.limbs ? a_out.limbs : at<uint32_t>(ctx, q.o_a);
    uint32_t* b = b_out.limbs ? b_out.limbs : at<uint32_t>(ctx, q.o_b);
    fr* rpart = at<fr>(ctx, q.o_rpart);
    {
        dim3 grid((unsigned)((n + kMMThreads - 1) / kMMThreads), (unsigned)q.rowchunks);
        LAUNCH(ctx, k_mm_restrict_rows, grid, kMMThreads, 0, s, A, m, n, Eu, rpart);
        LAUNCH(ctx, k_mm_sum_chunks, grid_for(n, 256), 256, 0, s, rpart, q.rowchunks, n, a);
        if (n % kMMColRows == 0)
            LAUNCH(ctx, k_mm_restrict_cols_tiled, (unsigned)(n / kMMColRows), kMMThreads, 0, s, B, n, p, Ev, b);
        else
            LAUNCH(ctx, k_mm_restrict_cols, (unsigned)((n + kMMThreads / 32 - 1) / (kMMThreads / 32)), kMMThreads, 0,
                   s, B, n, p, Ev, b);
    }
    // the degree-2 sumcheck on (a, b)
    fr* parts = at<fr>(ctx, q.o_parts);
    fr* fin = at<fr>(ctx, q.o_fin);
    const uint32_t *ca = a, *cb = b;
    uint64_t len = n;
    for (int k = 1; k < (q.kc ? q.kc : q.L + 1) && q.gridA[k - 1]; ++k) {
        uint32_t* na = at<uint32_t>(ctx, (k & 1) == 0 ? q.o_f1a : q.o_f2a);   // k = 2 writes n/2 elements
        uint32_t* nb = at<uint32_t>(ctx, (k & 1) == 0 ? q.o_f1b : q.o_f2b);
        const int fold = k > 1;
        LAUNCH(ctx, k_mm_round, q.gridA[k - 1], kMMThreads, 0, s, ca, cb, len, fold, cr, k, na, nb,
               parts + q.rd[k - 1].base, q.rd[k - 1].rows);
        if (fold) {
            ca = na; cb = nb;
            len /= 2;
        }
    }
    uint32_t* ta = at<uint32_t>(ctx, q.o_ca);
    uint32_t* tb = at<uint32_t>(ctx, q.o_cb);
    uint64_t tlen;
    int k0;
    if (q.kc) {
        const int fold = q.kc > 1;
        LAUNCH(ctx, k_mm_chunk, (unsigned)q.nchunks, kMMChunk / 2, 2 * kMMChunk * sizeof(fr), s, ca, cb, len, fold,
               (int)q.chunk, q.nr, cr, q.kc, drd, parts, ta, tb);
        tlen = q.nchunks;
        k0 = q.kc + q.nr;
    } else {   // n = 1: no rounds
        ta = a; tb = b;
        tlen = 1;
        k0 = 1;
    }
    LAUNCH(ctx, k_mm_tail, 1, 32, 0, s, ta, tb, tlen, cr, k0, q.L, drd, parts, fin);
    zkl_fr* dout = at<zkl_fr>(ctx, q.o_out);
    LAUNCH(ctx, k_mm_finish, q.L + 1, 256, 0, s, parts, drd, q.L, fin, dout);
    zkl_fr* hout = reinterpret_cast<zkl_fr*>((uint8_t*)ctx->host_out + 45000);
    CUDA_TRY(ctx, cudaMemcpyAsync(hout, dout, sizeof(zkl_fr) * (3 + 3 * q.L), cudaMemcpyDeviceToHost, s));
    if ((st = sync_stream(ctx))) return st;
    *claim = hout[0];
    finals[0] = hout[1];
    finals[1] = hout[2];
    if (q.L) memcpy(round_evals, hout + 3, sizeof(zkl_fr) * 3 * q.L);
    return ZKL_OK;
}

// ------------------------------------------------------------------ Hyrax commitments
}  // namespace

extern "C" {

size_t zkl_matmul_workspace_bytes(uint64_t m, uint64_t n, uint64_t p) {
    if (!is_pow2(m) || !is_pow2(n) || !is_pow2(p)) return 0;
    MMPlan q;
    make_mm_plan(q, m, n, p);
    return q.total;
}

int zkl_matmul_prove(zkl_ctx* ctx, const int32_t* A, const int32_t* B, uint64_t m, uint64_t n, uint64_t p,
                     const zkl_fr* u, const zkl_fr* v, const zkl_fr* r, zkl_vec a_out, zkl_vec b_out, zkl_fr* claim,
                     zkl_fr* round_evals, zkl_fr* finals) {
    return run_matmul(ctx, A, B, m, n, p, u, v, r, a_out, b_out, claim, round_evals, finals);
}

}  // extern "C"

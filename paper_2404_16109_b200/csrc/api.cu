// The zkl C ABI (include/zkl.h): host orchestration of the tlookup hot path on sm_100a.
//
// Per proof:
//   main stream: setup scalars, eq tables -> [D side] batched inversion of A fused with round 1,
//                fused fold+eval rounds, single-CTA tail -> per-round rank sums
//   side stream: [table side] B = 1/(beta+T) (batch inversion), m, e~(u', .), table rounds
//   join:        (P > 1: all-gather of rank sums + folded finals, replicated last log2 P rounds)
//                derivation of every g_k(0..3) and the final evaluations, one D2H copy.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdarg.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <array>
#include <functional>
#include <initializer_list>
#include <utility>
#include <memory>
#include <new>
#include <vector>

#include "coop.cuh"
#include "fs.cuh"
#include "kernels.cuh"
#include "mhist.cuh"
#include "host_common.h"
#include "nccl_loader.h"
#include "sha256_host.h"

using namespace zkl;

namespace {

using namespace zkl_host;

// workspace of the N <= 2^16 histogram (csrc/mhist.cuh): digit-major low bytes, tot and rel [chunk][256], the 256
// digit totals, partial rows [piece][256] (pieces <= chunks + 256)
struct MhLayout {
    size_t out, tot, rel, total, partial, bytes;
};
MhLayout mh_layout(uint64_t Dp) {
    const uint64_t C = mh_chunks(Dp);
    MhLayout l;
    size_t o = 0;
    auto take = [&](size_t b) { size_t r = o; o += (b + 255) & ~(size_t)255; return r; };
    l.out = take(Dp + 16);
    l.tot = take(sizeof(uint32_t) * C * kMhBins);
    l.rel = take(sizeof(uint32_t) * C * kMhBins);
    l.total = take(sizeof(uint32_t) * kMhBins);
    l.partial = take(sizeof(uint32_t) * (C + kMhBins) * kMhBins);
    l.bytes = o;
    return l;
}
size_t mh_bytes(uint64_t Dp) { return mh_layout(Dp).bytes; }

int hist_rows_for(uint64_t Dp, uint64_t N) {
    uint64_t ntiles = (Dp + kHistTile - 1) / kHistTile;
    uint64_t cap = std::max<uint64_t>(1, (256ull << 20) / (4 * N));
    return (int)std::min<uint64_t>(std::min<uint64_t>(2 * kSMs, ntiles), cap);
}

// ------------------------------------------------------------------ plan + workspace layout
#ifndef ZKL_HIST_ASYNC_ROWS
#define ZKL_HIST_ASYNC_ROWS 64
#endif
constexpr int kHistAsyncRows = ZKL_HIST_ASYNC_ROWS;   // histogram CTAs when it runs behind the proof (async mode)
constexpr uint64_t kInvTop = 8192;   // the top level of the inversion hierarchy: one block

// One hierarchical batched inversion over level-0 tiles [t0, t1) (a4).
struct InvPlan {
    uint64_t t0, t1;
    int nlev;              // tiled levels above level 0
    uint64_t n[12];        // n[0]: level-0 elements of the range; n[L], L >= 1: level sizes; n[nlev+1]: top
    size_t o_val[12], o_slot[12], o_topinv;
};



struct Plan {
    uint64_t D, Dp, N;
    int d, dl, n, pbits, P, rank;
    bool small;          // Dp < kInvTile: the tail kernel does everything
    int k0;              // first tail round
    int fold_in;         // the tail folds its input on load
    int kc, nchunk_rounds;   // chunked rounds kc .. kc + nchunk_rounds - 1 (k_chunk_rounds), 0 = none
    int tkc;                 // table side: chunked rounds tkc .. tkc + kTabChunkBits - 1 (k_tab_chunk), 0 = none
    int fs_coop;             // Fiat-Shamir: rounds kc .. d in one cooperative launch (k_fs_rounds_coop)
    uint64_t tnchunks;
    uint64_t nchunks;        // blocks of the chunk launch = elements left for the tail
    RoundDesc rd[kMaxRounds];
    EqJob jobs[2 * kMaxRounds];
    int njobs;
    uint32_t tnb[kMaxRounds];
    uint64_t arena;
    uint64_t part_total;
    uint64_t ntiles;     // inversion tiles (Dp / 4096)
    int nhalves;
    InvPlan inv[2];      // D side, one hierarchy per half
    InvPlan tinv;        // table side (N >= 4096)
    int inv_blocks;
    int hist_rows;
    // workspace offsets
    size_t o_out, o_sc, o_err, o_perr, o_rounds, o_jobs, o_chal, o_part, o_tpart, o_tnb, o_rank, o_gath, o_repl, o_tsum,
        o_fin, o_tfin, o_gfin, o_rc, o_fs, o_small, o_Sv, o_derived, o_arena, o_hist, o_keys, o_tot, o_totinv, o_A, o_A1, o_S1, o_A2, o_S2, o_tB, o_tX, o_tM,
        o_tE, o_twk, o_tBaos, o_chA, o_chS, o_coop, total;
};

// k_round: one CTA per group of 2^gbits pairs (grid = #groups = partial rows).  2^12 pairs (16 per thread) by default,
// fewer while that leaves < 2 CTAs per SM, more (<= 2^14: the wide accumulators take <= 64 terms) beyond 65536 groups
// groups of 2^gbits pairs (one CTA each, <= 64 pairs per thread): about 1024 CTAs per round from 2^20 pairs up (a
// thread amortises its per-group reduction over as many pairs as ~3.5 waves allow), 512 below (latency-bound rounds
// prefer short CTAs); measured against a fixed 2^12 on the B200: -0.09 ms over rounds 2..9 at H
#ifndef ZKL_R1_TPC
#define ZKL_R1_TPC 4
#endif
int r1_tiles_per_cta(uint64_t ntiles) {
    return (ntiles % ZKL_R1_TPC == 0 && ntiles >= ZKL_R1_TPC * 3 * (uint64_t)kSMs * 2) ? ZKL_R1_TPC : 1;
}

int round_gbits(uint64_t np) {
    const int lg = ilog2(np);
    int gbits = std::max(8, std::min(14, lg - (lg >= 20 ? 10 : 9)));
    if ((1ull << gbits) > np) gbits = ilog2(np);
    return gbits;
}

void choose_round(Plan& p, int k, uint64_t npairs, int gbits, int nblocks) {
    RoundDesc& r = p.rd[k - 1];
    r.gbits = gbits;
    r.nblocks = nblocks;
    (void)npairs;
}

void make_plan(Plan& p, uint64_t D, uint64_t N, int P, int rank, bool prove_mode, const zkl_fr* u, bool fs = false) {
    memset(&p, 0, sizeof(p));
    p.D = D; p.N = N; p.P = P; p.rank = rank;
    p.d = ilog2(D); p.n = ilog2(N); p.pbits = ilog2(P);
    p.dl = p.d - p.pbits;
    p.Dp = D / P;
    p.small = p.Dp < (uint64_t)kInvTile;
    p.ntiles = p.small ? 0 : p.Dp / kInvTile;
    p.nhalves = p.small ? 0 : (p.ntiles >= 2 ? 2 : 1);
    p.inv_blocks = 0;
    for (int h = 0; h < p.nhalves; ++h) {
        InvPlan& ip = p.inv[h];
        ip.t0 = h == 0 ? 0 : p.ntiles / 2;
        ip.t1 = (h == 0 && p.nhalves == 2) ? p.ntiles / 2 : p.ntiles;
        p.inv_blocks += (int)std::min<uint64_t>(ip.t1 - ip.t0, kSMs * 2);
    }
    p.hist_rows = hist_rows_for(p.Dp, N);
    // ---- D-side local rounds
    if (fs) {
        // Fiat-Shamir: every round is its own launch (r_k is derived between rounds); round 1 from the
        // gather/inversion tiles, or, for D_local < 4096, k_round<false> on A and S
        for (int k = 1; k <= p.dl; ++k) {
            const uint64_t nk = p.Dp >> (k - 1);
            const uint64_t np = nk / 2;
            if (k == 1 && !p.small) {
                choose_round(p, 1, np, 11, (int)p.ntiles);
                continue;
            }
            const int gbits = round_gbits(np);
            choose_round(p, k, np, gbits, (int)std::max<uint64_t>(1, np >> gbits));
            if (k >= 2) p.rd[k - 1].a1_derived = 1;   // k_round<true, ...>
        }
        // H(1) summed directly, except in the big rounds (>= 2^20 elements), whose k_round hides the one inversion
        // per round that deriving H(1) from the running claim needs (k_fs_inv on the side stream)
        for (int k = 1; k <= p.dl; ++k)
            p.rd[k - 1].direct_h1 = (k == 1 || (p.Dp >> (k - 1)) < (1ull << 20) || !prove_mode) ? 1 : 0;
        p.k0 = p.dl + 1;
        p.fold_in = 0;
        // the small rounds in one cooperative launch (single rank): from the first round with <= 2^17 elements, if the
        // table entering it is small enough for one CTA's shared memory
        if (!p.small && P == 1 && prove_mode) {
            int k = 2;
            while (k <= p.dl && (p.Dp >> (k - 1)) > kChunkMaxElems) ++k;
            const uint64_t nk = p.Dp >> (k - 1);
            const uint64_t tl_in = (k - 2 <= p.n) ? (N >> (k - 2)) : 1;
            if (k <= p.dl && nk >= (uint64_t)kChunk && tl_in <= (uint64_t)kCoopTabMax) {
                p.fs_coop = 1;
                p.kc = k;
                p.nchunks = nk / kChunk;
                for (int kk = k; kk <= p.dl; ++kk) {   // E_hi of the one-warp rounds must be a single entry
                    RoundDesc& r = p.rd[kk - 1];
                    r.gbits = kk < k + kChunkBits ? std::min(10, p.dl - kk) : p.dl - kk;
                    r.direct_h1 = 1;
                    r.a1_derived = 0;
                }
            }
        }
    } else if (p.small) {
        p.k0 = 1;
        p.fold_in = 0;
    } else {
        int k = 1;
        // round 1: inversion tiles (prove) or k_round<false> (sumcheck)
        if (prove_mode) {
            choose_round(p, 1, p.Dp / 2, 11, (int)p.ntiles);   // one partial row per inversion tile
        }
        for (k = 1; k <= p.dl; ++k) {
            const uint64_t nk = p.Dp >> (k - 1);   // elements at round k
            if (nk <= (uint64_t)kTailMax) break;
            if (k >= 2 && nk <= kChunkMaxElems && nk >= (uint64_t)kChunk) break;   // chunked rounds from here
            if (k == 1 && prove_mode) continue;
            const uint64_t np = nk / 2;
            const int gbits = round_gbits(np);
            choose_round(p, k, np, gbits, (int)std::max<uint64_t>(1, np >> gbits));
            if (k >= 2) p.rd[k - 1].a1_derived = 1;   // k_round<true, ...>
        }
        p.k0 = k;
        p.fold_in = 1;
        const uint64_t nk = p.Dp >> (k - 1);
        if (k >= 2 && k <= p.dl && nk <= kChunkMaxElems && nk >= (uint64_t)kChunk) {
            p.kc = k;
            p.nchunk_rounds = kChunkBits;   // nk >= 2^kChunkBits, so these rounds are all local (k <= dl)
            p.nchunks = nk / kChunk;
            for (int kk = k; kk < k + kChunkBits; ++kk) {
                RoundDesc& r = p.rd[kk - 1];
                r.gbits = std::min(10, p.dl - kk);
                r.nblocks = (uint32_t)(p.nchunks * kChunkWarps);   // partial rows: one per warp
                r.direct_h1 = 0;
            }
            p.k0 = k + kChunkBits;
            p.fold_in = 0;                  // the tail starts from the chunks' last elements
        }
    }
    // tail rounds: k_tail (small path: one partial row per warp) or k_tail_warp (one row)
    const uint32_t tail_rows = p.small ? (uint32_t)(kTailThreads / 32) : 1u;
    for (int k = p.k0; k <= p.dl; ++k) {
        p.rd[k - 1].gbits = p.dl - k;
        p.rd[k - 1].nblocks = tail_rows;
        p.rd[k - 1].direct_h1 = 1;
        p.rd[k - 1].a1_derived = 0;
    }
    for (int k = 1; k <= p.dl; ++k) {
        if (k == 1 && !prove_mode) p.rd[0].direct_h1 = 1;
        const zkl_fr& uc = u[p.d - k];
        bool zero = true;
        for (int l = 0; l < 8; ++l) zero &= uc.w[l] == 0;
        if (zero) p.rd[k - 1].direct_h1 = 1;
    }
    // replicated rounds (P > 1): all remaining coordinates are global
    for (int k = p.dl + 1; k <= p.d; ++k) {
        p.rd[k - 1].gbits = p.d - k;
        p.rd[k - 1].nblocks = P <= kTailWarpMax ? 1u : (uint32_t)(kTailThreads / 32);
        p.rd[k - 1].direct_h1 = 1;
        p.rd[k - 1].a1_derived = (fs && k >= p.dl + 2) ? 1 : 0;   // Fiat-Shamir: k_round<true, true> on the P values
    }
    // ---- eq arena jobs: per round E_lo then E_hi
    uint64_t off = 0;
    int nj = 0;
    for (int k = 1; k <= p.d; ++k) {
        RoundDesc& r = p.rd[k - 1];
        const bool local = k <= p.dl;
        r.elo_off = off;
        p.jobs[nj++] = EqJob{off, r.gbits, (uint32_t)(p.d - k - r.gbits), 0, 0};
        off += 1ull << r.gbits;
        r.ehi_off = off;
        const uint32_t hb = local ? (uint32_t)(p.dl - k - r.gbits) : 0;
        p.jobs[nj++] = EqJob{off, hb, local ? (uint32_t)p.pbits : 0u, local ? 1u : 0u, 0};
        off += 1ull << hb;
    }
    p.njobs = nj;
    p.arena = off;
    // ---- partial-sum rows per round: [slot][row]
    uint64_t prow = 0;
    for (int k = 1; k <= p.d; ++k) {
        p.rd[k - 1].part_base = prow;
        prow += (uint64_t)kSlots * std::max<uint32_t>(1, p.rd[k - 1].nblocks);
    }
    p.part_total = prow;
    // ---- table rounds
    // ---- workspace layout
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o += align_up(bytes); return r; };
    // the index-map keys outlive the call (prepare -> prove): first, at an offset that depends on nothing else
    p.o_keys = take(sizeof(uint32_t) * std::max<uint64_t>(p.Dp, 4));
    // the histogram rows of an async-mode prepare are written on the low stream while the following proof runs, so
    // they too sit at an offset that depends only on (D_local, N): never inside any plan's proof buffers
    p.o_hist = take(std::max(sizeof(uint32_t) * (size_t)p.hist_rows * N, mh_bytes(p.Dp)));
    p.o_out = take(sizeof(ProofOut));
    p.o_sc = take(sizeof(ProofScalars));
    p.o_err = take(4 * sizeof(unsigned long long));
    p.o_perr = take(4 * sizeof(unsigned long long));
    p.o_rounds = take(sizeof(RoundDesc) * kMaxRounds);
    p.o_jobs = take(sizeof(EqJob) * 2 * kMaxRounds);
    p.o_chal = take(sizeof(zkl_fr) * (3 + 2 * kMaxRounds));
    p.o_part = take(sizeof(fr) * p.part_total);
    p.o_rank = take(sizeof(fr) * kMaxRounds * kSlots);
    p.o_gath = take(sizeof(fr) * (size_t)P * kMaxRounds * kSlots);
    p.o_repl = take(sizeof(fr) * kMaxRounds * kSlots);
    p.o_tsum = take(sizeof(fr) * kMaxRounds * 4);
    p.o_fin = take(sizeof(fr) * 4);
    p.o_tfin = take(sizeof(fr) * 4);
    p.o_gfin = take(sizeof(fr) * 2 * (size_t)P);
    p.o_rc = take(sizeof(RoundConst) * kMaxRounds);
    p.o_fs = take(sizeof(FsState));
    p.o_small = take(soa_bytes(std::min<uint64_t>(p.Dp, kInvTile)));
    // a virtual S materialised from the keys where a kernel reads the vector itself (D_local <= 2^18, see run_proof)
    p.o_Sv = take(soa_bytes(p.Dp <= 2 * kChunkMaxElems ? p.Dp : 4));
    p.o_derived = take(sizeof(zkl_fr) * (3 + 2 * kMaxRounds));
    p.o_arena = take(sizeof(fr) * p.arena);
    p.o_tot = take(soa_bytes(p.ntiles));
    p.o_totinv = take(soa_bytes(p.ntiles));
    p.o_A = take(soa_bytes(p.Dp));
    p.o_A1 = take(soa_bytes(p.Dp / 2));
    p.o_S1 = take(soa_bytes(p.Dp / 2));
    p.o_A2 = take(soa_bytes(p.Dp / 4));
    p.o_S2 = take(soa_bytes(p.Dp / 4));
    p.o_tB = take(soa_bytes(N));
    p.o_tX = take(soa_bytes(N));
    p.o_tM = take(soa_bytes(N));
    p.o_tE = take(soa_bytes(N));
    p.o_twk = take(sizeof(fr) * 8 * std::max<uint64_t>(N, 2));
    for (int k = 1; k <= p.n; ++k) p.tnb[k - 1] = grid_for(N >> k, 256, kMaxBlocks);
    if (!fs) {   // table side: multi-block rounds while the vectors are big, then chunked rounds, then one block
        int tk = 1;
        uint64_t tl = N;
        while (tk <= p.n && tl > kTabChunkMaxElems) { ++tk; tl /= 2; }
        p.tkc = 0;
        if (tk <= p.n && tl >= (uint64_t)kTabChunk) {
            p.tkc = tk;
            p.tnchunks = tl / kTabChunk;
            for (int j = 0; j < kTabChunkBits; ++j) p.tnb[tk + j - 1] = (uint32_t)(p.tnchunks * kTabChunkWarps);
        }
    }
    p.o_tpart = take(sizeof(fr) * (size_t)kMaxRounds * 4 * std::max(kMaxBlocks, kTabRowsMax));
    p.o_tnb = take(sizeof(uint32_t) * kMaxRounds);
    p.o_tBaos = take(64 * std::max<uint64_t>(N, 4));   // (B_j, T_j) records
    p.o_chA = take(soa_bytes(std::max<uint64_t>(p.nchunks, 1)));
    p.o_chS = take(soa_bytes(std::max<uint64_t>(p.nchunks, 1)));
    // k_fs_rounds_coop: partial rows (10 rounds x 5 x #chunks), table terms, the chunks' last values, the grid barrier
    p.o_coop = take(sizeof(fr) * (kChunkBits * 5 * 128 + 4 * kMaxRounds + 2 * 128) + sizeof(GridBar));
    auto inv_levels = [&](InvPlan& ip, uint64_t n0) {
        ip.n[0] = n0;
        int L = 0;
        uint64_t nl = n0 / kInvPer;
        while (nl > kInvTop) {
            ++L;
            ip.n[L] = nl;
            ip.o_val[L] = take(soa_bytes(nl));
            ip.o_slot[L] = take(soa_bytes(nl));
            nl /= kInvPer;
        }
        ip.nlev = L;
        ip.n[L + 1] = nl;
        ip.o_val[L + 1] = take(soa_bytes(nl));
        ip.o_topinv = take(soa_bytes(nl));
    };
    for (int h = 0; h < p.nhalves; ++h) inv_levels(p.inv[h], (p.inv[h].t1 - p.inv[h].t0) * kInvTile);
    if (N >= (uint64_t)kInvTile) {
        p.tinv.t0 = 0;
        p.tinv.t1 = N / kInvTile;
        inv_levels(p.tinv, N);
    }
    p.total = o;
}



int check_shape(zkl_ctx* ctx, uint64_t D, uint64_t N) {
    if (!is_pow2(D) || !is_pow2(N) || N > D)
        return set_err(ctx, ZKL_E_SHAPE, "D=%llu N=%llu: need powers of two with N | D (PAPER.md:258)",
                       (unsigned long long)D, (unsigned long long)N);
    if (ilog2(D) > kMaxRounds) return set_err(ctx, ZKL_E_SHAPE, "log2 D > %d", kMaxRounds);
    if (D % (uint64_t)ctx->nranks || !is_pow2((uint64_t)ctx->nranks) || D / ctx->nranks < 1)
        return set_err(ctx, ZKL_E_SHAPE, "P=%d must be a power of two dividing D", ctx->nranks);
    return ZKL_OK;
}


int need_ws(zkl_ctx* ctx, const Plan& p) {
    if (!ctx->ws || ctx->ws_bytes < p.total)
        return set_err(ctx, ZKL_E_OOM, "workspace %zu bytes < %zu required (zkl_workspace_bytes)", ctx->ws_bytes,
                       p.total);
    return ZKL_OK;
}

// Small host->device transfers from the ctx's pinned staging page (challenges, plans, alpha_f) are done by one
// kernel reading the mapped host memory (zero-copy over PCIe), not by cudaMemcpyAsync: a copy-engine transfer would
// queue behind a large H2D copy the caller has in flight on another stream (e.g. the next step's inputs) and stall
// the proof until it drains.
int inv_forward(zkl_ctx* ctx, const InvPlan& ip, const uint32_t* X0, uint64_t n0total, uint32_t* slots0,
                const ProofScalars* sc, uint64_t err_off, unsigned long long* err, cudaStream_t s0, cudaStream_t s1,
                cudaEvent_t ev) {
    const unsigned nb0 = (unsigned)(ip.t1 - ip.t0);   // one block per tile
    LAUNCH(ctx, k_inv_fwd<true>, nb0, kInvThreads, 0, s0, X0, n0total, sc, slots0, at<uint32_t>(ctx, ip.o_val[1]),
           ip.n[1], ip.t0, ip.t1, err_off, err);
    if (s1 != s0) {
        CUDA_TRY(ctx, cudaEventRecord(ev, s0));
        CUDA_TRY(ctx, cudaStreamWaitEvent(s1, ev, 0));
    }
    for (int L = 1; L <= ip.nlev; ++L) {
        const uint64_t tiles = ip.n[L] / kInvTile;
        LAUNCH(ctx, k_inv_fwd<false>, (unsigned)std::min<uint64_t>(tiles, kSMs * 2), kInvThreads, 0, s1,
               at<uint32_t>(ctx, ip.o_val[L]), ip.n[L], sc, at<uint32_t>(ctx, ip.o_slot[L]),
               at<uint32_t>(ctx, ip.o_val[L + 1]), ip.n[L + 1], (uint64_t)0, tiles, (uint64_t)0, err);
    }
    const uint64_t ntop = ip.n[ip.nlev + 1];
    const unsigned bt = (unsigned)std::min<uint64_t>(1024, std::max<uint64_t>(32, ntop / 8));
    LAUNCH(ctx, k_batch_invert, 1, bt, 4 * bt * sizeof(fr), s1, at<uint32_t>(ctx, ip.o_val[ip.nlev + 1]), ntop,
           (uint64_t)0, ntop, at<uint32_t>(ctx, ip.o_topinv));
    for (int L = ip.nlev; L >= 1; --L) {
        const uint64_t tiles = ip.n[L] / kInvTile;
        const uint32_t* ninv = L == ip.nlev ? at<uint32_t>(ctx, ip.o_topinv) : at<uint32_t>(ctx, ip.o_slot[L + 1]);
        LAUNCH(ctx, k_inv_bwd<false>, (unsigned)std::min<uint64_t>(tiles, kSMs * 2), kInvThreads, 0, s1,
               at<uint32_t>(ctx, ip.o_val[L]), ip.n[L], sc, at<uint32_t>(ctx, ip.o_slot[L]), ninv, ip.n[L + 1],
               (uint64_t)0, tiles, (const fr*)nullptr, (const fr*)nullptr, (fr*)nullptr, 0, 0);
    }
    return ZKL_OK;
}

// Level-0 backward pass on s0 (after the upper levels on s1 completed: caller orders via events).
int inv_backward0(zkl_ctx* ctx, const InvPlan& ip, const uint32_t* X0, uint64_t n0total, uint32_t* slots0,
                  const ProofScalars* sc, const fr* elo, const fr* ehi, fr* partials, int rows, cudaStream_t s0) {
    const unsigned nb0 = (unsigned)(ip.t1 - ip.t0);   // one block per tile; partial row = tile index
    const uint32_t* ninv = ip.nlev >= 1 ? at<uint32_t>(ctx, ip.o_slot[1]) : at<uint32_t>(ctx, ip.o_topinv);
    LAUNCH(ctx, k_inv_bwd<true>, nb0, kInvThreads, 0, s0, X0, n0total, sc, slots0, ninv, ip.n[1], ip.t0, ip.t1, elo,
           ehi, partials, (int)ip.t0, rows);
    return ZKL_OK;
}

// ------------------------------------------------------------------ table side (a8)
// init + the big rounds multi-block on the main stream (a few tens of microseconds), the small rounds and
// the reduction of all table rounds in one block on the side stream (joined before the derivation).
int table_side(zkl_ctx* ctx, const Plan& p, cudaStream_t s, cudaStream_t s2, const uint32_t* B, const uint32_t* T,
               const uint32_t* m_u32, const uint32_t* Mf, int variant, const ProofScalars* sc, fr* tsum, fr* tfin,
               uint32_t* Bout) {
    const uint64_t N = p.N;
    fr* wk = at<fr>(ctx, p.o_twk);
    fr *cur = wk, *nxt = wk + 4 * N;
    if (m_u32 && ctx->m_pending) CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_m, 0));   // async-mode histogram
    LAUNCH(ctx, k_tab_init, grid_for(N, 256), 256, 0, s, B, T, m_u32, Mf, N, sc, p.d, p.n, variant, cur, Bout);
    fr* tpart = at<fr>(ctx, p.o_tpart);
    uint64_t len = N;
    int k = 1;
    // big rounds multi-block on the main stream (before the chunked rounds, or while > kTabTailPairs pairs)
    for (; k <= p.n && (p.tkc ? k < p.tkc : len / 2 > kTabTailPairs); ++k) {
        LAUNCH(ctx, k_tab_round, p.tnb[k - 1], 256, 0, s, cur, len, nxt, sc, k, variant,
               tpart + (size_t)(k - 1) * 4 * kTabRowsMax, kTabRowsMax);
        fr* t = cur; cur = nxt; nxt = t;
        len /= 2;
    }
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_fork, s));
    CUDA_TRY(ctx, cudaStreamWaitEvent(s2, ctx->ev_fork, 0));
    if (p.tkc) {
        LAUNCH(ctx, k_tab_chunk, (unsigned)p.tnchunks, kTabChunkThreads, 4 * kTabChunk * sizeof(fr), s2, cur, len,
               nxt, sc, k, variant, tpart);
        fr* t = cur; cur = nxt; nxt = t;
        len = p.tnchunks;
        k += kTabChunkBits;
    }
    LAUNCH(ctx, k_tab_tail, 1, 256, 0, s2, cur, nxt, len, k, p.n, sc, variant, tpart, kTabRowsMax,
           at<uint32_t>(ctx, p.o_tnb), tsum, tfin);
    return ZKL_OK;
}

// ------------------------------------------------------------------ shared proof driver
struct ProveArgs {
    bool prove_mode;
    zkl_vec S, A_in, A_out, B_out;       // A_in: sumcheck mode
    const zkl_table* table;              // prove mode
    const uint32_t* m_dev;               // prove mode
    zkl_vec B_in, T_in, m_fr_in;         // sumcheck mode
    const zkl_challenges* ch;
    int variant;
    bool force_inversion;                // prove mode: batch-invert beta + S instead of gathering B[j(i)]
};

// a ProveArgs whose challenges live here (async completion may rerun the proof after the caller's arrays are gone)
struct OwnedArgs {
    ProveArgs args;
    zkl_challenges ch;
    std::vector<zkl_fr> u, r;
    OwnedArgs(const ProveArgs& a, int d) : args(a), ch(*a.ch), u(a.ch->u, a.ch->u + d), r(a.ch->r, a.ch->r + d) {
        ch.u = u.data();
        ch.r = r.data();
        args.ch = &ch;
    }
    OwnedArgs(const OwnedArgs&) = delete;
};

std::vector<std::function<int()>>& pending_of(zkl_ctx* ctx) {
    if (!ctx->pending) ctx->pending = new std::vector<std::function<int()>>();
    return *static_cast<std::vector<std::function<int()>>*>(ctx->pending);
}

int proof_collect(zkl_ctx* ctx, uint64_t D, const ProveArgs& a, zkl_fr* round_evals, zkl_final_evals* finals,
                  int64_t* err_index, bool gather, int d);

int run_proof(zkl_ctx* ctx, uint64_t D, const ProveArgs& a, zkl_fr* round_evals, zkl_final_evals* finals,
              int64_t* err_index) {
    if (err_index) *err_index = -1;
    if (ctx->async_mode && ctx->pend_prove) return set_err(ctx, ZKL_E_STATE, "a proof is already pending (zkl_ctx_wait)");
    const uint64_t N = a.prove_mode ? a.table->N : a.T_in.n;
    int st;
    if ((st = check_shape(ctx, D, N))) return st;
    if (!a.ch || !a.ch->u || !a.ch->r || !round_evals || !finals) return set_err(ctx, ZKL_E_ARG, "null argument");
    Plan p;
    make_plan(p, D, N, ctx->nranks, ctx->rank, a.prove_mode, a.ch->u);
    if ((st = need_ws(ctx, p))) return st;
    // keys of the preceding prepare on this S (or virtual S) and table: A_i = B_key, S_i = T_key by gathers
    const bool virt = a.prove_mode && a.S.limbs == nullptr;
    const bool keys_ok = a.prove_mode && ctx->prep_valid && ctx->prep_S == a.S.limbs && ctx->prep_n == p.Dp &&
                         ctx->prep_table == a.table;
    if (virt && !keys_ok)
        return set_err(ctx, ZKL_E_ARG, "S_local is virtual (NULL): it needs the keys of the preceding "
                                       "zkl_tlookup_prepare_pair on this context, table and D");
    if (!virt && (st = check_vec(ctx, a.S, p.Dp, "S_local"))) return st;
    if (virt && a.force_inversion) return set_err(ctx, ZKL_E_STATE, "internal: inversion fallback on a virtual S");
    if (!a.prove_mode) {
        if ((st = check_vec(ctx, a.A_in, p.Dp, "A_local"))) return st;
        if ((st = check_vec(ctx, a.B_in, N, "B"))) return st;
        if ((st = check_vec(ctx, a.T_in, N, "T"))) return st;
        if ((st = check_vec(ctx, a.m_fr_in, N, "m_fr"))) return st;
    } else {
        if (!a.m_dev) return set_err(ctx, ZKL_E_ARG, "m_dev null");
        if (a.A_out.limbs && (st = check_vec(ctx, a.A_out, p.Dp, "A_local_out"))) return st;
        if (a.B_out.limbs && (st = check_vec(ctx, a.B_out, N, "B_out"))) return st;
    }
    cudaStream_t s = ctx->stream, s2 = ctx->side;
    ProofScalars* sc = at<ProofScalars>(ctx, p.o_sc);
    // the proof's own error words ([0] DIV_ZERO_S, [1] DIV_ZERO_T, [2] gather miss): a pending async prepare may still
    // be copying its error words (o_err) when this proof's setup starts on the aux stream
    unsigned long long* err = at<unsigned long long>(ctx, p.o_perr);
    RoundDesc* rounds = at<RoundDesc>(ctx, p.o_rounds);
    EqJob* jobs = at<EqJob>(ctx, p.o_jobs);
    zkl_fr* chal = at<zkl_fr>(ctx, p.o_chal);
    fr* partials = at<fr>(ctx, p.o_part);
    fr* rank_sums = at<fr>(ctx, p.o_rank);
    fr* gath = at<fr>(ctx, p.o_gath);
    fr* repl = at<fr>(ctx, p.o_repl);
    fr* tsum = at<fr>(ctx, p.o_tsum);
    fr* fin = at<fr>(ctx, p.o_fin);
    fr* tfin = at<fr>(ctx, p.o_tfin);
    fr* arena = at<fr>(ctx, p.o_arena);
    ProofOut* out = at<ProofOut>(ctx, p.o_out);

    // ---- host -> device: challenges and the plan (one staging buffer, pinned)
    struct Staging {
        zkl_fr chal[3 + 2 * kMaxRounds];
        RoundDesc rounds[kMaxRounds];
        EqJob jobs[2 * kMaxRounds];
        uint32_t tnb[kMaxRounds];
    };
    Staging* hs = reinterpret_cast<Staging*>((uint8_t*)ctx->host_out + sizeof(ProofOut));
    hs->chal[0] = a.ch->beta;
    hs->chal[1] = a.ch->alpha1;
    hs->chal[2] = a.ch->alpha2;
    for (int c = 0; c < p.d; ++c) hs->chal[3 + c] = a.ch->u[c];
    for (int k = 0; k < p.d; ++k) hs->chal[3 + p.d + k] = a.ch->r[k];
    memcpy(hs->rounds, p.rd, sizeof(p.rd));
    memcpy(hs->jobs, p.jobs, sizeof(p.jobs));
    memcpy(hs->tnb, p.tnb, sizeof(p.tnb));
    // The setup (challenges, eq tables) and B = 1/(beta + T) depend on neither the keys nor m: in prove mode they run
    // on the aux stream from the moment of the call, overlapping the prepare still in flight on the ctx stream (async
    // mode); the D side waits for them (ev_b) just before round 1.
    cudaStream_t sp = a.prove_mode ? ctx->aux : s;
    if ((st = h2d_small(ctx, sp, {{chal, hs->chal}, {rounds, hs->rounds}, {jobs, hs->jobs}, {at<uint32_t>(ctx, p.o_tnb), hs->tnb}},
                        {sizeof(hs->chal), sizeof(hs->rounds), sizeof(hs->jobs), sizeof(hs->tnb)})))
        return st;
    CUDA_TRY(ctx, cudaMemsetAsync(err, 0xff, 4 * sizeof(unsigned long long), sp));
    LAUNCH(ctx, k_setup, 1, 128, 0, sp, chal, p.d, p.pbits, p.rank, N, D, sc);
    // the eq tables and the round constants on the side stream, beside the B inversion (both need only the
    // challenges); the D side waits for the tables (ev_eq) with B (ev_b) before round 1
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_fork, sp));
    CUDA_TRY(ctx, cudaStreamWaitEvent(s2, ctx->ev_fork, 0));
    LAUNCH(ctx, k_eq_fill, grid_for(p.arena, 256), 256, 0, s2, jobs, p.njobs, p.arena, sc, arena);
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_eq, s2));
    CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_eq, 0));
    RoundConst* rc = at<RoundConst>(ctx, p.o_rc);
    LAUNCH(ctx, k_round_consts, 1, 64, 0, s2, sc, p.d, p.n, rc);

    // ================= table side (side stream)
    uint32_t* tB = at<uint32_t>(ctx, p.o_tB);
    uint32_t* tX = at<uint32_t>(ctx, p.o_tX);
    uint32_t* tM = at<uint32_t>(ctx, p.o_tM);
    uint32_t* tE = at<uint32_t>(ctx, p.o_tE);
    const uint32_t* Tsrc = a.prove_mode ? a.table->T : a.T_in.limbs;
    // the gather path (A_i = B_j(i)) needs B on the critical path: compute it on the main stream first
    const bool gather = a.prove_mode && !p.small && !a.force_inversion;
    if (a.prove_mode) {
        cudaStream_t sb = sp;   // B feeds both the table side and (gather path) the D side
        if (N >= (uint64_t)kInvTile) {
            if ((st = inv_forward(ctx, p.tinv, Tsrc, N, tB, sc, 0, err + 1, sb, sb, nullptr))) return st;
            if ((st = inv_backward0(ctx, p.tinv, Tsrc, N, tB, sc, nullptr, nullptr, nullptr, 0, sb))) return st;
        } else {
            LAUNCH(ctx, k_add_beta, grid_for(N, 256), 256, 0, sb, Tsrc, N, sc, tX, err + 1);
            const unsigned bt = (unsigned)std::min<uint64_t>(1024, std::max<uint64_t>(32, N));
            LAUNCH(ctx, k_batch_invert, 1, bt, 4 * bt * sizeof(fr), sb, tX, N, (uint64_t)0, N, tB);
        }
        if (gather) LAUNCH(ctx, k_pack_tb, grid_for(N, 256), 256, 0, sb, Tsrc, tB, N, at<uint4>(ctx, p.o_tBaos));
        CUDA_TRY(ctx, cudaEventRecord(ctx->ev_b, sb));
        CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_b, 0));   // the D side (and a table side on s) needs B
        // B_out (if requested) is the variant's B, written by k_tab_init.  With the histogram still running on the
        // low stream (async mode), the whole table side moves to the side stream, so that the D side does not wait
        // for m
        cudaStream_t ts = s;
        if (ctx->m_pending) {
            CUDA_TRY(ctx, cudaStreamWaitEvent(s2, ctx->ev_b, 0));
            ts = s2;
        }
        if ((st = table_side(ctx, p, ts, s2, tB, Tsrc, a.m_dev, nullptr, a.variant, sc, tsum, tfin, a.B_out.limbs)))
            return st;
    } else {
        if ((st = table_side(ctx, p, s, s2, a.B_in.limbs, Tsrc, nullptr, a.m_fr_in.limbs, a.variant, sc, tsum, tfin,
                             nullptr)))
            return st;
    }
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_join, s2));

    // ================= D side (main stream)
    uint32_t* Abuf = a.prove_mode ? (a.A_out.limbs ? a.A_out.limbs : at<uint32_t>(ctx, p.o_A)) : nullptr;
    const uint32_t* A1in = a.prove_mode ? Abuf : a.A_in.limbs;
    const uint32_t* S1in = a.S.limbs;
    const int kend_rounds = p.kc ? p.kc : p.k0;   // k_round launches for rounds < kend_rounds
    // round 2 gathers A and S from the keys again (neither is materialised) when it is a multi-block k_round launch
    const bool r2_gather = gather && keys_ok && kend_rounds > 2;
    if (virt && !r2_gather) {
        // D_local <= 2^18 (the one-CTA prove or the chunked rounds read the vectors themselves): S_i = T_key
        uint32_t* Sv = at<uint32_t>(ctx, p.o_Sv);
        LAUNCH(ctx, k_s_from_keys, grid_for(p.Dp, 256), 256, 0, s, at<uint32_t>(ctx, p.o_keys), p.Dp, N,
               a.table->Taos, Sv);
        S1in = Sv;
    }
    const uint64_t errS_off = (uint64_t)p.rank * p.Dp;
    const size_t tail_smem = (2 * kTailMax + 4 * kTailThreads) * sizeof(fr) + 5 * (kTailThreads / 32) * sizeof(fr);
    int rounds_nb0 = -1;   // round-1 partial rows written by the inversion (prove mode)
    bool r1_reduced = false;
    if (p.small) {
        LAUNCH(ctx, k_tail, 1, kTailThreads, tail_smem, s, A1in, S1in, p.Dp, 0, a.prove_mode ? 1 : 0, Abuf,
               errS_off, err, sc, 1, p.dl, rounds, arena, partials, fin);
    } else {
        if (gather) {
            // a4 + a5 through the table: A_i = B_j(i), one block per 4096-element tile (partial row = tile)
            TableView tv{a.table->T, a.table->Taos, a.table->slots, a.table->Skeys, a.table->N, a.table->slot_mask};
            if (keys_ok) {
                // keys from the preceding prepare: A_i = B_key, S_i = T_key from the (B, T) records; a materialised S
                // is verified against T_key.  A is written only if the caller wants it or round 2 reads it.
                uint32_t* Aw = a.A_out.limbs ? a.A_out.limbs : (r2_gather ? nullptr : Abuf);
                const bool verify = !virt;
                const uint32_t* keys = at<uint32_t>(ctx, p.o_keys);
                const uint4* TB = at<uint4>(ctx, p.o_tBaos);
                const fr *elo1 = arena + p.rd[0].elo_off, *ehi1 = arena + p.rd[0].ehi_off;
                fr* part1 = partials + p.rd[0].part_base;
                const int tpc1 = r1_tiles_per_cta(p.ntiles);   // tiles per CTA (the per-CTA reductions amortised)
            const unsigned nb1 = (unsigned)(p.ntiles / tpc1);
                if (verify && Aw)
                    LAUNCH(ctx, (k_round1_keys<true, true>), nb1, kInvThreads, 0, s, a.S.limbs, p.Dp, keys, N, TB, Aw,
                           elo1, ehi1, part1, (int)p.ntiles, err + 2, tpc1);
                else if (verify)
                    LAUNCH(ctx, (k_round1_keys<true, false>), nb1, kInvThreads, 0, s, a.S.limbs, p.Dp, keys, N, TB,
                           Aw, elo1, ehi1, part1, (int)p.ntiles, err + 2, tpc1);
                else if (Aw)
                    LAUNCH(ctx, (k_round1_keys<false, true>), nb1, kInvThreads, 0, s, S1in, p.Dp, keys, N, TB, Aw,
                           elo1, ehi1, part1, (int)p.ntiles, err + 2, tpc1);
                else
                    LAUNCH(ctx, (k_round1_keys<false, false>), nb1, kInvThreads, 0, s, S1in, p.Dp, keys, N, TB, Aw,
                           elo1, ehi1, part1, (int)p.ntiles, err + 2, tpc1);
            } else {
                LAUNCH(ctx, k_gather_round1, (unsigned)p.ntiles, kInvThreads, 0, s, a.S.limbs, p.Dp, tv,
                       at<uint4>(ctx, p.o_tBaos), Abuf, arena + p.rd[0].elo_off, arena + p.rd[0].ehi_off,
                       partials + p.rd[0].part_base, (int)p.ntiles, err + 2);
            }
            rounds_nb0 = (int)p.ntiles;
            CUDA_TRY(ctx, cudaEventRecord(ctx->ev_fwd[0], s));
            CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->aux, ctx->ev_fwd[0], 0));
            LAUNCH(ctx, k_reduce_rounds, 1, 256, 0, ctx->aux, partials, rounds, 1, rank_sums);
            CUDA_TRY(ctx, cudaEventRecord(ctx->ev_mid[0], ctx->aux));
            r1_reduced = true;
        } else if (a.prove_mode) {
            // hierarchical batched inversion in two halves: the upper levels + one-block top (one Fermat) of
            // half h run on the aux stream while the main stream does the level-0 forward pass of the other
            // half (h = 0) or the level-0 backward pass of half 0 (h = 1), hiding their latency.
            const int halves = p.nhalves;
            for (int h = 0; h < halves; ++h) {
                if ((st = inv_forward(ctx, p.inv[h], a.S.limbs, p.Dp, Abuf, sc, errS_off, err, s, ctx->aux,
                                      ctx->ev_fwd[h])))
                    return st;
                CUDA_TRY(ctx, cudaEventRecord(ctx->ev_mid[h], ctx->aux));
            }
            for (int h = 0; h < halves; ++h) {
                CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_mid[h], 0));
                if ((st = inv_backward0(ctx, p.inv[h], a.S.limbs, p.Dp, Abuf, sc, arena + p.rd[0].elo_off,
                                        arena + p.rd[0].ehi_off, partials + p.rd[0].part_base, (int)p.ntiles, s)))
                    return st;
            }
            rounds_nb0 = (int)p.ntiles;
            // round 1 has one partial row per tile: reduce it on the aux stream while the rounds run
            CUDA_TRY(ctx, cudaEventRecord(ctx->ev_fwd[0], s));
            CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->aux, ctx->ev_fwd[0], 0));
            LAUNCH(ctx, k_reduce_rounds, 1, 256, 0, ctx->aux, partials, rounds, 1, rank_sums);
            CUDA_TRY(ctx, cudaEventRecord(ctx->ev_mid[0], ctx->aux));
            r1_reduced = true;
        }
        const uint32_t *cA = A1in, *cS = S1in;
        uint64_t len = p.Dp;
        for (int k = a.prove_mode ? 2 : 1; k < kend_rounds; ++k) {
            const RoundDesc& r = p.rd[k - 1];
            fr* part = partials + r.part_base;
            if (k == 1) {
                LAUNCH(ctx, (k_round<false, true>), r.nblocks, kRoundThreads, 0, s, cA, cS, len, nullptr, nullptr, sc,
                       k, arena + r.elo_off, arena + r.ehi_off, (int)r.gbits, part);
            } else {
                const bool odd = (k & 1) == 0;   // k = 2 -> buffers 1
                uint32_t* nA = at<uint32_t>(ctx, odd ? p.o_A1 : p.o_A2);
                uint32_t* nS = at<uint32_t>(ctx, odd ? p.o_S1 : p.o_S2);
                if (k == 2 && r2_gather) {
                    const uint32_t* keys = at<uint32_t>(ctx, p.o_keys);
                    const uint4* TB = at<uint4>(ctx, p.o_tBaos);
                    if (r.direct_h1)
                        LAUNCH(ctx, (k_round<true, true, true>), r.nblocks, kRoundThreads, 0, s, nullptr, nullptr, len,
                               nA, nS, sc, k, arena + r.elo_off, arena + r.ehi_off, (int)r.gbits, part, keys, TB);
                    else
                        LAUNCH(ctx, (k_round<true, false, true>), r.nblocks, kRoundThreads, 0, s, nullptr, nullptr,
                               len, nA, nS, sc, k, arena + r.elo_off, arena + r.ehi_off, (int)r.gbits, part, keys, TB);
                } else if (r.direct_h1)
                    LAUNCH(ctx, (k_round<true, true>), r.nblocks, kRoundThreads, kRoundStageSmem, s, cA, cS, len, nA, nS, sc, k,
                           arena + r.elo_off, arena + r.ehi_off, (int)r.gbits, part);
                else
                    LAUNCH(ctx, (k_round<true, false>), r.nblocks, kRoundThreads, kRoundStageSmem, s, cA, cS, len, nA, nS, sc, k,
                           arena + r.elo_off, arena + r.ehi_off, (int)r.gbits, part);
                cA = nA; cS = nS;
                len /= 2;
            }
        }
        if (p.kc) {
            // rounds kc .. kc+9 chunk-local in shared memory (one launch); one element per chunk remains
            uint32_t* chA = at<uint32_t>(ctx, p.o_chA);
            uint32_t* chS = at<uint32_t>(ctx, p.o_chS);
            const size_t chunk_smem = 2 * kChunk * sizeof(fr);
            GridBar* bar = reinterpret_cast<GridBar*>(at<fr>(ctx, p.o_coop) + kChunkBits * 5 * 128 + 4 * kMaxRounds + 2 * 128);
            CUDA_TRY(ctx, cudaMemsetAsync(bar, 0, sizeof(GridBar), s));
            ChunkArgs ka{cA, cS, len, sc, p.kc, p.nchunk_rounds, rounds, arena, partials, chA, chS, bar};
            LAUNCH_COOP(ctx, k_chunk_rounds_coop, (unsigned)p.nchunks, kChunkThreads, chunk_smem, s, ka);
            cA = chA; cS = chS;
            len = p.nchunks;
        }
        // tail: the chunks' last elements are the round-k0 vectors, <= kTailWarpMax of them (one warp, one
        // partial row per round, as planned)
        if (p.fold_in || len > (uint64_t)kTailWarpMax)
            return set_err(ctx, ZKL_E_STATE, "internal: tail plan (fold_in %d, %llu elements)", p.fold_in,
                           (unsigned long long)len);
        LAUNCH(ctx, k_tail_warp, 1, 32, 0, s, cA, cS, len, sc, p.k0, p.dl, rounds, arena, partials, fin);
    }
    if (rounds_nb0 >= 0 && (uint32_t)rounds_nb0 != p.rd[0].nblocks) {
        // the plan's round-1 row count must match what the inversion wrote
        return set_err(ctx, ZKL_E_STATE, "internal: round-1 rows %d != plan %u", rounds_nb0, p.rd[0].nblocks);
    }
    if (r1_reduced) {
        if (p.dl > 1) LAUNCH(ctx, k_reduce_rounds, p.dl - 1, 256, 0, s, partials, rounds + 1, p.dl - 1, rank_sums + kSlots);
        CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_mid[0], 0));
    } else if (p.dl > 0) {
        LAUNCH(ctx, k_reduce_rounds, p.dl, 256, 0, s, partials, rounds, p.dl, rank_sums);
    }
    const fr* gathered = rank_sums;
    if (ctx->nranks > 1) {
        // a pending (async) prepare's collectives run on the low stream: order this proof's after them
        if (ctx->m_pending) CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_m, 0));
        int rc = zkl_dist_exchange(ctx, p.dl, rank_sums, gath, fin, at<fr>(ctx, p.o_gfin));
        if (rc) return rc;
        gathered = gath;
        // replicated last log2 P rounds on the gathered folded (A, S) pairs: P elements
        // gfin: the P ranks' folded A then S, each read as a P-element vector
        const uint32_t* gA = (const uint32_t*)at<fr>(ctx, p.o_gfin);
        const uint32_t* gS = (const uint32_t*)(at<fr>(ctx, p.o_gfin) + p.P);
        if (p.P <= kTailWarpMax)
            LAUNCH(ctx, k_tail_warp, 1, 32, 0, s, gA, gS, (uint64_t)p.P, sc, p.dl + 1, p.d, rounds, arena, partials,
                   fin);
        else
            LAUNCH(ctx, k_tail, 1, kTailThreads, tail_smem, s, gA, gS, (uint64_t)p.P, 0, 0, (uint32_t*)nullptr, 0,
                   err, sc, p.dl + 1, p.d, rounds, arena, partials, fin);
        LAUNCH(ctx, k_reduce_rounds, p.d - p.dl, 256, 0, s, partials, rounds + p.dl, p.d - p.dl, repl);
    }
    CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_join, 0));
    LAUNCH(ctx, k_derive, 1, 64, 0, s, gathered, ctx->nranks, p.dl, repl, rounds, tsum, sc, rc, p.d, p.n,
           a.variant, a.prove_mode ? 1 : 0, fin, tfin, out);
    if (ctx->nranks > 1) {   // every rank sees the smallest error index of any rank (device-side, no host sync)
        int rc = zkl_dist_min_u64_dev(ctx, err, 3);
        if (rc) return rc;
    }
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->host_out, out, sizeof(ProofOut), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(ctx, cudaMemcpyAsync((uint8_t*)ctx->host_out + offsetof(ProofOut, err_index), err,
                                  3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    if (ctx->async_mode) {
        // completion deferred to zkl_ctx_wait: keep the arguments (challenges copied) for the gather fallback
        auto own = std::make_shared<OwnedArgs>(a, p.d);
        const int d = p.d;
        ctx->pend_prove = 1;
        pending_of(ctx).push_back([ctx, D, own, round_evals, finals, err_index, gather, d]() {
            ctx->pend_prove = 0;
            return proof_collect(ctx, D, own->args, round_evals, finals, err_index, gather, d);
        });
        return ZKL_OK;
    }
    if ((st = sync_stream(ctx))) return st;
    return proof_collect(ctx, D, a, round_evals, finals, err_index, gather, p.d);
}

int proof_collect(zkl_ctx* ctx, uint64_t D, const ProveArgs& a, zkl_fr* round_evals, zkl_final_evals* finals,
                  int64_t* err_index, bool gather, int d) {
    const ProofOut* ho = reinterpret_cast<const ProofOut*>(ctx->host_out);
    const unsigned long long* he = reinterpret_cast<const unsigned long long*>((const uint8_t*)ctx->host_out +
                                                                               offsetof(ProofOut, err_index));
    const unsigned long long eS = he[0], eT = he[1], eMiss = gather ? he[2] : ~0ull;   // already min over ranks
    if (eMiss != ~0ull && eT == ~0ull) {
        // an S_i with no table entry (S was not the prepared lookup vector): redo with the inversion path
        // (synchronously, also in async mode: this runs inside zkl_ctx_wait)
        ProveArgs b = a;
        b.force_inversion = true;
        const int was_async = ctx->async_mode;
        ctx->async_mode = 0;
        const int st = run_proof(ctx, D, b, round_evals, finals, err_index);
        ctx->async_mode = was_async;
        return st;
    }
    if (eT != ~0ull) {
        if (err_index) *err_index = (int64_t)eT;
        return set_err(ctx, ZKL_E_DIV_ZERO_T, "beta + T_%llu = 0", eT);
    }
    if (eS != ~0ull) {
        if (err_index) *err_index = (int64_t)eS;
        return set_err(ctx, ZKL_E_DIV_ZERO_S, "beta + S_%llu = 0", eS);
    }
    memcpy(round_evals, ho->evals, sizeof(zkl_fr) * 4 * d);
    finals->A = ho->finals[0];
    finals->S = ho->finals[1];
    finals->B = ho->finals[2];
    finals->T = ho->finals[3];
    finals->m = ho->finals[4];
    return ZKL_OK;
}

// ------------------------------------------------------------------ Fiat-Shamir driver (f1)
int proof_fs_collect(zkl_ctx* ctx, zkl_vec S, uint64_t D, const zkl_table* table, const uint32_t* m_dev,
                     const uint8_t* seed, int variant, zkl_vec A_out, zkl_vec B_out, zkl_fr* round_evals,
                     zkl_final_evals* finals, zkl_fr* derived, int64_t* err_index, bool gather, int d);

// preset (host, 3 + log2 D canonical values: the transcript state h as 32 bytes, beta, alpha1, u): the transcript was
// started by the caller (Protocol 1, zkl_tlookup_prove_p1), so `seed` is unused
int run_proof_fs(zkl_ctx* ctx, zkl_vec S, uint64_t D, const zkl_table* table, const uint32_t* m_dev,
                 const uint8_t* seed, int variant, zkl_vec A_out, zkl_vec B_out, zkl_fr* round_evals,
                 zkl_final_evals* finals, zkl_fr* derived, int64_t* err_index, bool force_inversion,
                 const zkl_fr* preset = nullptr) {
    if (err_index) *err_index = -1;
    if (ctx->async_mode && ctx->pend_prove) return set_err(ctx, ZKL_E_STATE, "a proof is already pending (zkl_ctx_wait)");
    int st;
    const uint64_t N = table->N;
    if ((st = check_shape(ctx, D, N))) return st;
    if (D < 2 || D / ctx->nranks < 2)
        return set_err(ctx, ZKL_E_SHAPE, "Fiat-Shamir mode needs D >= 2 and D_local >= 2");
    if ((!seed && !preset) || !m_dev || !round_evals || !finals || !derived)
        return set_err(ctx, ZKL_E_ARG, "null argument");
    std::vector<zkl_fr> u1(kMaxRounds);
    for (auto& x : u1) { memset(&x, 0, sizeof(x)); x.w[0] = 1; }
    Plan p;
    make_plan(p, D, N, ctx->nranks, ctx->rank, true, u1.data(), true);
    const int P = ctx->nranks;
    fr* rank_sums = at<fr>(ctx, p.o_rank);   // P > 1: this rank's sums of the current round (5 fr)
    fr* gath = at<fr>(ctx, p.o_gath);        // P > 1: the ranks' sums of the current round, rank-major (P x 5 fr)
    if ((st = need_ws(ctx, p))) return st;
    const bool virt = S.limbs == nullptr;
    const bool keys_ok = ctx->prep_valid && ctx->prep_S == S.limbs && ctx->prep_n == p.Dp && ctx->prep_table == table;
    if (virt && !keys_ok)
        return set_err(ctx, ZKL_E_ARG, "S_local is virtual (NULL): it needs the keys of the preceding "
                                       "zkl_tlookup_prepare_pair on this context, table and D");
    if (virt && force_inversion) return set_err(ctx, ZKL_E_STATE, "internal: inversion fallback on a virtual S");
    if (!virt && (st = check_vec(ctx, S, p.Dp, "S_local"))) return st;
    if (A_out.limbs && (st = check_vec(ctx, A_out, p.Dp, "A_local_out"))) return st;
    if (B_out.limbs && (st = check_vec(ctx, B_out, N, "B_out"))) return st;
    cudaStream_t s = ctx->stream;
    ProofScalars* sc = at<ProofScalars>(ctx, p.o_sc);
    unsigned long long* err = at<unsigned long long>(ctx, p.o_err);
    RoundDesc* rounds = at<RoundDesc>(ctx, p.o_rounds);
    EqJob* jobs = at<EqJob>(ctx, p.o_jobs);
    fr* partials = at<fr>(ctx, p.o_part);
    fr* fin = at<fr>(ctx, p.o_fin);
    fr* tfin = at<fr>(ctx, p.o_tfin);
    fr* arena = at<fr>(ctx, p.o_arena);
    fr* tpart = at<fr>(ctx, p.o_tpart);
    FsState* fst = at<FsState>(ctx, p.o_fs);
    zkl_fr* dder = at<zkl_fr>(ctx, p.o_derived);
    ProofOut* out = at<ProofOut>(ctx, p.o_out);
    uint8_t* dseed = reinterpret_cast<uint8_t*>(at<zkl_fr>(ctx, p.o_chal));
    struct Staging {
        uint8_t seed[32];
        RoundDesc rounds[kMaxRounds];
        EqJob jobs[2 * kMaxRounds];
        zkl_fr pre[3 + kMaxRounds];
    };
    Staging* hs = reinterpret_cast<Staging*>((uint8_t*)ctx->host_out + sizeof(ProofOut));
    if (seed) memcpy(hs->seed, seed, 32);
    memcpy(hs->rounds, p.rd, sizeof(p.rd));
    memcpy(hs->jobs, p.jobs, sizeof(p.jobs));
    zkl_fr* dpre = at<zkl_fr>(ctx, p.o_chal) + 2;   // after the 32-byte seed slot
    if (preset) memcpy(hs->pre, preset, sizeof(zkl_fr) * (3 + p.d));
    if ((st = h2d_small(ctx, s, {{dseed, hs->seed}, {rounds, hs->rounds}, {jobs, hs->jobs}, {dpre, hs->pre}},
                        {sizeof(hs->seed), sizeof(hs->rounds), sizeof(hs->jobs),
                         preset ? sizeof(zkl_fr) * (3 + p.d) : (size_t)0})))
        return st;
    CUDA_TRY(ctx, cudaMemsetAsync(err, 0xff, 4 * sizeof(unsigned long long), s));
    if (preset)
        LAUNCH(ctx, k_fs_init_preset, 1, 1, 0, s, dpre, p.d, sc, fst, dder, p.pbits, p.rank);
    else
        LAUNCH(ctx, k_fs_init, 1, 32, 0, s, dseed, D, N, variant, p.d, sc, fst, dder, p.pbits, p.rank);
    LAUNCH(ctx, k_eq_fill, grid_for(p.arena, 256), 256, 0, s, jobs, p.njobs, p.arena, sc, arena);
    // ---- B = 1/(beta + T) and the table working vectors
    uint32_t* tB = at<uint32_t>(ctx, p.o_tB);
    uint32_t* tX = at<uint32_t>(ctx, p.o_tX);
    if (N >= (uint64_t)kInvTile) {
        if ((st = inv_forward(ctx, p.tinv, table->T, N, tB, sc, 0, err + 1, s, s, nullptr))) return st;
        if ((st = inv_backward0(ctx, p.tinv, table->T, N, tB, sc, nullptr, nullptr, nullptr, 0, s))) return st;
    } else {
        LAUNCH(ctx, k_add_beta, grid_for(N, 256), 256, 0, s, table->T, N, sc, tX, err + 1);
        const unsigned bt = (unsigned)std::min<uint64_t>(1024, std::max<uint64_t>(32, N));
        LAUNCH(ctx, k_batch_invert, 1, bt, 4 * bt * sizeof(fr), s, tX, N, (uint64_t)0, N, tB);
    }
    fr* wk = at<fr>(ctx, p.o_twk);
    fr *tcur = wk, *tnxt = wk + 4 * N;
    // the table's round-1 work needs m: with the async histogram still running it goes to the side stream, so the
    // D side (the gather) does not wait for m
    cudaStream_t ts = s;
    const bool tab_side = ctx->m_pending != 0;
    if (tab_side) {
        CUDA_TRY(ctx, cudaEventRecord(ctx->ev_b, s));
        CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->side, ctx->ev_b, 0));
        CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->side, ctx->ev_m, 0));
        ts = ctx->side;
    }
    LAUNCH(ctx, k_tab_init, grid_for(N, 256), 256, 0, ts, tB, table->T, m_dev, (const uint32_t*)nullptr, N, sc, p.d,
           p.n, variant, tcur, B_out.limbs);
    uint64_t tlen = N;
    if (p.n == 0) LAUNCH(ctx, k_tab_fin_copy, 1, 32, 0, ts, tcur, tfin);   // the table is fully bound from the start
    if (p.n >= 1) LAUNCH(ctx, k_tab_eval, p.tnb[0], 256, 0, ts, tcur, tlen, sc, variant, tpart);
    if (tab_side) CUDA_TRY(ctx, cudaEventRecord(ctx->ev_join, ts));
    // ---- round 1: A (gather through the prepared index, or inversion) + the round-1 sums
    uint32_t* Abuf = A_out.limbs ? A_out.limbs : at<uint32_t>(ctx, p.o_A);
    const bool gather = !p.small && !force_inversion;
    // round 2 gathers A, S from the keys again (unless the cooperative rounds start at round 2 and read round 1's)
    const bool r2_gather = gather && keys_ok && p.d >= 2 && !(p.fs_coop && p.kc == 2);
    const uint32_t* Sin = S.limbs;
    if (virt && !r2_gather) {   // D_local < 4096: the small path reads S itself
        uint32_t* Sv = at<uint32_t>(ctx, p.o_Sv);
        LAUNCH(ctx, k_s_from_keys, grid_for(p.Dp, 256), 256, 0, s, at<uint32_t>(ctx, p.o_keys), p.Dp, N, table->Taos,
               Sv);
        Sin = Sv;
    }
    int h01 = 1;
    if (gather) {
        LAUNCH(ctx, k_pack_tb, grid_for(N, 256), 256, 0, s, table->T, tB, N, at<uint4>(ctx, p.o_tBaos));
        TableView tv{table->T, table->Taos, table->slots, table->Skeys, table->N, table->slot_mask};
        if (keys_ok) {
            uint32_t* Aw = A_out.limbs ? A_out.limbs : (r2_gather ? nullptr : Abuf);
            const uint32_t* keys = at<uint32_t>(ctx, p.o_keys);
            const uint4* TB = at<uint4>(ctx, p.o_tBaos);
            const fr *elo1 = arena + p.rd[0].elo_off, *ehi1 = arena + p.rd[0].ehi_off;
            fr* part1 = partials + p.rd[0].part_base;
            const int tpc1 = r1_tiles_per_cta(p.ntiles);   // tiles per CTA (the per-CTA reductions amortised)
            const unsigned nb1 = (unsigned)(p.ntiles / tpc1);
            if (!virt && Aw)
                LAUNCH(ctx, (k_round1_keys<true, true>), nb1, kInvThreads, 0, s, S.limbs, p.Dp, keys, N, TB, Aw, elo1,
                       ehi1, part1, (int)p.ntiles, err + 2, tpc1);
            else if (!virt)
                LAUNCH(ctx, (k_round1_keys<true, false>), nb1, kInvThreads, 0, s, S.limbs, p.Dp, keys, N, TB, Aw, elo1,
                       ehi1, part1, (int)p.ntiles, err + 2, tpc1);
            else if (Aw)
                LAUNCH(ctx, (k_round1_keys<false, true>), nb1, kInvThreads, 0, s, Sin, p.Dp, keys, N, TB, Aw, elo1,
                       ehi1, part1, (int)p.ntiles, err + 2, tpc1);
            else
                LAUNCH(ctx, (k_round1_keys<false, false>), nb1, kInvThreads, 0, s, Sin, p.Dp, keys, N, TB, Aw, elo1,
                       ehi1, part1, (int)p.ntiles, err + 2, tpc1);
        } else
            LAUNCH(ctx, k_gather_round1, (unsigned)p.ntiles, kInvThreads, 0, s, S.limbs, p.Dp, tv,
                   at<uint4>(ctx, p.o_tBaos), Abuf, arena + p.rd[0].elo_off, arena + p.rd[0].ehi_off,
                   partials + p.rd[0].part_base, (int)p.ntiles, err + 2);
    } else if (!p.small) {
        for (int h = 0; h < p.nhalves; ++h)
            if ((st = inv_forward(ctx, p.inv[h], S.limbs, p.Dp, Abuf, sc, 0, err, s, s, nullptr))) return st;
        for (int h = 0; h < p.nhalves; ++h)
            if ((st = inv_backward0(ctx, p.inv[h], S.limbs, p.Dp, Abuf, sc, arena + p.rd[0].elo_off,
                                    arena + p.rd[0].ehi_off, partials + p.rd[0].part_base, (int)p.ntiles, s)))
                return st;
    } else {
        // small D: A by one batch inversion, round 1 summed directly from A and S
        LAUNCH(ctx, k_add_beta, grid_for(p.Dp, 256), 256, 0, s, Sin, p.Dp, sc, at<uint32_t>(ctx, p.o_small), err);
        const unsigned bt = (unsigned)std::min<uint64_t>(1024, std::max<uint64_t>(32, p.Dp));
        LAUNCH(ctx, k_batch_invert, 1, bt, 4 * bt * sizeof(fr), s, at<uint32_t>(ctx, p.o_small), p.Dp, (uint64_t)0,
               p.Dp, Abuf);
        const RoundDesc& r = p.rd[0];
        LAUNCH(ctx, (k_round<false, true>), r.nblocks, kRoundThreads, 0, s, Abuf, Sin, p.Dp, nullptr, nullptr, sc, 1,
               arena + r.elo_off, arena + r.ehi_off, (int)r.gbits, partials + r.part_base);
        h01 = 0;
    }
    if (tab_side) CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_join, 0));
    {
        // round 1 has one partial row per 4096-element tile: fold them to 32 rows with 32 CTAs first, so the
        // single-CTA derivation below (on the critical path of every round) does not sum 16K rows
        const fr* r1 = partials + p.rd[0].part_base;
        uint32_t r1rows = p.rd[0].nblocks;
        if (P > 1) {
            // the rank's round-1 sums, all-gathered: every rank derives g_1 and r_1 from the same global sums
            LAUNCH(ctx, k_rows_fold, 1, 256, 0, s, r1, r1rows, rank_sums, 1u);
            if ((st = zkl_dist_allgather(ctx, rank_sums, gath, kSlots * sizeof(fr)))) return st;
            LAUNCH(ctx, k_fs_round, 1, 256, 0, s, 1, p.d, p.n, variant, gath, (uint32_t)P, h01, tpart,
                   p.n >= 1 ? p.tnb[0] : 0u, tfin, sc, fst, out, dder, 0, err + 2, 1u, (uint32_t)kSlots, 0);
        } else {
            if (r1rows > 256) {
                fr* folded = at<fr>(ctx, p.o_rank);   // kMaxRounds x kSlots fr >= 5 x 32
                LAUNCH(ctx, k_rows_fold, 32, 256, 0, s, r1, r1rows, folded, 32u);
                r1 = folded;
                r1rows = 32;
            }
            LAUNCH(ctx, k_fs_round, 1, 256, 0, s, 1, p.d, p.n, variant, r1, r1rows, h01, tpart,
                   p.n >= 1 ? p.tnb[0] : 0u, tfin, sc, fst, out, dder, 0, err + 2, r1rows, 1u, 0);
        }
    }
    // ---- rounds 2..d
    const uint32_t *cA = Abuf, *cS = Sin;
    uint64_t len = p.Dp;
    bool coop_done = false;
    for (int k = 2; k <= p.d; ++k) {
        if (p.fs_coop && k == p.kc) {
            // rounds kc .. d: one cooperative launch, a grid barrier per round (csrc/coop.cuh)
            fr* cb = at<fr>(ctx, p.o_coop);
            GridBar* bar = reinterpret_cast<GridBar*>(cb + kChunkBits * 5 * 128 + 4 * kMaxRounds + 2 * 128);
            CUDA_TRY(ctx, cudaMemsetAsync(bar, 0, sizeof(GridBar), s));
            CoopFsArgs ca;
            ca.Ain = cA; ca.Sin = cS; ca.nin = len;
            ca.kc = p.kc; ca.d = p.d; ca.n = p.n; ca.variant = variant;
            ca.rounds = rounds; ca.arena = arena;
            ca.rows = cb; ca.tabbuf = cb + kChunkBits * 5 * 128; ca.chA = ca.tabbuf + 4 * kMaxRounds;
            ca.chS = ca.chA + 128;
            ca.tcur = tcur; ca.tlen = (int)tlen; ca.tfin = tfin; ca.fin = fin;
            ca.sc = sc; ca.st = fst; ca.out = out; ca.derived = dder; ca.bar = bar;
            const size_t smem = (2 * kChunk + 4 * kCoopTabMax) * sizeof(fr);
            LAUNCH_COOP(ctx, k_fs_rounds_coop, (unsigned)p.nchunks, kChunkThreads, smem, s, ca);
            coop_done = true;
            break;
        }
        const RoundDesc& r = p.rd[k - 1];
        const bool derive = !force_inversion && !r.direct_h1;
        uint32_t* nA = at<uint32_t>(ctx, (k & 1) == 0 ? p.o_A1 : p.o_A2);
        uint32_t* nS = at<uint32_t>(ctx, (k & 1) == 0 ? p.o_S1 : p.o_S2);
        // r_{k-1} is known: the table-side fold(k-1) + eval(k) and (derived rounds) the inversion of cl1 run on the
        // side stream while the D-side fold + eval of round k runs on the main stream
        const bool side = derive || k - 1 <= p.n;
        if (side) {
            CUDA_TRY(ctx, cudaEventRecord(ctx->ev_fork, s));
            CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
            if (derive) LAUNCH(ctx, k_fs_inv, 1, 32, 0, ctx->side, k, p.d, sc, fst);
            if (k - 1 <= p.n) {   // fold the table with r_{k-1}
                LAUNCH(ctx, k_tab_fold, grid_for(tlen / 2, 256, kMaxBlocks), 256, 0, ctx->side, tcur, tlen, tnxt, sc,
                       k - 1, tfin);
                fr* t = tcur; tcur = tnxt; tnxt = t;
                tlen /= 2;
            }
            if (k <= p.n) LAUNCH(ctx, k_tab_eval, p.tnb[k - 1], 256, 0, ctx->side, tcur, tlen, sc, variant, tpart);
            CUDA_TRY(ctx, cudaEventRecord(ctx->ev_join, ctx->side));
        }
        if (k == p.dl + 1) {
            // the local rounds are done: fold the rank's last pair with r_dl, all-gather the P folded (A, S), and run
            // the last log2 P rounds identically on every rank on the gathered vectors (replicated, no exchange)
            LAUNCH(ctx, k_fold_final, 1, 32, 0, s, cA, cS, len, sc, p.dl, fin);
            fr* g2 = gath + (size_t)P * kSlots;
            if ((st = zkl_dist_allgather(ctx, fin, g2, 2 * sizeof(fr)))) return st;
            uint32_t* gfin = reinterpret_cast<uint32_t*>(at<fr>(ctx, p.o_gfin));
            LAUNCH(ctx, k_pairs_to_soa, 1, 32, 0, s, g2, P, gfin);
            cA = gfin;
            cS = gfin + 8 * (size_t)P;
            len = (uint64_t)P;
            LAUNCH(ctx, (k_round<false, true>), r.nblocks, kRoundThreads, 0, s, cA, cS, len, nullptr, nullptr, sc, k,
                   arena + r.elo_off, arena + r.ehi_off, (int)r.gbits, partials + r.part_base);
        } else if (k == 2 && r2_gather) {
            const uint32_t* keys = at<uint32_t>(ctx, p.o_keys);
            const uint4* TB = at<uint4>(ctx, p.o_tBaos);
            if (derive)
                LAUNCH(ctx, (k_round<true, false, true>), r.nblocks, kRoundThreads, 0, s, nullptr, nullptr, len, nA,
                       nS, sc, k, arena + r.elo_off, arena + r.ehi_off, (int)r.gbits, partials + r.part_base, keys, TB);
            else
                LAUNCH(ctx, (k_round<true, true, true>), r.nblocks, kRoundThreads, 0, s, nullptr, nullptr, len, nA,
                       nS, sc, k, arena + r.elo_off, arena + r.ehi_off, (int)r.gbits, partials + r.part_base, keys, TB);
        } else if (derive)
            LAUNCH(ctx, (k_round<true, false>), r.nblocks, kRoundThreads, kRoundStageSmem, s, cA, cS, len, nA, nS, sc, k,
                   arena + r.elo_off, arena + r.ehi_off, (int)r.gbits, partials + r.part_base);
        else
            LAUNCH(ctx, (k_round<true, true>), r.nblocks, kRoundThreads, kRoundStageSmem, s, cA, cS, len, nA, nS, sc, k,
                   arena + r.elo_off, arena + r.ehi_off, (int)r.gbits, partials + r.part_base);
        if (k != p.dl + 1) {
            cA = nA; cS = nS;
            len /= 2;
        }
        if (side) CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_join, 0));
        // the round's partial rows (one per k_round CTA: thousands in the big rounds) are first folded to 32 rows by 32
        // CTAs, so the single-CTA derivation on the critical path of every round sums only those
        const fr* rows = partials + r.part_base;
        uint32_t nrows = r.nblocks;
        if (nrows > 32) {
            fr* folded = at<fr>(ctx, p.o_coop);   // scratch: the cooperative rounds use it only after this loop
            LAUNCH(ctx, k_rows_fold, 32, 256, 0, s, rows, nrows, folded, 32u);
            rows = folded;
            nrows = 32;
        }
        if (P > 1 && k <= p.dl) {   // a local round: its sums become global with one small all-gather
            LAUNCH(ctx, k_rows_fold, 1, 256, 0, s, rows, nrows, rank_sums, 1u);
            if ((st = zkl_dist_allgather(ctx, rank_sums, gath, kSlots * sizeof(fr)))) return st;
            LAUNCH(ctx, k_fs_round, 1, 256, 0, s, k, p.d, p.n, variant, gath, (uint32_t)P, 0, tpart,
                   k <= p.n ? p.tnb[k - 1] : 0u, tfin, sc, fst, out, dder, derive ? 1 : 0, err + 2, 1u,
                   (uint32_t)kSlots, (int)r.a1_derived);
        } else {
            LAUNCH(ctx, k_fs_round, 1, 256, 0, s, k, p.d, p.n, variant, rows, nrows, 0, tpart,
                   k <= p.n ? p.tnb[k - 1] : 0u, tfin, sc, fst, out, dder, derive ? 1 : 0, err + 2, nrows, 1u,
                   (int)r.a1_derived);
        }
    }
    if (!coop_done) {
        LAUNCH(ctx, k_fold_final, 1, 32, 0, s, cA, cS, len, sc, p.d, fin);
        if (p.n == p.d) LAUNCH(ctx, k_tab_fold, 1, 32, 0, s, tcur, tlen, tnxt, sc, p.d, tfin);
    }
    LAUNCH(ctx, k_fs_finish, 1, 32, 0, s, fin, tfin, out);
    if (P > 1 && (st = zkl_dist_min_u64_dev(ctx, err, 3))) return st;
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->host_out, out, sizeof(ProofOut), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(ctx, cudaMemcpyAsync((uint8_t*)ctx->host_out + offsetof(ProofOut, err_index), err,
                                  3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    zkl_fr* hder_w = reinterpret_cast<zkl_fr*>((uint8_t*)ctx->host_out + 32768);
    CUDA_TRY(ctx, cudaMemcpyAsync(hder_w, dder, sizeof(zkl_fr) * (3 + 2 * p.d), cudaMemcpyDeviceToHost, s));
    if (ctx->async_mode) {
        std::array<uint8_t, 32> sd;
        memcpy(sd.data(), seed, 32);
        const int d = p.d;
        ctx->pend_prove = 1;
        pending_of(ctx).push_back([=]() {
            ctx->pend_prove = 0;
            return proof_fs_collect(ctx, S, D, table, m_dev, sd.data(), variant, A_out, B_out, round_evals, finals,
                                    derived, err_index, gather, d);
        });
        return ZKL_OK;
    }
    if ((st = sync_stream(ctx))) return st;
    return proof_fs_collect(ctx, S, D, table, m_dev, seed, variant, A_out, B_out, round_evals, finals, derived,
                            err_index, gather, p.d);
}

int proof_fs_collect(zkl_ctx* ctx, zkl_vec S, uint64_t D, const zkl_table* table, const uint32_t* m_dev,
                     const uint8_t* seed, int variant, zkl_vec A_out, zkl_vec B_out, zkl_fr* round_evals,
                     zkl_final_evals* finals, zkl_fr* derived, int64_t* err_index, bool gather, int d) {
    const ProofOut* ho = reinterpret_cast<const ProofOut*>(ctx->host_out);
    const zkl_fr* hder = reinterpret_cast<const zkl_fr*>((uint8_t*)ctx->host_out + 32768);
    const unsigned long long* he = reinterpret_cast<const unsigned long long*>((const uint8_t*)ctx->host_out +
                                                                               offsetof(ProofOut, err_index));
    if (he[1] != ~0ull) {
        if (err_index) *err_index = (int64_t)he[1];
        return set_err(ctx, ZKL_E_DIV_ZERO_T, "beta + T_%llu = 0", he[1]);
    }
    if (gather && he[2] != ~0ull) {
        const int was_async = ctx->async_mode;
        ctx->async_mode = 0;
        const int st = run_proof_fs(ctx, S, D, table, m_dev, seed, variant, A_out, B_out, round_evals, finals,
                                    derived, err_index, true);
        ctx->async_mode = was_async;
        return st;
    }
    if (he[0] != ~0ull) {
        if (err_index) *err_index = (int64_t)he[0];
        return set_err(ctx, ZKL_E_DIV_ZERO_S, "beta + S_%llu = 0", he[0]);
    }
    memcpy(round_evals, ho->evals, sizeof(zkl_fr) * 4 * d);
    finals->A = ho->finals[0];
    finals->S = ho->finals[1];
    finals->B = ho->finals[2];
    finals->T = ho->finals[3];
    finals->m = ho->finals[4];
    memcpy(derived, hder, sizeof(zkl_fr) * (3 + 2 * d));
    return ZKL_OK;
}

// ------------------------------------------------------------------ matmul sumcheck
}  // namespace

// ====================================================================== ABI
extern "C" {

const char* zkl_strerror(int st) {
    switch (st) {
        case ZKL_OK: return "ok";
        case ZKL_E_ARG: return "bad argument";
        case ZKL_E_SHAPE: return "bad shape";
        case ZKL_E_NONCANONICAL: return "non-canonical field element";
        case ZKL_E_DUP_TABLE: return "duplicate table entry";
        case ZKL_E_NOT_IN_TABLE: return "lookup not in table";
        case ZKL_E_DIV_ZERO_T: return "division by zero (beta + T_j = 0)";
        case ZKL_E_DIV_ZERO_S: return "division by zero (beta + S_i = 0)";
        case ZKL_E_CUDA: return "CUDA error";
        case ZKL_E_NCCL: return "NCCL error";
        case ZKL_E_OOM: return "insufficient workspace";
        case ZKL_E_STATE: return "context poisoned";
        default: return "unknown status";
    }
}

static int ctx_create_common(int device, void* stream, zkl_ctx** out) {
    if (!out) return ZKL_E_ARG;
    *out = nullptr;
    zkl_ctx* c = (zkl_ctx*)calloc(1, sizeof(zkl_ctx));
    if (!c) return ZKL_E_OOM;
    c->device = device;
    c->stream = (cudaStream_t)stream;
    c->nranks = 1;
    if (cudaSetDevice(device) != cudaSuccess ||
        cudaDeviceGetStreamPriorityRange(&c->prio_lo, &c->prio_hi) != cudaSuccess ||
        cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, c->prio_hi) != cudaSuccess ||
        cudaStreamCreateWithPriority(&c->aux, cudaStreamNonBlocking, c->prio_hi) != cudaSuccess ||
        cudaStreamCreateWithPriority(&c->low, cudaStreamNonBlocking, c->prio_lo) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_keys, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_m, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_b, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_eq, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fwd[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fwd[1], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_mid[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_mid[1], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaMallocHost(&c->host_out, 1 << 16) != cudaSuccess || cudaMalloc(&c->dscratch, 4096) != cudaSuccess) {
        cudaGetLastError();
        free(c);
        return ZKL_E_CUDA;
    }
    // stream-ordered allocations (host-sourced import/export only) must not be trimmed at every sync
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    const size_t tail_smem = (2 * kTailMax + 4 * kTailThreads) * sizeof(fr) + 5 * (kTailThreads / 32) * sizeof(fr);
    cudaFuncSetAttribute(k_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tail_smem);
    cudaFuncSetAttribute(k_batch_invert, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 1024 * (int)sizeof(fr));
    cudaFuncSetAttribute(k_tab_chunk, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kTabChunk * (int)sizeof(fr));
    cudaFuncSetAttribute(k_round<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRoundStageSmem);
    cudaFuncSetAttribute(k_round<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRoundStageSmem);
    cudaFuncSetAttribute(k_mh_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMhSmem);
    cudaFuncSetAttribute(k_mh_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMhScatterSmem);
    cudaFuncSetAttribute(k_mh_lo, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMhSmem);
    cudaFuncSetAttribute(k_fs_rounds_coop, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)((2 * kChunk + 4 * kCoopTabMax) * sizeof(fr)));
    cudaFuncSetAttribute(k_chunk_rounds_coop, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(2 * kChunk * sizeof(fr)));
    *out = c;
    return ZKL_OK;
}

int zkl_ctx_create(int device, void* cuda_stream, zkl_ctx** out) { return ctx_create_common(device, cuda_stream, out); }

int zkl_nccl_unique_id(uint8_t id[128]) { return zkl_nccl_get_unique_id(id); }

int zkl_ctx_create_dist(int device, void* cuda_stream, const uint8_t nccl_id[128], int rank, int nranks,
                        zkl_ctx** out) {
    int st = ctx_create_common(device, cuda_stream, out);
    if (st) return st;
    if (nranks > 1) {
        st = zkl_nccl_init(*out, nccl_id, rank, nranks);
        if (st) {
            zkl_ctx_destroy(*out);
            *out = nullptr;
            return st;
        }
    }
    (*out)->rank = rank;
    (*out)->nranks = nranks;
    return ZKL_OK;
}

int zkl_group_create(int device, int nranks, uint64_t max_D_local, uint64_t max_N, zkl_group** out) {
    if (!out || nranks < 1) return ZKL_E_ARG;
    zkl_group* g = new (std::nothrow) zkl_group();
    if (!g) return ZKL_E_OOM;
    g->nranks = nranks;
    g->device = device;
    // largest block: m (N u32) or the round sums (kMaxRounds x kSlots fr)
    g->staging_bytes = (size_t)nranks * std::max<size_t>(4 * max_N, sizeof(fr) * kMaxRounds * kSlots) + 4096;
    (void)max_D_local;
    if (cudaSetDevice(device) != cudaSuccess || cudaMalloc(&g->staging, g->staging_bytes) != cudaSuccess) {
        cudaGetLastError();
        delete g;
        return ZKL_E_CUDA;
    }
    *out = g;
    return ZKL_OK;
}

void zkl_group_destroy(zkl_group* g) {
    if (!g) return;
    cudaSetDevice(g->device);
    cudaFree(g->staging);
    delete g;
}

int zkl_ctx_create_loopback(int device, void* cuda_stream, zkl_group* group, int rank, zkl_ctx** out) {
    if (!group || rank < 0 || rank >= group->nranks) return ZKL_E_ARG;
    int st = ctx_create_common(device, cuda_stream, out);
    if (st) return st;
    (*out)->group = group;
    (*out)->rank = rank;
    (*out)->nranks = group->nranks;
    return ZKL_OK;
}

int zkl_ctx_set_async(zkl_ctx* ctx, int on) {
    if (!ctx) return ZKL_E_ARG;
    // P > 1: allowed with NCCL (the prepare's histogram and its all-reduce go to the low-priority stream); the
    // loopback communicator synchronises the host inside every collective, so its prepare stays synchronous
    if (!on && (ctx->pend_prepare || ctx->pend_prove)) return set_err(ctx, ZKL_E_STATE, "pending work: zkl_ctx_wait first");
    ctx->async_mode = on ? 1 : 0;
    return ZKL_OK;
}

int zkl_ctx_wait(zkl_ctx* ctx) {
    if (!ctx) return ZKL_E_ARG;
    if (ctx->m_pending) {   // m (written on the low stream) is complete for the ctx stream from here on
        cudaStreamWaitEvent(ctx->stream, ctx->ev_m, 0);
        ctx->m_pending = 0;
    }
    int st = sync_stream(ctx);
    std::vector<std::function<int()>> work;
    if (ctx->pending) work.swap(pending_of(ctx));
    for (auto& f : work) {
        if (st == ZKL_OK) {
            st = f();
        } else {   // an earlier completion failed: later results are not delivered
            ctx->pend_prepare = ctx->pend_prove = 0;
            ctx->prep_valid = 0;
        }
    }
    return st;
}

void zkl_ctx_destroy(zkl_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->hs.table) zkl_table_destroy(c->hs.table);
    if (c->hs.buf) cudaFree(c->hs.buf);
    if (c->p1.table) zkl_table_destroy(c->p1.table);
    if (c->p1.buf) cudaFree(c->p1.buf);
    if (c->p1.hxws) cudaFree(c->p1.hxws);
    if (c->prof[0].a)
        for (int i = 0; i < 256; ++i) { cudaEventDestroy(c->prof[i].a); cudaEventDestroy(c->prof[i].b); }
    if (c->nccl_comm) zkl_nccl_destroy(c);
    cudaStreamSynchronize(c->side);
    cudaStreamSynchronize(c->aux);
    cudaStreamDestroy(c->side);
    cudaStreamDestroy(c->aux);
    cudaStreamDestroy(c->low);
    cudaEventDestroy(c->ev_keys);
    cudaEventDestroy(c->ev_m);
    cudaEventDestroy(c->ev_b);
    cudaEventDestroy(c->ev_eq);
    for (int i = 0; i < 2; ++i) { cudaEventDestroy(c->ev_fwd[i]); cudaEventDestroy(c->ev_mid[i]); }
    cudaEventDestroy(c->ev_fork);
    cudaEventDestroy(c->ev_join);
    cudaFreeHost(c->host_out);
    cudaFree(c->dscratch);
    delete static_cast<std::vector<std::function<int()>>*>(c->pending);
    free(c);
}

const char* zkl_last_error(const zkl_ctx* c) { return c ? c->last_error : "null ctx"; }

size_t zkl_workspace_bytes(uint64_t D_local, uint64_t N, int nranks) {
    if (!is_pow2(D_local) || !is_pow2(N) || nranks < 1) return 0;
    std::vector<zkl_fr> u(kMaxRounds);
    for (auto& x : u) { memset(&x, 0, sizeof(x)); x.w[0] = 1; }
    Plan p, q;
    make_plan(p, D_local * nranks, N, nranks, 0, true, u.data());
    make_plan(q, D_local * nranks, N, nranks, 0, false, u.data());
    return std::max(p.total, q.total);
}

int zkl_ctx_set_workspace(zkl_ctx* c, void* ptr, size_t bytes) {
    if (!c) return ZKL_E_ARG;
    if (((uintptr_t)ptr) & 255) return set_err(c, ZKL_E_ARG, "workspace must be 256-byte aligned");
    c->ws = (uint8_t*)ptr;
    c->ws_bytes = bytes;
    c->prep_valid = 0;   // the cached index-map keys lived in the old workspace
    return ZKL_OK;
}

uint64_t zkl_ctx_launch_count(const zkl_ctx* c) { return c ? c->launches : 0; }

int zkl_ctx_set_profiling(zkl_ctx* c, int on) {
    if (!c) return ZKL_E_ARG;
    if (on && !c->prof[0].a) {
        for (int i = 0; i < 256; ++i) {
            if (cudaEventCreate(&c->prof[i].a) != cudaSuccess || cudaEventCreate(&c->prof[i].b) != cudaSuccess)
                return ZKL_E_CUDA;
        }
    }
    c->profiling = on;
    c->nprof = 0;
    return ZKL_OK;
}

int zkl_ctx_profile_read(zkl_ctx* c, char* names, int name_len, float* ms, float* start_ms, int* stream_tag,
                         int cap) {
    if (!c) return -ZKL_E_ARG;
    int n = 0;
    for (int i = 0; i < c->nprof && n < cap; ++i, ++n) {
        float t = 0, t0 = 0;
        cudaEventSynchronize(c->prof[i].b);
        cudaEventElapsedTime(&t, c->prof[i].a, c->prof[i].b);
        cudaEventElapsedTime(&t0, c->prof[0].a, c->prof[i].a);
        ms[n] = t;
        if (start_ms) start_ms[n] = t0;
        if (stream_tag)
            stream_tag[n] = c->prof[i].stream == c->side ? 1
                            : c->prof[i].stream == c->aux ? 2
                            : c->prof[i].stream == c->low ? 3
                                                          : 0;
        snprintf(names + (size_t)n * name_len, name_len, "%s", c->prof[i].name);
    }
    c->nprof = 0;
    return n;
}

// ---------------------------------------------------------------- a1
int zkl_vec_import(zkl_ctx* ctx, const void* canon, int src_on_device, zkl_vec dst, int64_t* err_index) {
    int st;
    if ((st = check_ctx(ctx))) return st;
    if ((st = check_idle(ctx))) return st;
    if (err_index) *err_index = -1;
    if (!canon) return set_err(ctx, ZKL_E_ARG, "null source");
    if ((st = check_vec(ctx, dst, dst.n, "dst"))) return st;
    if (dst.n == 0) return ZKL_OK;
    const uint32_t* src = (const uint32_t*)canon;
    void* tmp = nullptr;
    if (!src_on_device) {
        CUDA_TRY(ctx, cudaMallocAsync(&tmp, 32 * dst.n, ctx->stream));
        CUDA_TRY(ctx, cudaMemcpyAsync(tmp, canon, 32 * dst.n, cudaMemcpyHostToDevice, ctx->stream));
        src = (const uint32_t*)tmp;
    }
    unsigned long long* err = reinterpret_cast<unsigned long long*>((uint8_t*)ctx->host_out + 60000);
    unsigned long long* derr = reinterpret_cast<unsigned long long*>(ctx->dscratch);
    CUDA_TRY(ctx, cudaMemsetAsync(derr, 0xff, sizeof(unsigned long long), ctx->stream));
    LAUNCH(ctx, k_import_canon, grid_for(dst.n, 256), 256, 0, ctx->stream, src, dst.n, dst.limbs, derr);
    CUDA_TRY(ctx, cudaMemcpyAsync(err, derr, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
    if (tmp) CUDA_TRY(ctx, cudaFreeAsync(tmp, ctx->stream));
    if ((st = sync_stream(ctx))) return st;
    if (*err != ~0ull) {
        if (err_index) *err_index = (int64_t)*err;
        return set_err(ctx, ZKL_E_NONCANONICAL, "element %llu >= r", *err);
    }
    return ZKL_OK;
}

int zkl_vec_import_i64(zkl_ctx* ctx, const int64_t* x, zkl_vec dst) {
    int st;
    if ((st = check_ctx(ctx))) return st;
    if (!x) return set_err(ctx, ZKL_E_ARG, "null source");
    if ((st = check_vec(ctx, dst, dst.n, "dst"))) return st;
    if (dst.n == 0) return ZKL_OK;
    LAUNCH(ctx, k_import_i64, grid_for(dst.n, 256), 256, 0, ctx->stream, x, dst.n, dst.limbs);
    return sync_stream(ctx);
}

int zkl_vec_import_pair(zkl_ctx* ctx, const int32_t* x, const int32_t* y, const zkl_fr* alpha_f, zkl_vec dst) {
    int st;
    if ((st = check_ctx(ctx))) return st;
    if ((st = check_idle(ctx))) return st;
    if (!x || !y || !alpha_f) return set_err(ctx, ZKL_E_ARG, "null argument");
    if ((st = check_vec(ctx, dst, dst.n, "dst"))) return st;
    if (dst.n == 0) return ZKL_OK;
    // alpha_f -> Montgomery on the device (one launch, no host arithmetic)
    fr* af = reinterpret_cast<fr*>(ctx->dscratch + 64);
    zkl_fr* staged = reinterpret_cast<zkl_fr*>((uint8_t*)ctx->host_out + 62000);
    *staged = *alpha_f;
    if ((st = h2d_small(ctx, ctx->stream, {{af, staged}}, {sizeof(fr)}))) return st;
    LAUNCH(ctx, k_import_canon, 1, 32, 0, ctx->stream, (const uint32_t*)af, 1, (uint32_t*)af,
           (unsigned long long*)nullptr);
    fr* consts = af + 1;
    LAUNCH(ctx, k_pair_consts, 1, 32, 0, ctx->stream, af, consts);
    LAUNCH(ctx, k_import_pair_dev, grid_for(dst.n, 256), 256, 0, ctx->stream, x, y, dst.n, consts, dst.limbs);
    return sync_stream(ctx);
}

int zkl_vec_export(zkl_ctx* ctx, zkl_vec src, void* canon, int dst_on_device) {
    int st;
    if ((st = check_ctx(ctx))) return st;
    if (!canon) return set_err(ctx, ZKL_E_ARG, "null destination");
    if ((st = check_vec(ctx, src, src.n, "src"))) return st;
    if (src.n == 0) return ZKL_OK;
    uint32_t* dst = (uint32_t*)canon;
    void* tmp = nullptr;
    if (!dst_on_device) {
        CUDA_TRY(ctx, cudaMallocAsync(&tmp, 32 * src.n, ctx->stream));
        dst = (uint32_t*)tmp;
    }
    LAUNCH(ctx, k_export, grid_for(src.n, 256), 256, 0, ctx->stream, src.limbs, src.n, dst);
    if (tmp) {
        CUDA_TRY(ctx, cudaMemcpyAsync(canon, tmp, 32 * src.n, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_TRY(ctx, cudaFreeAsync(tmp, ctx->stream));
    }
    return sync_stream(ctx);
}

// ---------------------------------------------------------------- a2
size_t zkl_table_bytes(uint64_t N) {
    if (!is_pow2(N)) return 0;
    uint64_t slots = std::max<uint64_t>(64, 4 * N);   // load factor <= 1/4
    return soa_bytes(N) + align_up(32 * N) + align_up(4 * slots) + align_up(32 * slots) + align_up(4 * N);
}

int zkl_table_create(zkl_ctx* ctx, zkl_vec T, void* mem, size_t mem_bytes, zkl_table** out, int64_t* err_index) {
    int st;
    if (err_index) *err_index = -1;
    if (!out) return ZKL_E_ARG;
    *out = nullptr;
    if ((st = check_ctx(ctx))) return st;
    if ((st = check_idle(ctx))) return st;
    if (!is_pow2(T.n)) return set_err(ctx, ZKL_E_SHAPE, "N=%llu is not a power of two", (unsigned long long)T.n);
    if ((st = check_vec(ctx, T, T.n, "T"))) return st;
    const uint64_t N = T.n;
    if (!mem || mem_bytes < zkl_table_bytes(N) || ((uintptr_t)mem & 255))
        return set_err(ctx, ZKL_E_OOM, "table memory: need %zu bytes, 256-byte aligned", zkl_table_bytes(N));
    zkl_table* t = (zkl_table*)calloc(1, sizeof(zkl_table));
    if (!t) return ZKL_E_OOM;
    const uint64_t nslots = std::max<uint64_t>(64, 4 * N);
    t->N = N;
    t->T = (uint32_t*)mem;
    t->Taos = (uint4*)((uint8_t*)mem + soa_bytes(N));
    t->slots = (uint32_t*)((uint8_t*)mem + soa_bytes(N) + align_up(32 * N));
    t->Skeys = (uint4*)((uint8_t*)mem + soa_bytes(N) + align_up(32 * N) + align_up(4 * nslots));
    t->ty = (int32_t*)((uint8_t*)mem + soa_bytes(N) + align_up(32 * N) + align_up(4 * nslots) + align_up(32 * nslots));
    t->has_pair = 0;
    t->nslots = nslots;
    t->slot_mask = (uint32_t)(nslots - 1);
    t->device = ctx->device;
    unsigned long long* derr = reinterpret_cast<unsigned long long*>(ctx->dscratch + 8);
    auto fail = [&](int code) { free(t); return code; };
    cudaMemsetAsync(derr, 0xff, sizeof(unsigned long long), ctx->stream);
    cudaMemsetAsync(t->slots, 0, 4 * nslots, ctx->stream);
    {
        auto launch_all = [&]() -> int {
            LAUNCH(ctx, k_table_copy, grid_for(N, 256), 256, 0, ctx->stream, T.limbs, N, t->T, t->Taos);
            LAUNCH(ctx, k_table_insert, grid_for(N, 256), 256, 0, ctx->stream, t->T, N, t->slots, t->slot_mask);
            LAUNCH(ctx, k_table_fill_keys, grid_for(nslots, 256), 256, 0, ctx->stream, t->T, N, t->slots, nslots,
                   t->Skeys);
            LAUNCH(ctx, k_table_dups, grid_for(N, 256), 256, 0, ctx->stream, t->T, t->Taos, N, t->slots, t->Skeys,
                   t->slot_mask, derr);
            return ZKL_OK;
        };
        if ((st = launch_all())) return fail(st);
    }
    unsigned long long* herr = reinterpret_cast<unsigned long long*>((uint8_t*)ctx->host_out + 60000);
    cudaMemcpyAsync(herr, derr, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream);
    if ((st = sync_stream(ctx))) return fail(st);
    if (*herr != ~0ull) {
        if (err_index) *err_index = (int64_t)*herr;
        set_err(ctx, ZKL_E_DUP_TABLE, "T_%llu repeats an earlier entry", *herr);
        return fail(ZKL_E_DUP_TABLE);
    }
    *out = t;
    return ZKL_OK;
}

void zkl_table_destroy(zkl_table* t) { free(t); }

int zkl_table_attach_pair(zkl_ctx* ctx, zkl_table* t, const int32_t* tx, const int32_t* ty, const zkl_fr* alpha_f) {
    int st;
    if ((st = check_ctx(ctx))) return st;
    if ((st = check_idle(ctx))) return st;
    if (!t || !tx || !ty || !alpha_f) return set_err(ctx, ZKL_E_ARG, "null argument");
    if (fr_ge_r_host(*alpha_f)) return set_err(ctx, ZKL_E_NONCANONICAL, "alpha_f is not canonical");
    t->has_pair = 0;
    const uint64_t N = t->N;
    fr* af = reinterpret_cast<fr*>(ctx->dscratch + 64);
    unsigned long long* bad = reinterpret_cast<unsigned long long*>(ctx->dscratch + 8);
    zkl_fr* staged = reinterpret_cast<zkl_fr*>((uint8_t*)ctx->host_out + 62000);
    *staged = *alpha_f;
    if ((st = h2d_small(ctx, ctx->stream, {{af, staged}}, {sizeof(fr)}))) return st;
    CUDA_TRY(ctx, cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), ctx->stream));
    LAUNCH(ctx, k_import_canon, 1, 32, 0, ctx->stream, (const uint32_t*)af, 1, (uint32_t*)af,
           (unsigned long long*)nullptr);
    LAUNCH(ctx, k_pair_consts, 1, 32, 0, ctx->stream, af, af + 1);
    LAUNCH(ctx, k_table_check_pair, grid_for(N, 256), 256, 0, ctx->stream, tx, ty, N, af + 1, t->T, t->ty, bad);
    unsigned long long* hb = reinterpret_cast<unsigned long long*>((uint8_t*)ctx->host_out + 60000);
    int32_t* hx0 = reinterpret_cast<int32_t*>((uint8_t*)ctx->host_out + 60016);
    CUDA_TRY(ctx, cudaMemcpyAsync(hb, bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaMemcpyAsync(hx0, tx, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    if ((st = sync_stream(ctx))) return st;
    if (*hb != ~0ull)
        return set_err(ctx, ZKL_E_ARG, "not a pair-range table at entry %llu (tx not x0 + j, or T_j != tx_j + alpha ty_j)",
                       *hb);
    t->x0 = *hx0;
    t->alpha = *alpha_f;
    t->has_pair = 1;
    return ZKL_OK;
}

// ---------------------------------------------------------------- a3
// Shared body of the two prepare entry points.  pair != nullptr: x, y (int32) are imported into S first,
// fused with the index map.
struct PairIn {
    const int32_t* x;
    const int32_t* y;
    const zkl_fr* alpha_f;
};

struct PrepArgs {
    zkl_vec S;
    uint64_t D;
    const zkl_table* T;
    uint32_t* m_dev;
    int64_t* err_index;
    bool has_pair;
    PairIn pair;
    zkl_fr alpha;   // owned copy (PairIn.alpha_f may point to caller memory that is gone at completion)
};

static int prepare_collect(zkl_ctx* ctx, const PrepArgs& a, uint64_t Dp, bool range_path);
static int prepare_impl(zkl_ctx* ctx, zkl_vec S, uint64_t D, const zkl_table* T, uint32_t* m_dev, int64_t* err_index,
                        const PairIn* pair, bool force_hash = false);

static int prepare_impl(zkl_ctx* ctx, zkl_vec S, uint64_t D, const zkl_table* T, uint32_t* m_dev, int64_t* err_index,
                        const PairIn* pair, bool force_hash) {
    int st;
    if (err_index) *err_index = -1;
    if ((st = check_ctx(ctx))) return st;
    if (ctx->async_mode && ctx->pend_prepare)
        return set_err(ctx, ZKL_E_STATE, "a prepare is already pending (zkl_ctx_wait)");
    if (!T || !m_dev) return set_err(ctx, ZKL_E_ARG, "null argument");
    if ((st = check_shape(ctx, D, T->N))) return st;
    Plan p;
    std::vector<zkl_fr> u(kMaxRounds);
    for (auto& x : u) { memset(&x, 0, sizeof(x)); x.w[0] = 1; }
    make_plan(p, D, T->N, ctx->nranks, ctx->rank, true, u.data());
    if ((st = need_ws(ctx, p))) return st;
    // prepare_pair may leave S virtual (S_local_out.limbs == NULL): only the keys are kept, S_i = T_key(i)
    if ((!pair || S.limbs) && (st = check_vec(ctx, S, p.Dp, "S_local"))) return st;
    ctx->prep_valid = 0;
    unsigned long long* err = at<unsigned long long>(ctx, p.o_err);
    uint32_t* rows = at<uint32_t>(ctx, p.o_hist);
    CUDA_TRY(ctx, cudaMemsetAsync(err, 0xff, 2 * sizeof(unsigned long long), ctx->stream));   // [0] NOT_IN, [1] range miss
    TableView tv{T->T, T->Taos, T->slots, T->Skeys, T->N, T->slot_mask};
    uint32_t* keys = at<uint32_t>(ctx, p.o_keys);
    bool range_path = false;
    if (pair) {
        if (!pair->x || !pair->y || !pair->alpha_f) return set_err(ctx, ZKL_E_ARG, "null argument");
        fr* af = reinterpret_cast<fr*>(ctx->dscratch + 64);
        zkl_fr* staged = reinterpret_cast<zkl_fr*>((uint8_t*)ctx->host_out + 62000);
        *staged = *pair->alpha_f;
        if ((st = h2d_small(ctx, ctx->stream, {{af, staged}}, {sizeof(fr)}))) return st;
        LAUNCH(ctx, k_import_canon, 1, 32, 0, ctx->stream, (const uint32_t*)af, 1, (uint32_t*)af,
               (unsigned long long*)nullptr);
        LAUNCH(ctx, k_pair_consts, 1, 32, 0, ctx->stream, af, af + 1);
        range_path = !force_hash && T->has_pair && memcmp(&T->alpha, pair->alpha_f, sizeof(zkl_fr)) == 0;
        if (range_path)   // the table's x column is a range: index x - x0, checked against ty (no hash probe)
            LAUNCH(ctx, k_import_pair_range, grid_for(p.Dp, 256, kSMs * 32), 256, 0, ctx->stream, pair->x, pair->y,
                   p.Dp, af + 1, S.limbs, T->x0, T->ty, T->N, keys, err + 1);
        else
            LAUNCH(ctx, k_import_pair_index, grid_for(p.Dp, 256, kSMs * 32), 256, 0, ctx->stream, pair->x, pair->y,
                   p.Dp, af + 1, S.limbs, (uint64_t)ctx->rank * p.Dp, tv, keys, err);
    } else {
        LAUNCH(ctx, k_index_map, grid_for(p.Dp, 256, kSMs * 32), 256, 0, ctx->stream, S.limbs, p.Dp,
               (uint64_t)ctx->rank * p.Dp, tv, keys, err);
    }
    // key bits: n (+1 for the sentinel of a partial tile when D_local < 4096)
    const int key_bits = std::max(1, p.n + (p.Dp < (uint64_t)kHistTile ? 1 : 0));
    // async mode (single rank): the histogram runs on the low-priority stream, overlapping the proof that follows
    // (which needs m only for the table side: it waits for ev_m there; zkl_ctx_wait orders the ctx stream after it)
    const bool hist_low = ctx->async_mode && !ctx->group;
    cudaStream_t hs = ctx->stream;
    if (hist_low) {
        CUDA_TRY(ctx, cudaEventRecord(ctx->ev_keys, ctx->stream));
        CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->low, ctx->ev_keys, 0));
        hs = ctx->low;
    }
    if (p.n <= 16) {
        // N <= 2^16: the atomic-free two-digit counting passes (csrc/mhist.cuh)
        const MhLayout l = mh_layout(p.Dp);
        uint8_t* wsh = reinterpret_cast<uint8_t*>(rows);
        uint32_t* tot = reinterpret_cast<uint32_t*>(wsh + l.tot);
        uint32_t* rel = reinterpret_cast<uint32_t*>(wsh + l.rel);
        uint32_t* total = reinterpret_cast<uint32_t*>(wsh + l.total);
        uint32_t* partial = reinterpret_cast<uint32_t*>(wsh + l.partial);
        const unsigned C = (unsigned)mh_chunks(p.Dp);
        const bool two = p.n > 8;
        LAUNCH(ctx, k_mh_count, C, kMhThreads, kMhSmem, hs, keys, p.Dp, two ? 8 : 0, tot);
        LAUNCH(ctx, k_mh_scan, kMhBins, 256, 0, hs, tot, C, two ? rel : nullptr, total, two ? nullptr : m_dev,
               (uint32_t)T->N);
        if (two) {
            LAUNCH(ctx, k_mh_scatter, C, kMhThreads, kMhScatterSmem, hs, keys, p.Dp, tot, rel, total, wsh + l.out);
            LAUNCH(ctx, k_mh_lo, C + kMhBins, kMhThreads, kMhSmem, hs, wsh + l.out, total, m_dev, partial);
            LAUNCH(ctx, k_mh_fix, (unsigned)(T->N >> 8), kMhThreads, 0, hs, total, partial, m_dev);
        }
    } else {
        // in the background a few CTAs suffice (the proof's kernels keep the rest of the GPU)
        const int hrows = hist_low ? std::min(p.hist_rows, kHistAsyncRows) : p.hist_rows;
        LAUNCH(ctx, k_hist_count, hrows, kHistThreads, 0, hs, keys, p.Dp, (uint32_t)T->N, rows, key_bits);
        LAUNCH(ctx, k_hist_colsum, grid_for(T->N, 256), 256, 0, hs, rows, hrows, T->N, m_dev);
    }
    unsigned long long* herr = reinterpret_cast<unsigned long long*>((uint8_t*)ctx->host_out + 60000);
    {
        // the collectives follow the histogram on its stream (NCCL calls of one communicator stay in one order)
        cudaStream_t cs = hist_low ? ctx->low : ctx->stream;
        cudaStream_t main_s = ctx->stream;
        ctx->stream = cs;   // the dist helpers enqueue on ctx->stream
        int rc = ZKL_OK;
        if (ctx->nranks > 1) rc = zkl_dist_allreduce_u32(ctx, m_dev, T->N);
        if (!rc && ctx->nranks > 1) rc = zkl_dist_min_u64_dev(ctx, err, 2);   // NOT_IN_TABLE index, range miss
        ctx->stream = main_s;
        if (rc) return rc;
        CUDA_TRY(ctx, cudaMemcpyAsync(herr, err, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, cs));
    }
    if (hist_low) {
        CUDA_TRY(ctx, cudaEventRecord(ctx->ev_m, ctx->low));
        ctx->m_pending = 1;
    }
    PrepArgs pa;
    memset(&pa, 0, sizeof(pa));
    pa.S = S; pa.D = D; pa.T = T; pa.m_dev = m_dev; pa.err_index = err_index;
    if (pair) {
        pa.has_pair = true;
        pa.pair = *pair;
        pa.alpha = *pair->alpha_f;
        pa.pair.alpha_f = nullptr;
    }
    if (ctx->async_mode) {
        // the keys are valid for a proof enqueued after this (the completion below clears them on error)
        ctx->prep_valid = 1;
        ctx->prep_S = S.limbs;
        ctx->prep_n = p.Dp;
        ctx->prep_table = T;
        ctx->pend_prepare = 1;
        const uint64_t Dp = p.Dp;
        pending_of(ctx).push_back([ctx, pa, Dp, range_path]() {
            ctx->pend_prepare = 0;
            return prepare_collect(ctx, pa, Dp, range_path);
        });
        return ZKL_OK;
    }
    if ((st = sync_stream(ctx))) return st;
    return prepare_collect(ctx, pa, p.Dp, range_path);
}

static int prepare_collect(zkl_ctx* ctx, const PrepArgs& a, uint64_t Dp, bool range_path) {
    const unsigned long long* he = reinterpret_cast<const unsigned long long*>((const uint8_t*)ctx->host_out + 60000);
    const unsigned long long e = he[0], miss = he[1];   // already min over ranks (device-side all-reduce)
    if (range_path && miss != ~0ull) {
        // some (x, y) is not (x0 + j, ty_j): redo with the exact hash index (NOT_IN_TABLE, or an entry that a
        // special alpha made equal), synchronously
        PairIn pin = a.pair;
        pin.alpha_f = &a.alpha;
        const int was_async = ctx->async_mode;
        ctx->async_mode = 0;
        const int st = prepare_impl(ctx, a.S, a.D, a.T, a.m_dev, a.err_index, &pin, true);
        ctx->async_mode = was_async;
        return st;
    }
    zkl_vec S = a.S;
    const zkl_table* T = a.T;
    int64_t* err_index = a.err_index;
    if (e != ~0ull) {
        if (err_index) *err_index = (int64_t)e;
        ctx->prep_valid = 0;
        return set_err(ctx, ZKL_E_NOT_IN_TABLE, "S_%llu is not in T", e);
    }
    ctx->prep_valid = 1;
    ctx->prep_S = S.limbs;   // the index-map keys in the workspace belong to this S (or a virtual S) and table
    ctx->prep_n = Dp;
    ctx->prep_table = T;
    return ZKL_OK;
}

int zkl_tlookup_prepare(zkl_ctx* ctx, zkl_vec S, uint64_t D, const zkl_table* T, uint32_t* m_dev, int64_t* err_index) {
    return prepare_impl(ctx, S, D, T, m_dev, err_index, nullptr);
}

int zkl_tlookup_prepare_pair(zkl_ctx* ctx, const int32_t* x_dev, const int32_t* y_dev, const zkl_fr* alpha_f,
                             uint64_t D, const zkl_table* T, zkl_vec S_local_out, uint32_t* m_dev, int64_t* err_index) {
    PairIn pin{x_dev, y_dev, alpha_f};
    return prepare_impl(ctx, S_local_out, D, T, m_dev, err_index, &pin);
}

// ---------------------------------------------------------------- a4-a9
int zkl_tlookup_prove(zkl_ctx* ctx, zkl_vec S, uint64_t D, const zkl_table* T, const uint32_t* m_dev,
                      const zkl_challenges* ch, zkl_variant variant, zkl_vec A_out, zkl_vec B_out,
                      zkl_fr* round_evals, zkl_final_evals* finals, int64_t* err_index) {
    int st;
    if ((st = check_ctx(ctx))) return st;
    if (!T) return set_err(ctx, ZKL_E_ARG, "null table");
    ProveArgs a;
    memset(&a, 0, sizeof(a));
    a.prove_mode = true;
    a.S = S;
    a.A_out = A_out;
    a.B_out = B_out;
    a.table = T;
    a.m_dev = m_dev;
    a.ch = ch;
    a.variant = variant;
    return run_proof(ctx, D, a, round_evals, finals, err_index);
}

int zkl_tlookup_prove_pair_host(zkl_ctx* ctx, const int32_t* x_host, const int32_t* y_host, uint64_t D,
                                const int32_t* tx_host, const int32_t* ty_host, uint64_t N, const zkl_fr* alpha_f,
                                const zkl_challenges* ch, zkl_variant variant, zkl_fr* round_evals,
                                zkl_final_evals* finals, uint32_t* m_out, int64_t* err_index) {
    int st;
    if (err_index) *err_index = -1;
    if ((st = check_ctx(ctx))) return st;
    if ((st = check_idle(ctx))) return st;
    if (ctx->async_mode) return set_err(ctx, ZKL_E_STATE, "zkl_tlookup_prove_pair_host: synchronous calls only");
    if (!x_host || !y_host || !tx_host || !ty_host || !alpha_f) return set_err(ctx, ZKL_E_ARG, "null argument");
    if ((st = check_shape(ctx, D, N))) return st;
    const uint64_t Dp = D / ctx->nranks;
    // owned device buffers: x, y (Dp int32), tx, ty (N int32), T (SoA, N), table memory, m (N u32)
    const size_t o_x = 0, o_y = align_up(4 * Dp), o_tx = o_y + align_up(4 * Dp), o_ty = o_tx + align_up(4 * N),
                 o_T = o_ty + align_up(4 * N), o_tab = o_T + soa_bytes(N), o_m = o_tab + align_up(zkl_table_bytes(N)),
                 total = o_m + align_up(4 * N);
    if (ctx->hs.bytes < total) {
        if (ctx->hs.table) { zkl_table_destroy(ctx->hs.table); ctx->hs.table = nullptr; }
        if (ctx->hs.buf) { CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream)); cudaFree(ctx->hs.buf); ctx->hs.buf = nullptr; }
        ctx->hs.bytes = 0;
        CUDA_TRY(ctx, cudaMalloc(&ctx->hs.buf, total));
        ctx->hs.bytes = total;
    }
    uint8_t* b = reinterpret_cast<uint8_t*>(ctx->hs.buf);
    int32_t *xd = reinterpret_cast<int32_t*>(b + o_x), *yd = reinterpret_cast<int32_t*>(b + o_y);
    int32_t *txd = reinterpret_cast<int32_t*>(b + o_tx), *tyd = reinterpret_cast<int32_t*>(b + o_ty);
    uint32_t* md = reinterpret_cast<uint32_t*>(b + o_m);
    CUDA_TRY(ctx, cudaMemcpyAsync(xd, x_host, 4 * Dp, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(ctx, cudaMemcpyAsync(yd, y_host, 4 * Dp, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(ctx, cudaMemcpyAsync(txd, tx_host, 4 * N, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(ctx, cudaMemcpyAsync(tyd, ty_host, 4 * N, cudaMemcpyHostToDevice, ctx->stream));
    zkl_vec T{reinterpret_cast<uint32_t*>(b + o_T), N};
    if ((st = zkl_vec_import_pair(ctx, txd, tyd, alpha_f, T))) return st;
    if (ctx->hs.table) { zkl_table_destroy(ctx->hs.table); ctx->hs.table = nullptr; }
    if ((st = zkl_table_create(ctx, T, b + o_tab, zkl_table_bytes(N), &ctx->hs.table, err_index))) return st;
    if ((st = zkl_table_attach_pair(ctx, ctx->hs.table, txd, tyd, alpha_f))) return st;
    zkl_vec Sv{nullptr, Dp};
    if ((st = zkl_tlookup_prepare_pair(ctx, xd, yd, alpha_f, D, ctx->hs.table, Sv, md, err_index))) return st;
    if ((st = zkl_tlookup_prove(ctx, Sv, D, ctx->hs.table, md, ch, variant, zkl_vec{nullptr, Dp}, zkl_vec{nullptr, N},
                                round_evals, finals, err_index)))
        return st;
    if (m_out) {
        CUDA_TRY(ctx, cudaMemcpyAsync(m_out, md, 4 * N, cudaMemcpyDeviceToHost, ctx->stream));
        return sync_stream(ctx);
    }
    return ZKL_OK;
}

// ---------------------------------------------------------------- Protocol 1 with its commitments
namespace {

// the Protocol-1 transcript on the host (oracle/protocol1.py is the verifier's side)
struct P1Transcript {
    uint8_t h[32];
    void absorb_points(const char* label, const zkl_g1* C, uint64_t n) {
        Sha256 sh;
        sh.update(h, 32);
        sh.update(label, strlen(label));
        const uint32_t cnt = (uint32_t)n;
        uint8_t le[4] = {(uint8_t)cnt, (uint8_t)(cnt >> 8), (uint8_t)(cnt >> 16), (uint8_t)(cnt >> 24)};
        sh.update(le, 4);
        for (uint64_t i = 0; i < n; ++i) {
            uint8_t b[97];
            for (int w = 0; w < 12; ++w)
                for (int k = 0; k < 4; ++k) {
                    b[4 * w + k] = C[i].infinity ? 0 : (uint8_t)(C[i].x[w] >> (8 * k));
                    b[48 + 4 * w + k] = C[i].infinity ? 0 : (uint8_t)(C[i].y[w] >> (8 * k));
                }
            b[96] = C[i].infinity ? 1 : 0;
            sh.update(b, 97);
        }
        sh.final(h);
    }
    zkl_fr chal(const char* label, uint32_t i) const {
        Sha256 sh;
        sh.update(h, 32);
        sh.update(label, strlen(label));
        uint8_t le[4] = {(uint8_t)i, (uint8_t)(i >> 8), (uint8_t)(i >> 16), (uint8_t)(i >> 24)};
        sh.update(le, 4);
        uint8_t dg[32];
        sh.final(dg);
        zkl_fr z;
        for (int w = 0; w < 8; ++w)
            z.w[w] = (uint32_t)dg[4 * w] | ((uint32_t)dg[4 * w + 1] << 8) | ((uint32_t)dg[4 * w + 2] << 16) |
                     ((uint32_t)dg[4 * w + 3] << 24);
        static const uint32_t rl[8] = {0x00000001u, 0xffffffffu, 0xfffe5bfeu, 0x53bda402u,
                                       0x09a1d805u, 0x3339d808u, 0x299d7d48u, 0x73eda753u};
        while (fr_ge_r_host(z)) {   // a digest < 2^256 < 3r: at most two subtractions of r
            uint64_t bw = 0;
            for (int w = 0; w < 8; ++w) {
                const uint64_t d = (uint64_t)z.w[w] - rl[w] - bw;
                z.w[w] = (uint32_t)d;
                bw = (d >> 63) & 1;
            }
        }
        return z;
    }
};

// the Hyrax steps run in the context's own Hyrax workspace (they clear the prepared-keys flag: restored after)
struct HxScope {
    zkl_ctx* c;
    uint8_t* ws;
    size_t bytes;
    int prep;
    HxScope(zkl_ctx* ctx) : c(ctx), ws(ctx->ws), bytes(ctx->ws_bytes), prep(ctx->prep_valid) {
        c->ws = (uint8_t*)c->p1.hxws;
        c->ws_bytes = c->p1.hxbytes;
    }
    ~HxScope() {
        c->ws = ws;
        c->ws_bytes = bytes;
        c->prep_valid = prep;
    }
};

}  // namespace

int zkl_tlookup_prove_p1(zkl_ctx* ctx, const void* pp, uint64_t cols, const int32_t* x, const int32_t* y, uint64_t D,
                         const int32_t* tx, const int32_t* ty, uint64_t N, const uint8_t seed[32], zkl_variant variant,
                         zkl_p1_proof* out) {
    int st;
    if ((st = check_ctx(ctx))) return st;
    if ((st = check_idle(ctx))) return st;
    if (ctx->async_mode || ctx->nranks != 1)
        return set_err(ctx, ZKL_E_STATE, "zkl_tlookup_prove_p1: synchronous, single-rank calls only");
    if (!pp || !x || !y || !tx || !ty || !seed || !out || !out->C_X || !out->C_Y || !out->C_TX || !out->C_TY ||
        !out->C_m || !out->C_A || !out->C_B || !out->round_evals || !out->derived || !out->w_A || !out->w_X ||
        !out->w_Y || !out->w_TX || !out->w_TY || !out->w_m || !out->w_B)
        return set_err(ctx, ZKL_E_ARG, "null argument");
    if ((st = check_shape(ctx, D, N))) return st;
    if (!is_pow2(cols) || cols > N) return set_err(ctx, ZKL_E_SHAPE, "cols must be a power of two dividing N");
    const int d = ilog2(D), n = ilog2(N);
    // owned device memory: X, Y, A (D), TX, TY, T, m_fr, B (N) as SoA vectors, w (cols), the table, m (u32)
    const size_t o_X = 0, o_Y = o_X + soa_bytes(D), o_A = o_Y + soa_bytes(D), o_TX = o_A + soa_bytes(D),
                 o_TY = o_TX + soa_bytes(N), o_T = o_TY + soa_bytes(N), o_mf = o_T + soa_bytes(N),
                 o_B = o_mf + soa_bytes(N), o_w = o_B + soa_bytes(N), o_tab = o_w + soa_bytes(cols),
                 o_m = o_tab + align_up(zkl_table_bytes(N)), total = o_m + align_up(4 * N);
    const size_t hxb = zkl_hyrax_workspace_bytes(D, cols);
    if (ctx->p1.bytes < total || ctx->p1.hxbytes < hxb) {
        CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        if (ctx->p1.table) { zkl_table_destroy(ctx->p1.table); ctx->p1.table = nullptr; }
        if (ctx->p1.buf) cudaFree(ctx->p1.buf);
        if (ctx->p1.hxws) cudaFree(ctx->p1.hxws);
        ctx->p1.buf = ctx->p1.hxws = nullptr;
        ctx->p1.bytes = ctx->p1.hxbytes = 0;
        CUDA_TRY(ctx, cudaMalloc(&ctx->p1.buf, total));
        CUDA_TRY(ctx, cudaMalloc(&ctx->p1.hxws, hxb));
        ctx->p1.bytes = total;
        ctx->p1.hxbytes = hxb;
    }
    uint8_t* b = reinterpret_cast<uint8_t*>(ctx->p1.buf);
    auto vec = [&](size_t o, uint64_t len) { return zkl_vec{reinterpret_cast<uint32_t*>(b + o), len}; };
    const zkl_vec X = vec(o_X, D), Y = vec(o_Y, D), A = vec(o_A, D), TX = vec(o_TX, N), TY = vec(o_TY, N),
                  T = vec(o_T, N), Mf = vec(o_mf, N), B = vec(o_B, N), Wv = vec(o_w, cols);
    uint32_t* md = reinterpret_cast<uint32_t*>(b + o_m);
    cudaStream_t s = ctx->stream;
    LAUNCH(ctx, k_import_i32, grid_for(D, 256), 256, 0, s, x, D, 0, X.limbs);
    LAUNCH(ctx, k_import_i32, grid_for(D, 256), 256, 0, s, y, D, 0, Y.limbs);
    LAUNCH(ctx, k_import_i32, grid_for(N, 256), 256, 0, s, tx, N, 0, TX.limbs);
    LAUNCH(ctx, k_import_i32, grid_for(N, 256), 256, 0, s, ty, N, 0, TY.limbs);
    // tlookup-Setup and the lookups' commitments, then alpha_f
    P1Transcript tr;
    {
        Sha256 sh;
        sh.update("zkl-p1-v1", 9);
        sh.update(seed, 32);
        uint8_t le[8];
        for (int i = 0; i < 8; ++i) le[i] = (uint8_t)(D >> (8 * i));
        sh.update(le, 8);
        for (int i = 0; i < 8; ++i) le[i] = (uint8_t)(N >> (8 * i));
        sh.update(le, 8);
        const uint32_t vv = (uint32_t)variant;
        uint8_t l4[4] = {(uint8_t)vv, (uint8_t)(vv >> 8), (uint8_t)(vv >> 16), (uint8_t)(vv >> 24)};
        sh.update(l4, 4);
        for (int i = 0; i < 8; ++i) le[i] = (uint8_t)(cols >> (8 * i));
        sh.update(le, 8);
        sh.final(tr.h);
    }
    const uint64_t rD = D / cols, rN = N / cols;
    {
        HxScope hx(ctx);
        if ((st = zkl_hyrax_commit(ctx, pp, cols, TX, N, nullptr, out->C_TX))) return st;
        if ((st = zkl_hyrax_commit(ctx, pp, cols, TY, N, nullptr, out->C_TY))) return st;
        if ((st = zkl_hyrax_commit(ctx, pp, cols, X, D, nullptr, out->C_X))) return st;
        if ((st = zkl_hyrax_commit(ctx, pp, cols, Y, D, nullptr, out->C_Y))) return st;
    }
    tr.absorb_points("TX", out->C_TX, rN);
    tr.absorb_points("TY", out->C_TY, rN);
    tr.absorb_points("X", out->C_X, rD);
    tr.absorb_points("Y", out->C_Y, rD);
    const zkl_fr af = tr.chal("alpha_f", 0);
    out->alpha_f = af;
    // T = T_X + alpha_f T_Y, its index, and tlookup-Prep with a virtual S = X + alpha_f Y; then [m] and beta
    if ((st = zkl_vec_import_pair(ctx, tx, ty, &af, T))) return st;
    if (ctx->p1.table) { zkl_table_destroy(ctx->p1.table); ctx->p1.table = nullptr; }
    int64_t ei = -1;
    if ((st = zkl_table_create(ctx, T, b + o_tab, zkl_table_bytes(N), &ctx->p1.table, &ei))) return st;
    if ((st = zkl_table_attach_pair(ctx, ctx->p1.table, tx, ty, &af))) return st;
    const zkl_vec Sv{nullptr, D};
    if ((st = zkl_tlookup_prepare_pair(ctx, x, y, &af, D, ctx->p1.table, Sv, md, &ei))) return st;
    LAUNCH(ctx, k_import_i32, grid_for(N, 256), 256, 0, s, reinterpret_cast<const int32_t*>(md), N, 1, Mf.limbs);
    {
        HxScope hx(ctx);
        if ((st = zkl_hyrax_commit(ctx, pp, cols, Mf, N, nullptr, out->C_m))) return st;
    }
    tr.absorb_points("m", out->C_m, rN);
    const zkl_fr beta = tr.chal("beta", 0);
    // A = 1/(beta + S), B (the variant's): the explicit-challenge prove with this beta writes both
    {
        std::vector<zkl_fr> zeros((size_t)d), ev((size_t)4 * d);
        for (auto& z : zeros) memset(&z, 0, sizeof(z));
        zkl_fr one;
        memset(&one, 0, sizeof(one));
        one.w[0] = 1;
        zkl_challenges ch0{beta, one, one, zeros.data(), zeros.data()};
        zkl_final_evals f0;
        if ((st = zkl_tlookup_prove(ctx, Sv, D, ctx->p1.table, md, &ch0, variant, A, B, ev.data(), &f0, &ei)))
            return st;
    }
    {
        HxScope hx(ctx);
        if ((st = zkl_hyrax_commit(ctx, pp, cols, A, D, nullptr, out->C_A))) return st;
        if ((st = zkl_hyrax_commit(ctx, pp, cols, B, N, nullptr, out->C_B))) return st;
    }
    tr.absorb_points("A", out->C_A, rD);
    tr.absorb_points("B", out->C_B, rN);
    std::vector<zkl_fr> pre(3 + (size_t)d);
    for (int w = 0; w < 8; ++w)
        pre[0].w[w] = (uint32_t)tr.h[4 * w] | ((uint32_t)tr.h[4 * w + 1] << 8) | ((uint32_t)tr.h[4 * w + 2] << 16) |
                      ((uint32_t)tr.h[4 * w + 3] << 24);
    pre[1] = beta;
    pre[2] = tr.chal("alpha", 0);
    for (int c = 0; c < d; ++c) pre[3 + c] = tr.chal("u", (uint32_t)c);
    // the sumcheck, continuing the transcript on the device
    if ((st = run_proof_fs(ctx, Sv, D, ctx->p1.table, md, nullptr, variant, zkl_vec{nullptr, D}, zkl_vec{nullptr, N},
                           out->round_evals, &out->finals, out->derived, &ei, false, pre.data())))
        return st;
    // proofs of evaluation at v = (r_d, ..., r_1) and v' = v[d-n:]
    std::vector<zkl_fr> v((size_t)d);
    for (int c = 0; c < d; ++c) v[c] = out->derived[3 + d + (d - c - 1)];
    const zkl_fr* vt = v.data() + (d - n);
    struct EvalJob {
        zkl_vec src;
        uint64_t len;
        const zkl_fr* pt;
        zkl_fr* w;
        zkl_fr* y;
    } jobs[7] = {{A, D, v.data(), out->w_A, &out->y_A},   {X, D, v.data(), out->w_X, &out->y_X},
                 {Y, D, v.data(), out->w_Y, &out->y_Y},   {TX, N, vt, out->w_TX, &out->y_TX},
                 {TY, N, vt, out->w_TY, &out->y_TY},      {Mf, N, vt, out->w_m, &out->y_m},
                 {B, N, vt, out->w_B, &out->y_B}};
    for (const auto& j : jobs) {
        {
            HxScope hx(ctx);
            if ((st = zkl_hyrax_prove_eval(ctx, j.src, j.len, cols, j.pt, Wv, j.y))) return st;
        }
        if ((st = zkl_vec_export(ctx, Wv, j.w, 0))) return st;
    }
    return ZKL_OK;
}

int zkl_tlookup_prove_fs(zkl_ctx* ctx, zkl_vec S, uint64_t D, const zkl_table* T, const uint32_t* m_dev,
                         const uint8_t seed[32], zkl_variant variant, zkl_vec A_out, zkl_vec B_out, zkl_fr* round_evals,
                         zkl_final_evals* finals, zkl_fr* derived, int64_t* err_index) {
    int st;
    if ((st = check_ctx(ctx))) return st;
    if (!T) return set_err(ctx, ZKL_E_ARG, "null table");
    return run_proof_fs(ctx, S, D, T, m_dev, seed, variant, A_out, B_out, round_evals, finals, derived, err_index,
                        false);
}

int zkl_sumcheck_prove(zkl_ctx* ctx, zkl_vec A, zkl_vec S, uint64_t D, zkl_vec B, zkl_vec T, zkl_vec m_fr,
                       const zkl_challenges* ch, zkl_variant variant, zkl_fr* round_evals, zkl_final_evals* finals) {
    int st;
    if ((st = check_ctx(ctx))) return st;
    ProveArgs a;
    memset(&a, 0, sizeof(a));
    a.prove_mode = false;
    a.S = S;
    a.A_in = A;
    a.B_in = B;
    a.T_in = T;
    a.m_fr_in = m_fr;
    a.ch = ch;
    a.variant = variant;
    return run_proof(ctx, D, a, round_evals, finals, nullptr);
}

}  // extern "C"

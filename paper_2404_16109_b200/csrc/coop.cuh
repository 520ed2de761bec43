// Causal small rounds in ONE cooperative launch (SURVEY.md §8(a6) causality rule, a9).
//
// Once the vectors have <= 2^17 elements a round is latency-bound: one launch per round plus a one-block derivation
// launch costs ~60 us at H, against ~2 us of arithmetic.  Here the rounds kc .. d run in one cooperative kernel: CTA b
// owns the aligned chunk of 1024 consecutive round-kc elements (an aligned chunk folds into an aligned chunk, so the
// data never leaves the CTA's shared memory), and the rounds are separated by a grid barrier:
//   round k:  every CTA evaluates its pairs and writes one partial row  ->  grid barrier  ->  (Fiat-Shamir) every CTA
//             sums the rows, forms g_k(0..3), absorbs it into its copy of the transcript and derives r_k  ->  fold.
// No CTA folds with r_k before every CTA's round-k partial sums are written (the interactive order of PAPER.md:273-277:
// g_k is complete before r_k is used), so the kernel is a valid non-interactive prover.  The derivation is replicated
// in every CTA (identical inputs, exact arithmetic, so identical r_k); CTA 0 writes the transcript.  After the
// chunk rounds each CTA holds one element; CTA 0 runs the remaining log2(#chunks) rounds in one warp.
#pragma once
#include "fs.cuh"

namespace zkl {

// Transcript state one CTA carries through the rounds (a copy of FsState)
struct FsLocal {
    uint8_t h[32];
    fr C, tscale;
};

// Round k of the Fiat-Shamir transcript from the round's sums (H(1) summed directly): g_k(0..3), absorb, r_k.
// Warp-cooperative (all 32 lanes of one warp call): lanes 0..3 form g_k(t) for their t in parallel (the small
// constant multiples by additions), lane 0 hashes; the sequential chain is 7 Montgomery products plus two SHA-256
// calls, against ~20 products single-threaded.  s, tab: the round's sums (shared memory).  write: this warp also
// records the transcript (evals, derived r_k, sc->r).  Returns r_k (Montgomery) in every lane.
__device__ __noinline__ fr fs_round_warp(int k, int d, const fr* s, const fr* tab, const ProofScalars* sc,
                                         FsLocal& st, bool write, ProofOut* out, zkl_fr* derived, ProofScalars* scw) {
    const int lane = threadIdx.x & 31;
    const fr one = fr_one();
    const fr u = sc->u[d - k];
    const fr coef = fs_mul(sc->alpha1, st.C);
    zkl_fr c;
    for (int l = 0; l < 8; ++l) c.w[l] = 0;
    if (lane < 4) {
        const fr H0 = s[SLOT_H0], H1 = s[SLOT_H1], Hinf = s[SLOT_HINF], a0 = s[SLOT_A0], a1 = s[SLOT_A1];
        const fr da = fr_sub(a1, a0);
        const fr u2 = fr_add(u, u), H12 = fr_add(H1, H1), Hi2 = fr_add(Hinf, Hinf);
        fr lt, H, at;
        if (lane == 0) {            // l_0 = 1 - u
            lt = fr_sub(one, u); H = H0; at = a0;
        } else if (lane == 1) {     // l_1 = u
            lt = u; H = H1; at = a1;
        } else if (lane == 2) {     // l_2 = 3u - 1, H(2) = 2 H1 - H0 + 2 Hinf
            lt = fr_sub(fr_add(u2, u), one);
            H = fr_add(fr_sub(H12, H0), Hi2);
            at = fr_add(a0, fr_add(da, da));
        } else {                    // l_3 = 5u - 2, H(3) = 3 H1 - 2 H0 + 6 Hinf
            lt = fr_sub(fr_add(fr_add(u2, u2), u), fr_add(one, one));
            H = fr_add(fr_sub(fr_add(H12, H1), fr_add(H0, H0)), fr_add(fr_add(Hi2, Hi2), Hi2));
            at = fr_add(a0, fr_add(fr_add(da, da), da));
        }
        const fr g = fr_add(fr_add(fs_mul(fs_mul(coef, lt), H), at), tab[lane]);
        c = fs_canon(g);
        if (write) out->evals[k - 1][lane] = c;
    }
    uint32_t e[32];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int l = 0; l < 8; ++l) e[8 * t + l] = __shfl_sync(0xffffffffu, c.w[l], t);
    fr rm = fr_zero();
    if (lane == 0) {
        uint32_t hw[8];
        fs_h_load(st.h, hw);
        sha256_round_msg(hw, (uint32_t)k, e);
        fs_h_store(hw, st.h);
        const fr r = fs_challenge_w(hw, "r", 1, (uint32_t)k);
        rm = fs_mul(r, fr_r2());
        if (write) {
            derived[3 + d + (k - 1)] = fs_canon_out(r);
            scw->r[k - 1] = rm;
        }
        const fr l0 = fr_sub(one, u);
        st.C = fs_mul(st.C, fr_add(l0, fs_mul(rm, fr_sub(u, l0))));
    }
#pragma unroll
    for (int l = 0; l < 8; ++l) rm.v[l] = __shfl_sync(0xffffffffu, rm.v[l], 0);
    return rm;
}

// the constant table term tau 2^{-(k-n)} of a round k > n (lane 0; tau computed once, cached in *tau_cache)
__device__ __forceinline__ fr fs_table_const(const fr* tfin, const ProofScalars* sc, int variant, FsLocal& st,
                                             fr* tau_cache, bool& have_tau) {
    if (!have_tau) {
        const fr tb = tfin[0], tt = tfin[1], tm = tfin[2], te = tfin[3], beta = sc->beta;
        *tau_cache = (variant == ZKL_VARIANT_PAPER)
            ? fs_mul(tb, fr_sub(fs_mul(fs_mul(sc->alpha2, te), fr_add(tt, beta)), tm))
            : fr_sub(fs_mul(fs_mul(sc->alpha2, te), fr_sub(fs_mul(tb, fr_add(tt, beta)), tm)), tb);
        have_tau = true;
    }
    st.tscale = fs_mul(st.tscale, fr_inv2_m());
    return fs_mul(*tau_cache, st.tscale);
}

constexpr int kCoopTabMax = 512;   // table entries (per vector) CTA 0 keeps in shared memory

// table side of round k on the shared-memory table (AoS [B | T | M | E], stride len): fold with r_{k-1} first
// (fold = true), then, if k <= n, evaluate round k into tab[0..3] (block-wide, all threads call).
__device__ void coop_table_round(fr* V, int& len, bool fold, const fr& rprev, bool eval, const ProofScalars* sc,
                                 int variant, fr* tab_out, fr* tfin, fr* scratch) {
    const int t = threadIdx.x, nt = blockDim.x;
    if (fold) {
        const int np = len / 2;
        fr nv[4][2];
        int cnt = 0;
        for (int y = t; y < np; y += nt, ++cnt)
            for (int q = 0; q < 4; ++q) {
                const fr a = V[q * len + 2 * y], b = V[q * len + 2 * y + 1];
                nv[q][cnt] = fr_add(a, fr_mul(rprev, fr_sub(b, a)));
            }
        __syncthreads();
        cnt = 0;
        for (int y = t; y < np; y += nt, ++cnt)
            for (int q = 0; q < 4; ++q) V[q * np + y] = nv[q][cnt];
        __syncthreads();
        len = np;
        if (len == 1 && t < 4) tfin[t] = V[t];
    }
    if (!eval) return;
    fr g[4] = {fr_zero(), fr_zero(), fr_zero(), fr_zero()};
    const fr beta = sc->beta, alpha2 = sc->alpha2;
    for (int y = t; y < len / 2; y += nt) {
        const fr b0 = V[2 * y], t0 = V[len + 2 * y], m0 = V[2 * len + 2 * y], e0 = V[3 * len + 2 * y];
        const fr db = fr_sub(V[2 * y + 1], b0), dt = fr_sub(V[len + 2 * y + 1], t0);
        const fr dm = fr_sub(V[2 * len + 2 * y + 1], m0), de = fr_sub(V[3 * len + 2 * y + 1], e0);
        fr bt = b0, tt = t0, mt = m0, et = e0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (q > 0) { bt = fr_add(bt, db); tt = fr_add(tt, dt); mt = fr_add(mt, dm); et = fr_add(et, de); }
            g[q] = fr_add(g[q], tab_term(bt, tt, mt, et, beta, alpha2, variant));
        }
    }
    block_sum_fr<4>(g, scratch);
    if (t == 0)
        for (int q = 0; q < 4; ++q) tab_out[q] = g[q];
}

struct CoopFsArgs {
    const uint32_t* Ain;      // round-(kc-1) vectors (2 * nchunks * kChunk elements), folded with r_{kc-1} on load
    const uint32_t* Sin;
    uint64_t nin;
    int kc, d, n, variant;
    const RoundDesc* rounds;
    const fr* arena;
    fr* rows;                 // [round][slot][chunk]: 5 * nchunks per round, rounds kc .. kc + 9
    fr* tabbuf;               // [round][4]: the table term of rounds kc .. d (written by CTA 0)
    fr* chA;                  // the chunks' last elements
    fr* chS;
    const fr* tcur;           // table state entering round kc (folded with r_{kc-2}), AoS stride tlen
    int tlen;
    fr* tfin;
    fr* fin;
    ProofScalars* sc;
    FsState* st;
    ProofOut* out;
    zkl_fr* derived;
    GridBar* bar;
};

// smem: A, S chunk (2 x kChunk fr) | CTA 0: table (4 x kCoopTabMax fr) | scratch
__global__ void __launch_bounds__(kChunkThreads, 1) k_fs_rounds_coop(CoopFsArgs a) {
    extern __shared__ fr smem_fr[];
    fr* As = smem_fr;
    fr* Ss = smem_fr + kChunk;
    fr* V = smem_fr + 2 * kChunk;
    __shared__ fr scratch[5 * (kChunkThreads / 32)];
    __shared__ fr sh_r, sh_tab[4], sh_s[5], sh_tau;
    __shared__ FsLocal st;
    bool have_tau = false;   // (thread 0's) tau of the fully bound table
    const int t = threadIdx.x, nt = blockDim.x;
    const bool cta0 = blockIdx.x == 0;
    const uint32_t nchunks = gridDim.x;
    const ProofScalars* sc = a.sc;
    const fr beta = sc->beta;
    if (t == 0) {
        for (int i = 0; i < 32; ++i) st.h[i] = a.st->h[i];
        st.C = a.st->C;
        st.tscale = a.st->tscale;
    }
    int tlen = a.tlen;
    if (cta0)
        for (int i = t; i < tlen; i += nt)
            for (int q = 0; q < 4; ++q) V[q * tlen + i] = a.tcur[q * tlen + i];
    {
        const fr r = sc->r[a.kc - 2];
        const uint64_t base = 2 * (uint64_t)blockIdx.x * kChunk;
        for (int i = t; i < kChunk; i += nt) {
            fr x[2], y[2];
            ld_fr2(a.Ain, a.nin, base + 2 * i, x);
            ld_fr2(a.Sin, a.nin, base + 2 * i, y);
            As[i] = fr_add(x[0], fr_mul(r, fr_sub_lazy(x[1], x[0])));
            Ss[i] = fr_add(y[0], fr_mul(r, fr_sub_lazy(y[1], y[0])));
        }
    }
    __syncthreads();
    int len = kChunk;
    fr rprev = sc->r[a.kc - 2];
    const int kend = a.kc + kChunkBits - 1;
    for (int k = a.kc; k <= kend; ++k) {
        const RoundDesc rd = a.rounds[k - 1];
        const fr* elo = a.arena + rd.elo_off;
        const fr* ehi = a.arena + rd.ehi_off;
        const uint32_t gmask = (1u << rd.gbits) - 1u;
        const int half = len / 2;
        fr v[5] = {fr_zero(), fr_zero(), fr_zero(), fr_zero(), fr_zero()};
        for (int yl = t; yl < half; yl += nt) {
            const uint64_t y = (uint64_t)blockIdx.x * half + yl;
            const fr e = fr_mul(ehi[y >> rd.gbits], elo[y & gmask]);
            const fr A0 = As[2 * yl], A1 = As[2 * yl + 1], S0 = Ss[2 * yl], S1 = Ss[2 * yl + 1];
            v[SLOT_H0] = fr_add(v[SLOT_H0], fr_mul(e, fr_mul(A0, fr_add_lazy(S0, beta))));
            v[SLOT_H1] = fr_add(v[SLOT_H1], fr_mul(e, fr_mul(A1, fr_add_lazy(S1, beta))));
            v[SLOT_HINF] = fr_add(v[SLOT_HINF], fr_mul(e, fr_mul(fr_sub(A1, A0), fr_sub_lazy(S1, S0))));
            v[SLOT_A0] = fr_add(v[SLOT_A0], A0);
            v[SLOT_A1] = fr_add(v[SLOT_A1], A1);
        }
        block_sum_fr<5>(v, scratch);
        fr* rows = a.rows + (uint64_t)(k - a.kc) * 5 * nchunks;
        if (t == 0)
            for (int q = 0; q < 5; ++q) rows[(uint64_t)q * nchunks + blockIdx.x] = v[q];
        if (cta0) {   // the table term of round k (fold with r_{k-1} while the table is still being bound)
            const bool fold = (k - 1 <= a.n) && tlen > 1;
            coop_table_round(V, tlen, fold, rprev, k <= a.n, sc, a.variant, sh_tab, a.tfin, scratch);
            if (t == 0) for (int q = 0; q < 4; ++q) a.tabbuf[(k - a.kc) * 4 + q] = k <= a.n ? sh_tab[q] : fr_zero();
            __threadfence();
        }
        grid_sync(a.bar);
        // every CTA: the round's sums, g_k, the transcript, r_k
        fr s[5];
        for (int q = 0; q < 5; ++q) {
            s[q] = fr_zero();
            for (uint32_t b = t; b < nchunks; b += nt) s[q] = fr_add(s[q], rows[(uint64_t)q * nchunks + b]);
        }
        block_sum_fr<5>(s, scratch);
        if (t == 0) {
            for (int q = 0; q < 5; ++q) sh_s[q] = s[q];
            if (k <= a.n) {
                for (int q = 0; q < 4; ++q) sh_tab[q] = a.tabbuf[(k - a.kc) * 4 + q];
            } else {
                const fr c = fs_table_const(a.tfin, sc, a.variant, st, &sh_tau, have_tau);
                for (int q = 0; q < 4; ++q) sh_tab[q] = c;
            }
        }
        __syncthreads();
        if (t < 32) {
            const fr rk = fs_round_warp(k, a.d, sh_s, sh_tab, sc, st, cta0, a.out, a.derived, a.sc);
            if (t == 0) sh_r = rk;
        }
        __syncthreads();
        const fr rk = sh_r;
        rprev = rk;
        // fold the chunk with r_k
        fr na[kChunk / 2 / kChunkThreads], ns[kChunk / 2 / kChunkThreads];
        int cnt = 0;
        for (int yl = t; yl < half; yl += nt, ++cnt) {
            na[cnt] = fr_add(As[2 * yl], fr_mul(rk, fr_sub_lazy(As[2 * yl + 1], As[2 * yl])));
            ns[cnt] = fr_add(Ss[2 * yl], fr_mul(rk, fr_sub_lazy(Ss[2 * yl + 1], Ss[2 * yl])));
        }
        __syncthreads();
        cnt = 0;
        for (int yl = t; yl < half; yl += nt, ++cnt) {
            As[yl] = na[cnt];
            Ss[yl] = ns[cnt];
        }
        __syncthreads();
        len = half;
    }
    // one element per chunk: CTA 0 runs the remaining rounds (log2 #chunks) in one warp
    if (t == 0) {
        a.chA[blockIdx.x] = As[0];
        a.chS[blockIdx.x] = Ss[0];
    }
    __threadfence();
    grid_sync(a.bar);
    if (!cta0) return;
    int m = (int)nchunks;
    for (int i = t; i < m; i += nt) {
        As[i] = a.chA[i];
        Ss[i] = a.chS[i];
    }
    __syncthreads();
    for (int k = kend + 1; k <= a.d; ++k) {
        const RoundDesc rd = a.rounds[k - 1];
        const fr* elo = a.arena + rd.elo_off;
        const fr eh = a.arena[rd.ehi_off];
        const int half = m / 2;
        // the table (if still being bound) with all threads, then the D side in warp 0
        const bool fold = (k - 1 <= a.n) && tlen > 1;
        coop_table_round(V, tlen, fold, rprev, k <= a.n, sc, a.variant, sh_tab, a.tfin, scratch);
        if (t < 32) {
            fr v[5] = {fr_zero(), fr_zero(), fr_zero(), fr_zero(), fr_zero()};
            for (int y = t; y < half; y += 32) {
                const fr e = fr_mul(eh, elo[y]);
                const fr A0 = As[2 * y], A1 = As[2 * y + 1], S0 = Ss[2 * y], S1 = Ss[2 * y + 1];
                v[SLOT_H0] = fr_add(v[SLOT_H0], fr_mul(e, fr_mul(A0, fr_add_lazy(S0, beta))));
                v[SLOT_H1] = fr_add(v[SLOT_H1], fr_mul(e, fr_mul(A1, fr_add_lazy(S1, beta))));
                v[SLOT_HINF] = fr_add(v[SLOT_HINF], fr_mul(e, fr_mul(fr_sub(A1, A0), fr_sub_lazy(S1, S0))));
                v[SLOT_A0] = fr_add(v[SLOT_A0], A0);
                v[SLOT_A1] = fr_add(v[SLOT_A1], A1);
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1)
#pragma unroll
                for (int q = 0; q < 5; ++q) v[q] = fr_add(v[q], shfl_down_fr(v[q], off));
            if (t == 0) {
                for (int q = 0; q < 5; ++q) sh_s[q] = v[q];
                if (k > a.n) {
                    const fr c = fs_table_const(a.tfin, sc, a.variant, st, &sh_tau, have_tau);
                    for (int q = 0; q < 4; ++q) sh_tab[q] = c;
                }
            }
            __syncwarp();
            const fr rk = fs_round_warp(k, a.d, sh_s, sh_tab, sc, st, true, a.out, a.derived, a.sc);
            if (t == 0) sh_r = rk;
        }
        __syncthreads();
        const fr rk = sh_r;
        rprev = rk;
        fr na = fr_zero(), ns = fr_zero();
        if (t < half) {
            na = fr_add(As[2 * t], fr_mul(rk, fr_sub_lazy(As[2 * t + 1], As[2 * t])));
            ns = fr_add(Ss[2 * t], fr_mul(rk, fr_sub_lazy(Ss[2 * t + 1], Ss[2 * t])));
        }
        __syncthreads();
        if (t < half) {
            As[t] = na;
            Ss[t] = ns;
        }
        __syncthreads();
        m = half;
    }
    // the table's last fold (n = d: its final coordinate is bound by r_d)
    if (a.n == a.d && tlen > 1) coop_table_round(V, tlen, true, rprev, false, sc, a.variant, sh_tab, a.tfin, scratch);
    if (t == 0) {
        a.fin[0] = As[0];
        a.fin[1] = Ss[0];
        for (int i = 0; i < 32; ++i) a.st->h[i] = st.h[i];
        a.st->C = st.C;
        a.st->tscale = st.tscale;
    }
}

}  // namespace zkl

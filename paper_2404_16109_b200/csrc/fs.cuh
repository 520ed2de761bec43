// Fiat-Shamir mode: the verifier's challenges are derived on the device from a SHA-256
// transcript, so r_k depends on g_k and every round waits for the previous round's derivation (one small
// kernel per round).  Transcript:
//   h_0   = SHA256("zkl-fs-v1" || seed[32] || le64(D) || le64(N) || le32(variant))
//   chal(label, i) = le-integer(SHA256(h || label || le32(i))) mod r
//   beta = chal("beta", 0), alpha1 = chal("alpha", 0), alpha2 = alpha1^2, u_c = chal("u", c)
//   round k: h_k = SHA256(h_{k-1} || "g" || le32(k) || g_k(0) || g_k(1) || g_k(2) || g_k(3)),  r_k = chal("r", k)
// The seed stands for the commitments the prover would have sent ([T], [S], [m]); commitments are NEXT f3.
#pragma once
#include "kernels.cuh"
#include "sha256.cuh"

namespace zkl {

// Single-thread scalar code (the per-round derivation) executes each instruction once: with fr_mul inlined ~30
// times the kernel is instruction-fetch bound, so the scalar section calls one shared out-of-line copy.
static __device__ __noinline__ fr fs_mul(const fr a, const fr b) { return fr_mul(a, b); }
static __device__ __noinline__ zkl_fr fs_canon(const fr a) {
    fr one = fr_zero();   // the integer 1: mont(a, 1) = a / R, the canonical value
    one.v[0] = 1;
    const fr c = fs_mul(a, one);
    zkl_fr z;
    for (int l = 0; l < 8; ++l) z.w[l] = c.v[l];
    return z;
}

struct FsState {
    uint8_t h[32];
    fr C;        // C_k = prod_{j<k} l_{d-j}(r_j)
    fr tscale;   // 2^{-(k-n)} once the table coordinates are bound
    fr gprev[4]; // g_{k-1}(0..3), Montgomery: the running claim g_{k-1}(r_{k-1}) of a derived-H(1) round
    fr inv_cl1;  // 1 / (alpha1 C_k u_{d-k}) for round k (k_fs_inv, side stream, during round k's fold + eval)
    fr aprev[2]; // a0_{k-1}, a1_{k-1}: a(1) of a round whose kernel did not sum it (RoundDesc::a1_derived)
};

// 1 / (alpha1 C_k u_{d-k}) for round k: launched once r_{k-1} (hence C_k) is known, overlapping k_round(k)
__global__ void k_fs_inv(int k, int d, const ProofScalars* __restrict__ sc, FsState* st) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    st->inv_cl1 = fr_inv(fr_mul(fr_mul(sc->alpha1, st->C), sc->u[d - k]));
}

// canonical 256-bit little-endian value of a digest, reduced mod r (x < 2^256 < 3r)
__device__ inline fr fs_digest_to_fr(const uint8_t* dg) {
    fr x;
    for (int l = 0; l < 8; ++l)
        x.v[l] = (uint32_t)dg[4 * l] | ((uint32_t)dg[4 * l + 1] << 8) | ((uint32_t)dg[4 * l + 2] << 16) |
                 ((uint32_t)dg[4 * l + 3] << 24);
    fr_reduce_once(x);
    fr_reduce_once(x);
    return x;
}

__device__ inline fr fs_challenge(const uint8_t* h, const char* label, int llen, uint32_t idx) {
    uint8_t msg[48], dg[32];
    int p = 0;
    for (int i = 0; i < 32; ++i) msg[p++] = h[i];
    for (int i = 0; i < llen; ++i) msg[p++] = (uint8_t)label[i];
    for (int i = 0; i < 4; ++i) msg[p++] = (uint8_t)(idx >> (8 * i));
    sha256(msg, p, dg);
    return fs_digest_to_fr(dg);
}

// the transcript digest as its 8 big-endian words and back
__device__ __forceinline__ void fs_h_load(const uint8_t* h, uint32_t (&hw)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
        hw[i] = ((uint32_t)h[4 * i] << 24) | ((uint32_t)h[4 * i + 1] << 16) | ((uint32_t)h[4 * i + 2] << 8) | h[4 * i + 3];
}
__device__ __forceinline__ void fs_h_store(const uint32_t (&hw)[8], uint8_t* h) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        h[4 * i] = (uint8_t)(hw[i] >> 24);
        h[4 * i + 1] = (uint8_t)(hw[i] >> 16);
        h[4 * i + 2] = (uint8_t)(hw[i] >> 8);
        h[4 * i + 3] = (uint8_t)hw[i];
    }
}
// chal(label, idx) from the digest words (= fs_challenge on the digest bytes)
__device__ inline fr fs_challenge_w(const uint32_t (&hw)[8], const char* label, int llen, uint32_t idx) {
    uint32_t dg[8];
    sha256_chal_msg(hw, label, llen, idx, dg);
    fr x;
#pragma unroll
    for (int l = 0; l < 8; ++l) x.v[l] = __byte_perm(dg[l], 0, 0x0123);   // little-endian integer of the digest
    fr_reduce_once(x);
    fr_reduce_once(x);
    return x;
}

__device__ inline zkl_fr fs_canon_out(const fr& c) {
    zkl_fr z;
    for (int l = 0; l < 8; ++l) z.w[l] = c.v[l];
    return z;
}

// derive beta, alpha1, alpha2, u into sc (Montgomery) and `derived` (canonical: beta, alpha1, alpha2, u[d], r[d])
__global__ void k_fs_init(const uint8_t* __restrict__ seed, uint64_t D, uint64_t N, int variant, int d,
                          ProofScalars* sc, FsState* st, zkl_fr* derived, int pbits, int rank) {
    // thread 0: h_0, beta, alpha; then the d independent u_c in parallel (one warp, launched with 32 threads)
    if (blockIdx.x != 0) return;
    if (threadIdx.x == 0) {
    uint8_t msg[9 + 32 + 8 + 8 + 4];
    const char* tag = "zkl-fs-v1";
    int p = 0;
    for (int i = 0; i < 9; ++i) msg[p++] = (uint8_t)tag[i];
    for (int i = 0; i < 32; ++i) msg[p++] = seed[i];
    for (int i = 0; i < 8; ++i) msg[p++] = (uint8_t)(D >> (8 * i));
    for (int i = 0; i < 8; ++i) msg[p++] = (uint8_t)(N >> (8 * i));
    for (int i = 0; i < 4; ++i) msg[p++] = (uint8_t)((uint32_t)variant >> (8 * i));
    sha256(msg, p, st->h);
    const fr beta = fs_challenge(st->h, "beta", 4, 0);
    const fr a1 = fs_challenge(st->h, "alpha", 5, 0);
    const fr a1m = fr_to_mont(a1);
    const fr a2m = fr_mul(a1m, a1m);
    sc->beta = fr_to_mont(beta);
    sc->alpha1 = a1m;
    sc->alpha2 = a2m;
    derived[0] = fs_canon_out(beta);
    derived[1] = fs_canon_out(a1);
    derived[2] = to_canon(a2m);
    }
    __syncwarp();
    __threadfence_block();
    {
        uint32_t hw[8];
        fs_h_load(st->h, hw);
        for (int c = threadIdx.x; c < d; c += blockDim.x) {
            const fr u = fs_challenge_w(hw, "u", 1, (uint32_t)c);
            sc->u[c] = fr_to_mont(u);
            derived[3 + c] = fs_canon_out(u);
        }
    }
    __syncwarp();
    __threadfence_block();
    if (threadIdx.x != 0) return;
    // this rank's factor of e~(u, .): eq(u[0:log2 P], bits(rank)) (the top coordinates are the rank)
    fr re = fr_one();
    for (int b = 0; b < pbits; ++b) {
        const bool bit = (rank >> (pbits - 1 - b)) & 1;
        re = fr_mul(re, bit ? sc->u[b] : fr_sub(fr_one(), sc->u[b]));
    }
    sc->rank_eq = re;
    st->C = fr_one();
    st->tscale = fr_one();
}

// Protocol-1 transcript: the host absorbed the commitments and derived beta, alpha1 and u; the device
// continues the same transcript for the rounds.  pre (canonical zkl_fr): [0] h as 32 bytes, [1] beta, [2] alpha1,
// [3 ..] u[0 .. d-1].
__global__ void k_fs_init_preset(const zkl_fr* __restrict__ pre, int d, ProofScalars* sc, FsState* st,
                                 zkl_fr* derived, int pbits, int rank) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int i = 0; i < 8; ++i)
        for (int b = 0; b < 4; ++b) st->h[4 * i + b] = (uint8_t)(pre[0].w[i] >> (8 * b));
    auto canon = [](const zkl_fr& z) {
        fr x;
        for (int l = 0; l < 8; ++l) x.v[l] = z.w[l];
        return x;
    };
    const fr beta = canon(pre[1]), a1 = canon(pre[2]);
    const fr a1m = fr_to_mont(a1);
    sc->beta = fr_to_mont(beta);
    sc->alpha1 = a1m;
    sc->alpha2 = fr_mul(a1m, a1m);
    derived[0] = pre[1];
    derived[1] = pre[2];
    derived[2] = to_canon(sc->alpha2);
    for (int c = 0; c < d; ++c) {
        sc->u[c] = fr_to_mont(canon(pre[3 + c]));
        derived[3 + c] = pre[3 + c];
    }
    fr re = fr_one();
    for (int b = 0; b < pbits; ++b) {
        const bool bit = (rank >> (pbits - 1 - b)) & 1;
        re = fr_mul(re, bit ? sc->u[b] : fr_sub(fr_one(), sc->u[b]));
    }
    sc->rank_eq = re;
    st->C = fr_one();
    st->tscale = fr_one();
}

// table side, split for the causal order: fold with r_{k-1} (after it is derived), then evaluate round k
__global__ void __launch_bounds__(256)
k_tab_eval(const fr* __restrict__ cur, uint64_t len, const ProofScalars* __restrict__ sc, int variant, fr* tpart) {
    const fr beta = sc->beta, alpha2 = sc->alpha2;
    fr g[4] = {fr_zero(), fr_zero(), fr_zero(), fr_zero()};
    for (uint64_t y = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; y < len / 2; y += (uint64_t)gridDim.x * blockDim.x) {
        const fr b0 = cur[2 * y], b1 = cur[2 * y + 1];
        const fr t0 = cur[len + 2 * y], t1 = cur[len + 2 * y + 1];
        const fr m0 = cur[2 * len + 2 * y], m1 = cur[2 * len + 2 * y + 1];
        const fr e0 = cur[3 * len + 2 * y], e1 = cur[3 * len + 2 * y + 1];
        const fr db = fr_sub(b1, b0), dt = fr_sub(t1, t0), dm = fr_sub(m1, m0), de = fr_sub(e1, e0);
        fr bt = b0, tt = t0, mt = m0, et = e0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (q > 0) { bt = fr_add(bt, db); tt = fr_add(tt, dt); mt = fr_add(mt, dm); et = fr_add(et, de); }
            g[q] = fr_add(g[q], tab_term(bt, tt, mt, et, beta, alpha2, variant));
        }
    }
    __shared__ fr scratch[4 * 8];
    block_sum_fr<4>(g, scratch);
    if (threadIdx.x == 0)
        for (int q = 0; q < 4; ++q) tpart[q * kMaxBlocks + blockIdx.x] = g[q];
}

__global__ void k_tab_fold(const fr* __restrict__ cur, uint64_t len, fr* nxt, const ProofScalars* __restrict__ sc, int k,
                           fr* tfin) {
    const fr r = sc->r[k - 1];
    const uint64_t np = len / 2;
    for (uint64_t y = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; y < np; y += (uint64_t)gridDim.x * blockDim.x) {
        for (int v = 0; v < 4; ++v) {
            const fr a = cur[v * len + 2 * y], b = cur[v * len + 2 * y + 1];
            const fr f = fr_add(a, fr_mul(r, fr_sub(b, a)));
            nxt[v * np + y] = f;
            if (np == 1) tfin[v] = f;
        }
    }
}

__global__ void k_tab_fin_copy(const fr* __restrict__ cur, fr* tfin) {
    if (threadIdx.x < 4 && blockIdx.x == 0) tfin[threadIdx.x] = cur[threadIdx.x];
}

// fold the last pair of A, S with r_d: the finals A(v), S(v)
__global__ void k_fold_final(const uint32_t* __restrict__ A, const uint32_t* __restrict__ S, uint64_t n,
                             const ProofScalars* __restrict__ sc, int d, fr* fin) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const fr r = sc->r[d - 1];
    const fr a0 = ld_fr(A, n, 0), a1 = ld_fr(A, n, 1), s0 = ld_fr(S, n, 0), s1 = ld_fr(S, n, 1);
    fin[0] = fr_add(a0, fr_mul(r, fr_sub(a1, a0)));
    fin[1] = fr_add(s0, fr_mul(r, fr_sub(s1, s0)));
}

// Round k: reduce the D-side partial rows (and the table rows, k <= n), form g_k(0..3) directly, absorb it,
// derive r_k.  h01_one: round 1 of the gather/inversion path, where H(0) = H(1) = sum eq = 1.
// part [5][nrows] -> out [5][outrows]: CTA b sums rows [b per, (b+1) per) of every slot
__global__ void k_rows_fold(const fr* __restrict__ part, uint32_t nrows, fr* out, uint32_t outrows) {
    __shared__ fr scratch[5 * 8];
    const uint32_t per = (nrows + outrows - 1) / outrows, r0 = blockIdx.x * per, r1 = min(r0 + per, nrows);
    fr v[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        v[q] = fr_zero();
        for (uint32_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) v[q] = fr_add(v[q], part[(uint64_t)q * nrows + r]);
    }
    block_sum_fr<5>(v, scratch);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < 5; ++q) out[(uint64_t)q * outrows + blockIdx.x] = v[q];
    }
}

// derive_h1: the round's k_round did not sum H(1) (k_round<true, false>); it follows from the running claim,
// H(1) = (g_{k-1}(r_{k-1}) - cl0 H(0) - a0 - a1 - tab(0) - tab(1)) / cl1.  cl1 = 0 with alpha1 C_k != 0 (u_{d-k} = 0,
// probability ~2^-255) cannot be derived: the proof is flagged through `miss` and redone with H(1) summed.
// part: the round's D-side rows; element (slot q, row b) at part[q * slot_stride + b * row_stride] (partial rows:
// slot-major, slot_stride = nrows, row_stride = 1; P > 1: the all-gathered rank sums, rank-major, 1 and kSlots).
#ifdef ZKL_FS_TIMING   // dev instrumentation (build variant only): per-phase clock64 deltas of k_fs_round, printed
#define FS_T(i) do { if (threadIdx.x == 0) tt[i] = clock64(); } while (0)
#else
#define FS_T(i) do { } while (0)
#endif
__global__ void k_fs_round(int k, int d, int n, int variant, const fr* __restrict__ part, uint32_t nrows,
                           int h01_one, const fr* __restrict__ tpart, uint32_t tnb, const fr* __restrict__ tfin,
                           ProofScalars* sc, FsState* st, ProofOut* out, zkl_fr* derived, int derive_h1,
                           unsigned long long* miss, uint32_t slot_stride, uint32_t row_stride, int a1_derived) {
#ifdef ZKL_FS_TIMING
    long long tt[10];
#endif
    FS_T(0);
    __shared__ fr scratch[5 * 8];
    fr s[5];
    for (int q = 0; q < 5; ++q) {
        s[q] = fr_zero();
        for (uint32_t b = threadIdx.x; b < nrows; b += blockDim.x)
            s[q] = fr_add(s[q], part[(uint64_t)q * slot_stride + (uint64_t)b * row_stride]);
    }
    block_sum_fr<5>(s, scratch);
    FS_T(1);
    fr tab[4] = {fr_zero(), fr_zero(), fr_zero(), fr_zero()};
    if (k <= n) {
        for (int q = 0; q < 4; ++q)
            for (uint32_t b = threadIdx.x; b < tnb; b += blockDim.x) tab[q] = fr_add(tab[q], tpart[q * kMaxBlocks + b]);
        block_sum_fr<4>(tab, scratch);
    }
    FS_T(2);
    // the scalar part: warp 0, lanes 0..3 form g_k(t) for their t (the derived H(1) by Lagrange, lane t the
    // term t), lane 0 hashes (word-level SHA-256): ~12 sequential products instead of ~35 on one thread
    __shared__ fr sh_s[5], sh_tab[4];
    if (threadIdx.x == 0) {
        if (a1_derived) {   // a0_k + a1_k = a0_{k-1} + r_{k-1} (a1_{k-1} - a0_{k-1})
            const fr p0 = st->aprev[0], p1 = st->aprev[1];
            s[SLOT_A1] = fr_sub(fr_add(p0, fs_mul(sc->r[k - 2], fr_sub(p1, p0))), s[SLOT_A0]);
        }
        st->aprev[0] = s[SLOT_A0];
        st->aprev[1] = s[SLOT_A1];
        if (k > n) {
            const fr tb = tfin[0], tt = tfin[1], tm = tfin[2], te = tfin[3];
            const fr tau = (variant == ZKL_VARIANT_PAPER)
                ? fs_mul(tb, fr_sub(fs_mul(fs_mul(sc->alpha2, te), fr_add(tt, sc->beta)), tm))
                : fr_sub(fs_mul(fs_mul(sc->alpha2, te), fr_sub(fs_mul(tb, fr_add(tt, sc->beta)), tm)), tb);
            st->tscale = fs_mul(st->tscale, fr_inv2_m());
            const fr c = fs_mul(tau, st->tscale);
            for (int q = 0; q < 4; ++q) tab[q] = c;
        }
        if (h01_one) { s[SLOT_H0] = fr_one(); s[SLOT_H1] = fr_one(); }
        for (int q = 0; q < 5; ++q) sh_s[q] = s[q];
        for (int q = 0; q < 4; ++q) sh_tab[q] = tab[q];
    }
    __syncthreads();
    FS_T(3);
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    const fr one = fr_one();
    const fr u = sc->u[d - k];
    const fr coef = fs_mul(sc->alpha1, st->C);
    const fr H0 = sh_s[SLOT_H0], Hinf = sh_s[SLOT_HINF], a0 = sh_s[SLOT_A0], a1 = sh_s[SLOT_A1];
    fr H1 = sh_s[SLOT_H1];
    if (derive_h1) {
        // claim = g_{k-1}(x), x = r_{k-1}, by Lagrange on the nodes 0..3: lane t its term g_{k-1}(t) L_t(x)
        fr term = fr_zero();
        if (lane < 4) {
            const fr x = sc->r[k - 2], two = fr_add(one, one), three = fr_add(two, one);
            const fr xm1 = fr_sub(x, one), xm2 = fr_sub(x, two), xm3 = fr_sub(x, three);
            fr L;
            if (lane == 0) L = fr_neg(fs_mul(fs_mul(xm1, fs_mul(xm2, xm3)), fr_inv6_m()));
            else if (lane == 1) L = fs_mul(fs_mul(x, fs_mul(xm2, xm3)), fr_inv2_m());
            else if (lane == 2) L = fr_neg(fs_mul(fs_mul(fs_mul(x, xm1), xm3), fr_inv2_m()));
            else L = fs_mul(fs_mul(fs_mul(x, xm1), xm2), fr_inv6_m());
            term = fs_mul(st->gprev[lane], L);
        }
#pragma unroll
        for (int off = 2; off > 0; off >>= 1) term = fr_add(term, shfl_down_fr(term, off));
        fr h1 = fr_zero();
        if (lane == 0) {
            const fr cl0 = fs_mul(coef, fr_sub(one, u));
            const fr rest = fr_sub(fr_sub(fr_sub(term, fs_mul(cl0, H0)), fr_add(a0, a1)), fr_add(sh_tab[0], sh_tab[1]));
            h1 = fs_mul(rest, st->inv_cl1);
            if (fr_is_zero(fs_mul(coef, u)) && !fr_is_zero(coef)) atomicMin(miss, 0ull);
        }
#pragma unroll
        for (int l = 0; l < 8; ++l) H1.v[l] = __shfl_sync(0xffffffffu, h1.v[l], 0);
    }
    FS_T(4);
    zkl_fr c;
    for (int l = 0; l < 8; ++l) c.w[l] = 0;
    if (lane < 4) {
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
        const fr g = fr_add(fr_add(fs_mul(fs_mul(coef, lt), H), at), sh_tab[lane]);
        st->gprev[lane] = g;
        c = fs_canon(g);
        out->evals[k - 1][lane] = c;
    }
    uint32_t e[32];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int l = 0; l < 8; ++l) e[8 * t + l] = __shfl_sync(0xffffffffu, c.w[l], t);
    if (lane != 0) return;
    FS_T(5);
    uint32_t hw[8];
    fs_h_load(st->h, hw);
    sha256_round_msg(hw, (uint32_t)k, e);
    fs_h_store(hw, st->h);
    FS_T(6);
    const fr r = fs_challenge_w(hw, "r", 1, (uint32_t)k);
    FS_T(7);
    derived[3 + d + (k - 1)] = fs_canon_out(r);
    const fr rm = fs_mul(r, fr_r2());
    sc->r[k - 1] = rm;
    const fr l0 = fr_sub(one, u);
    st->C = fs_mul(st->C, fr_add(l0, fs_mul(rm, fr_sub(u, l0))));
    FS_T(8);
#ifdef ZKL_FS_TIMING
    printf("fs_round k=%d rows=%lld tab=%lld t0sec=%lld coef+h1=%lld g=%lld sha=%lld chal=%lld tail=%lld total=%lld\n",
           k, tt[1] - tt[0], tt[2] - tt[1], tt[3] - tt[2], tt[4] - tt[3], tt[5] - tt[4], tt[6] - tt[5], tt[7] - tt[6],
           tt[8] - tt[7], tt[8] - tt[0]);
#endif
}

__global__ void k_fs_finish(const fr* __restrict__ fin, const fr* __restrict__ tfin, ProofOut* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    out->finals[0] = to_canon(fin[0]);
    out->finals[1] = to_canon(fin[1]);
    out->finals[2] = to_canon(tfin[0]);
    out->finals[3] = to_canon(tfin[1]);
    out->finals[4] = to_canon(tfin[2]);
}

}  // namespace zkl

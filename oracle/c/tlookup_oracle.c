/*
 * C tier of the CPU oracle for the zkLLM tlookup prover (arXiv 2404.16109).
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/ (oracle/c_oracle.py) and by bench.py's
 * cpu_baseline / --impl reference leg.  Shares no code with the CUDA path
 * (paper_2404_16109_b200/csrc): different radix (4 x 64-bit limbs, unsigned __int128),
 * different reduction code, different language, no common headers or tables.
 *
 * It computes exactly what oracle/tlookup.py computes, for sizes Python cannot reach:
 *   - Fr arithmetic: textbook Montgomery multiplication, radix 2^64 (Handbook of
 *     Applied Cryptography Alg. 14.36), operands kept in [0, r).
 *   - S for function lookups: S = X + alpha_f * Y.
 *   - m: Eq. hab22-coefs, by sorting T and binary search.
 *   - A, B: Eq. hab22-invs by Montgomery's batch-inversion trick
 *     (prefix products, one Fermat inversion a^(r-2), backward pass) — exact.
 *   - sumcheck on Eq. tlookup-sumcheck, LSB first, every round
 *     polynomial evaluated directly at t = 0,1,2,3 from the folded vectors (no
 *     derived values, no eq factoring).  D-side vectors A, S, e~(u,.) are D-sized.
 *     The table side uses the N-sized vectors B, T, m, e~(u[d-n:],.): while a table
 *     coordinate is free (round k <= n) the sum over the d-n repeated coordinates
 *     contributes (D/N) * (N/D) = 1 times the N-sized sum; once all table coordinates
 *     are bound (k > n) the term is a constant tau and contributes
 *     2^(d-k) * (N/D) * tau = tau / 2^(k-n) to every g_k(t).  Cross-checked against
 *     the D-repeated Python tier in tests/test_oracle_c.py.
 *
 * zko_tlookup_pair_stream (below) is the same computation for function / range lookups given as int32 pairs
 * (S_i = x_i + alpha_f y_i, T_j = tx_j + alpha_f ty_j), in memory bounded for D = 2^30 (SURVEY.md §7 step 8,
 * §8(d)): S is formed from (x_i, y_i) where it is used instead of being stored, A_i = 1/(beta + S_i) is
 * recomputed per block of 2^s consecutive elements (Montgomery batch inversion per batch of blocks), and the first
 * s rounds are evaluated block by block -- the pairs of round k inside an aligned block of 2^s elements fold into
 * the same block, so each block's contribution to g_1..g_s is computed from its own elements alone, exactly as the
 * unblocked loop computes it.  Vectors are materialised from round s+1 (D / 2^s elements).  Equality with
 * zko_tlookup for every s is checked in tests/test_oracle_c.py.
 *
 * Conventions: DESIGN.md §2 readings (coordinate 0 = MSB, j = x mod N, LSB-first
 * binding, g_k given at t = 0..3, weights (1, alpha1, alpha2)).
 * Threads: OpenMP over independent elements / pairs (sums reduced exactly mod r).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;
typedef struct { uint64_t l[4]; } fe;   /* little-endian 64-bit limbs */

static const fe P = {{0xffffffff00000001ULL, 0x53bda402fffe5bfeULL, 0x3339d80809a1d805ULL, 0x73eda753299d7d48ULL}};
static uint64_t PINV;      /* -P^{-1} mod 2^64 */
static fe R2;              /* 2^512 mod P */
static fe ONE_M;           /* 2^256 mod P (1 in Montgomery form) */
static int inited = 0;

static int geq(const fe *a, const fe *b) {
    for (int i = 3; i >= 0; --i) {
        if (a->l[i] != b->l[i]) return a->l[i] > b->l[i];
    }
    return 1;
}

static void sub_raw(fe *r, const fe *a, const fe *b) {
    u128 borrow = 0;
    for (int i = 0; i < 4; ++i) {
        u128 t = (u128)a->l[i] - b->l[i] - borrow;
        r->l[i] = (uint64_t)t;
        borrow = (t >> 64) ? 1 : 0;
    }
}

static fe fadd(fe a, fe b) {
    fe r;
    u128 c = 0;
    for (int i = 0; i < 4; ++i) {
        u128 t = (u128)a.l[i] + b.l[i] + c;
        r.l[i] = (uint64_t)t;
        c = t >> 64;
    }
    /* a, b < P < 2^255 so no carry out of 256 bits */
    if (geq(&r, &P)) sub_raw(&r, &r, &P);
    return r;
}

static fe fsub(fe a, fe b) {
    fe r;
    if (geq(&a, &b)) {
        sub_raw(&r, &a, &b);
    } else {
        fe t;
        sub_raw(&t, &P, &b);   /* P - b */
        r = fadd(a, t);
    }
    return r;
}

/* HAC Alg. 14.36: Montgomery multiplication, radix 2^64, n = 4 words. */
static fe fmul(fe x, fe y) {
    uint64_t a[6] = {0, 0, 0, 0, 0, 0};
    for (int i = 0; i < 4; ++i) {
        /* u_i = (a_0 + x_i y_0) m' mod b */
        uint64_t ui = (a[0] + x.l[i] * y.l[0]) * PINV;
        /* A = (A + x_i y + u_i m) / b */
        u128 c1 = 0, c2 = 0;
        for (int j = 0; j < 4; ++j) {
            u128 t = (u128)x.l[i] * y.l[j] + a[j] + (uint64_t)c1;
            c1 = t >> 64;
            u128 s = (u128)ui * P.l[j] + (uint64_t)t + (uint64_t)c2;
            c2 = s >> 64;
            a[j] = (uint64_t)s;          /* a[0] becomes 0 by construction */
        }
        u128 t = (u128)a[4] + (uint64_t)c1 + (uint64_t)c2;
        a[4] = (uint64_t)t;
        a[5] = (uint64_t)(t >> 64);
        for (int j = 0; j < 5; ++j) a[j] = a[j + 1];
        a[5] = 0;
    }
    fe r = {{a[0], a[1], a[2], a[3]}};
    if (a[4] || geq(&r, &P)) sub_raw(&r, &r, &P);
    return r;
}

static fe fe_from_u64(uint64_t v) { fe r = {{v, 0, 0, 0}}; return r; }
static int fe_is_zero(fe a) { return (a.l[0] | a.l[1] | a.l[2] | a.l[3]) == 0; }
static int fe_eq(fe a, fe b) { return !memcmp(&a, &b, sizeof(fe)); }
static fe to_m(fe a) { return fmul(a, R2); }
static fe from_m(fe a) { return fmul(a, fe_from_u64(1)); }

static fe fpow(fe a, const fe *e) {   /* a in Montgomery form; e canonical exponent */
    fe acc = ONE_M;
    for (int i = 255; i >= 0; --i) {
        acc = fmul(acc, acc);
        if ((e->l[i / 64] >> (i % 64)) & 1) acc = fmul(acc, a);
    }
    return acc;
}

static fe finv(fe a) {                /* Fermat: a^(P-2) */
    fe e = P;
    e.l[0] -= 2;
    return fpow(a, &e);
}

static void init(void) {
    if (inited) return;
    /* PINV = -P^{-1} mod 2^64 by Newton iteration */
    uint64_t inv = 1;
    for (int i = 0; i < 7; ++i) inv *= 2 - P.l[0] * inv;
    PINV = (uint64_t)0 - inv;
    /* 2^256 mod P by doubling 1 256 times; 2^512 mod P by doubling 512 times */
    fe x = fe_from_u64(1);
    for (int i = 0; i < 512; ++i) {
        x = fadd(x, x);
        if (i == 255) ONE_M = x;
    }
    R2 = x;
    inited = 1;
}

/* Signed integer -> Fr (x < 0 maps to r - |x|), canonical. */
static fe fe_from_i64(int64_t v) {
    if (v >= 0) return fe_from_u64((uint64_t)v);
    fe z = fe_from_u64(0);
    return fsub(z, fe_from_u64((uint64_t)(-(v + 1)) + 1));
}

/* ------------------------------------------------------------------ exported */

enum { ZKO_OK = 0, ZKO_E_SHAPE = 2, ZKO_E_NONCANONICAL = 3, ZKO_E_DUP_TABLE = 4,
       ZKO_E_NOT_IN_TABLE = 5, ZKO_E_DIV_ZERO_T = 6, ZKO_E_DIV_ZERO_S = 7, ZKO_E_OOM = 8 };

int zko_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void zko_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* Field primitives for the cross-check tests (canonical in/out). */
void zko_fr_mul(const fe *a, const fe *b, fe *out) { init(); *out = from_m(fmul(to_m(*a), to_m(*b))); }
void zko_fr_add(const fe *a, const fe *b, fe *out) { init(); *out = fadd(*a, *b); }
void zko_fr_sub(const fe *a, const fe *b, fe *out) { init(); *out = fsub(*a, *b); }
void zko_fr_inv(const fe *a, fe *out) { init(); *out = from_m(finv(to_m(*a))); }

/* S_i = x_i + alpha_f y_i; canonical out. */
void zko_pair_inputs(uint64_t n, const int32_t *x, const int32_t *y, const fe *alpha_f, fe *out) {
    init();
    fe af = to_m(*alpha_f);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) {
        fe xv = fe_from_i64(x[i]);
        fe yv = to_m(fe_from_i64(y[i]));
        out[i] = fadd(xv, from_m(fmul(af, yv)));
    }
}

void zko_int_inputs(uint64_t n, const int64_t *x, fe *out) {
    init();
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) out[i] = fe_from_i64(x[i]);
}

typedef struct { fe v; uint32_t idx; } keyed;

static int cmp_keyed(const void *pa, const void *pb) {
    const keyed *a = pa, *b = pb;
    for (int i = 3; i >= 0; --i) {
        if (a->v.l[i] != b->v.l[i]) return a->v.l[i] < b->v.l[i] ? -1 : 1;
    }
    return a->idx < b->idx ? -1 : (a->idx > b->idx);
}

static int cmp_fe(const fe *a, const fe *b) {
    for (int i = 3; i >= 0; --i) {
        if (a->l[i] != b->l[i]) return a->l[i] < b->l[i] ? -1 : 1;
    }
    return 0;
}

static int is_pow2(uint64_t x) { return x && !(x & (x - 1)); }
static int log2u(uint64_t x) { int k = 0; while ((1ULL << k) < x) ++k; return k; }

/* Batch inversion: out_i = 1/in_i (Montgomery in/out), chunked per thread, exact. */
static void batch_inverse(fe *out, const fe *in, uint64_t n) {
    int nt = zko_num_threads();
    uint64_t chunk = (n + nt - 1) / nt;
    #pragma omp parallel for schedule(static)
    for (int t = 0; t < nt; ++t) {
        uint64_t lo = (uint64_t)t * chunk, hi = lo + chunk < n ? lo + chunk : n;
        if (lo >= hi) continue;
        fe acc = ONE_M;
        for (uint64_t i = lo; i < hi; ++i) { out[i] = acc; acc = fmul(acc, in[i]); }  /* out_i = prod_{<i} */
        fe inv = finv(acc);
        for (uint64_t i = hi; i-- > lo;) { out[i] = fmul(out[i], inv); inv = fmul(inv, in[i]); }
    }
}

/* e~(u, .) on {0,1}^k, coordinate 0 = MSB: built by expanding the product formula one
 * coordinate at a time (new[2i] = old[i](1-u_c), new[2i+1] = old[i] u_c).  Montgomery in/out. */
static void eq_table(fe *out, const fe *u, int k) {
    fe *prev = (fe *)malloc(((size_t)1 << (k > 0 ? k - 1 : 0)) * sizeof(fe));
    out[0] = ONE_M;
    for (int c = 0; c < k; ++c) {
        uint64_t sz = 1ULL << c;
        memcpy(prev, out, sz * sizeof(fe));
        fe one_minus = fsub(ONE_M, u[c]);
        #pragma omp parallel for schedule(static) if (sz > 4096)
        for (int64_t i = 0; i < (int64_t)sz; ++i) {
            out[2 * i + 1] = fmul(prev[i], u[c]);
            out[2 * i] = fmul(prev[i], one_minus);
        }
    }
    free(prev);
}

/*
 * Full Protocol-1 computation (without commitments).
 * S: D canonical elements; T: N canonical elements (both 4 x u64 LE).
 * chal: beta, alpha1, alpha2, then u[0..d-1], then r[0..d-1] (canonical).
 * Outputs (any may be NULL except evals/finals): m (u32[N]), A (D), B (N),
 * evals (d x 4 canonical), finals (A, S, B, T, m) canonical.
 * mode: 0 = full (m, A, B computed here); 1 = sumcheck only on caller A, B, m (m_in as u32).
 */
int zko_tlookup(uint64_t D, uint64_t N, const fe *S, const fe *T, const fe *chal, int variant, int mode,
                const fe *A_in, const fe *B_in, const uint32_t *m_in,
                uint32_t *m_out, fe *A_out, fe *B_out, fe *evals, fe *finals, int64_t *err_index) {
    init();
    *err_index = -1;
    if (!is_pow2(D) || !is_pow2(N) || N > D) return ZKO_E_SHAPE;
    int d = log2u(D), n = log2u(N);
    fe beta = to_m(chal[0]), a1 = to_m(chal[1]), a2 = to_m(chal[2]);
    const fe *u = chal + 3, *r = chal + 3 + d;

    uint32_t *m = (uint32_t *)calloc(N, sizeof(uint32_t));
    fe *A = (fe *)malloc(D * sizeof(fe));
    fe *Sv = (fe *)malloc(D * sizeof(fe));
    fe *E = (fe *)malloc(D * sizeof(fe));
    fe *B = (fe *)malloc(N * sizeof(fe)), *Tv = (fe *)malloc(N * sizeof(fe));
    fe *Mv = (fe *)malloc(N * sizeof(fe)), *E2 = (fe *)malloc(N * sizeof(fe));
    fe *um = (fe *)malloc((d + 1) * sizeof(fe));
    fe *A2 = (fe *)malloc((D / 2 + 1) * sizeof(fe)), *S2 = (fe *)malloc((D / 2 + 1) * sizeof(fe));
    fe *Ed2 = (fe *)malloc((D / 2 + 1) * sizeof(fe));
    keyed *ks = NULL;
    int status = ZKO_OK;
    if (!m || !A || !Sv || !E || !B || !Tv || !Mv || !E2 || !um || !A2 || !S2 || !Ed2) { status = ZKO_E_OOM; goto done; }

    for (uint64_t j = 0; j < N; ++j) if (geq(&T[j], &P)) { *err_index = (int64_t)j; status = ZKO_E_NONCANONICAL; goto done; }
    for (uint64_t i = 0; i < D; ++i) if (geq(&S[i], &P)) { *err_index = (int64_t)i; status = ZKO_E_NONCANONICAL; goto done; }

    if (mode == 0) {
        /* m (Eq. hab22-coefs): sort (value, index) of T; duplicates -> smallest later index */
        ks = (keyed *)malloc(N * sizeof(keyed));
        if (!ks) { status = ZKO_E_OOM; goto done; }
        for (uint64_t j = 0; j < N; ++j) { ks[j].v = T[j]; ks[j].idx = (uint32_t)j; }
        qsort(ks, N, sizeof(keyed), cmp_keyed);
        int64_t dup = -1;
        for (uint64_t j = 1; j < N; ++j)
            if (fe_eq(ks[j].v, ks[j - 1].v) && (dup < 0 || ks[j].idx < dup)) dup = ks[j].idx;
        if (dup >= 0) { *err_index = dup; status = ZKO_E_DUP_TABLE; goto done; }
        int64_t miss = -1;
        for (uint64_t i = 0; i < D; ++i) {
            uint64_t lo = 0, hi = N;
            while (lo < hi) {
                uint64_t mid = (lo + hi) / 2;
                if (cmp_fe(&ks[mid].v, &S[i]) < 0) lo = mid + 1; else hi = mid;
            }
            if (lo < N && fe_eq(ks[lo].v, S[i])) m[ks[lo].idx]++;
            else { miss = (int64_t)i; break; }
        }
        if (miss >= 0) { *err_index = miss; status = ZKO_E_NOT_IN_TABLE; goto done; }
        /* A, B (Eq. hab22-invs); beta + T_j = 0 checked first, then beta + S_i = 0 */
        for (uint64_t j = 0; j < N; ++j) {
            Tv[j] = fadd(beta, to_m(T[j]));
            if (fe_is_zero(Tv[j])) { *err_index = (int64_t)j; status = ZKO_E_DIV_ZERO_T; goto done; }
        }
        #pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < (int64_t)D; ++i) Sv[i] = fadd(beta, to_m(S[i]));
        for (uint64_t i = 0; i < D; ++i)
            if (fe_is_zero(Sv[i])) { *err_index = (int64_t)i; status = ZKO_E_DIV_ZERO_S; goto done; }
        batch_inverse(A, Sv, D);
        batch_inverse(B, Tv, N);
        if (variant == 1)
            for (uint64_t j = 0; j < N; ++j) B[j] = fmul(B[j], to_m(fe_from_u64(m[j])));
    } else {
        memcpy(m, m_in, N * sizeof(uint32_t));
        #pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < (int64_t)D; ++i) A[i] = to_m(A_in[i]);
        for (uint64_t j = 0; j < N; ++j) B[j] = to_m(B_in[j]);
    }
    if (m_out) memcpy(m_out, m, N * sizeof(uint32_t));
    if (A_out) {
        #pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < (int64_t)D; ++i) A_out[i] = from_m(A[i]);
    }
    if (B_out) for (uint64_t j = 0; j < N; ++j) B_out[j] = from_m(B[j]);

    /* ---- sumcheck on Eq. tlookup-sumcheck ---- */
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)D; ++i) Sv[i] = to_m(S[i]);
    for (uint64_t j = 0; j < N; ++j) { Tv[j] = to_m(T[j]); Mv[j] = to_m(fe_from_u64(m[j])); }
    for (int c = 0; c < d; ++c) um[c] = to_m(u[c]);
    eq_table(E, um, d);                 /* e~(u, x) */
    eq_table(E2, um + (d - n), n);      /* e~(u[d-n:], j) */
    fe half = finv(to_m(fe_from_u64(2)));
    fe *Acur = A, *Scur = Sv, *Ecur = E, *Anx = A2, *Snx = S2, *Enx = Ed2;
    fe tau = fe_from_u64(0), tau_scale = ONE_M;   /* table term once fully bound; 2^{-(k-n)} */
    uint64_t len = D, tlen = N;
    int nt = zko_num_threads();
    fe *part = (fe *)calloc((size_t)nt * 4, sizeof(fe));
    if (!part) { status = ZKO_E_OOM; goto done; }
    for (int k = 1; k <= d; ++k) {
        uint64_t halfn = len / 2;
        memset(part, 0, (size_t)nt * 4 * sizeof(fe));
        #pragma omp parallel
        {
            int tid = 0;
#ifdef _OPENMP
            tid = omp_get_thread_num();
#endif
            fe acc[4] = {fe_from_u64(0), fe_from_u64(0), fe_from_u64(0), fe_from_u64(0)};
            #pragma omp for schedule(static)
            for (int64_t y = 0; y < (int64_t)halfn; ++y) {
                fe a0 = Acur[2 * y], s0 = Scur[2 * y], e0 = Ecur[2 * y];
                fe da = fsub(Acur[2 * y + 1], a0), ds = fsub(Scur[2 * y + 1], s0), de = fsub(Ecur[2 * y + 1], e0);
                fe at = a0, st = s0, et = e0;
                for (int t = 0; t < 4; ++t) {
                    if (t > 0) { at = fadd(at, da); st = fadd(st, ds); et = fadd(et, de); }
                    /* A_t (alpha1 e_t (S_t + beta) + 1) */
                    fe f = fmul(at, fadd(fmul(fmul(a1, et), fadd(st, beta)), ONE_M));
                    acc[t] = fadd(acc[t], f);
                }
            }
            for (int t = 0; t < 4; ++t) part[tid * 4 + t] = acc[t];
        }
        fe g[4] = {fe_from_u64(0), fe_from_u64(0), fe_from_u64(0), fe_from_u64(0)};
        for (int q = 0; q < nt; ++q) for (int t = 0; t < 4; ++t) g[t] = fadd(g[t], part[q * 4 + t]);
        /* table side */
        if (k <= n) {
            uint64_t th = tlen / 2;
            fe tg[4] = {fe_from_u64(0), fe_from_u64(0), fe_from_u64(0), fe_from_u64(0)};
            for (uint64_t y = 0; y < th; ++y) {
                fe b0 = B[2 * y], t0 = Tv[2 * y], m0 = Mv[2 * y], e0 = E2[2 * y];
                fe db = fsub(B[2 * y + 1], b0), dt = fsub(Tv[2 * y + 1], t0);
                fe dm = fsub(Mv[2 * y + 1], m0), de = fsub(E2[2 * y + 1], e0);
                fe bt = b0, ttv = t0, mt = m0, et = e0;
                for (int t = 0; t < 4; ++t) {
                    if (t > 0) { bt = fadd(bt, db); ttv = fadd(ttv, dt); mt = fadd(mt, dm); et = fadd(et, de); }
                    fe f;
                    if (variant == 0)   /* B (alpha2 e2 (T + beta) - m) */
                        f = fmul(bt, fsub(fmul(fmul(a2, et), fadd(ttv, beta)), mt));
                    else                /* -B + alpha2 e2 (B (T + beta) - m) */
                        f = fsub(fmul(fmul(a2, et), fsub(fmul(bt, fadd(ttv, beta)), mt)), bt);
                    tg[t] = fadd(tg[t], f);
                }
            }
            for (int t = 0; t < 4; ++t) g[t] = fadd(g[t], tg[t]);
            /* fold the table vectors with r_k */
            fe rk = to_m(r[k - 1]);
            for (uint64_t y = 0; y < th; ++y) {
                B[y] = fadd(B[2 * y], fmul(rk, fsub(B[2 * y + 1], B[2 * y])));
                Tv[y] = fadd(Tv[2 * y], fmul(rk, fsub(Tv[2 * y + 1], Tv[2 * y])));
                Mv[y] = fadd(Mv[2 * y], fmul(rk, fsub(Mv[2 * y + 1], Mv[2 * y])));
                E2[y] = fadd(E2[2 * y], fmul(rk, fsub(E2[2 * y + 1], E2[2 * y])));
            }
            tlen = th;
            if (k == n) {
                if (variant == 0) tau = fmul(B[0], fsub(fmul(fmul(a2, E2[0]), fadd(Tv[0], beta)), Mv[0]));
                else tau = fsub(fmul(fmul(a2, E2[0]), fsub(fmul(B[0], fadd(Tv[0], beta)), Mv[0])), B[0]);
            }
        } else {
            if (n == 0 && k == 1) {
                if (variant == 0) tau = fmul(B[0], fsub(fmul(fmul(a2, E2[0]), fadd(Tv[0], beta)), Mv[0]));
                else tau = fsub(fmul(fmul(a2, E2[0]), fsub(fmul(B[0], fadd(Tv[0], beta)), Mv[0])), B[0]);
            }
            tau_scale = fmul(tau_scale, half);
            fe c = fmul(tau, tau_scale);
            for (int t = 0; t < 4; ++t) g[t] = fadd(g[t], c);
        }
        for (int t = 0; t < 4; ++t) evals[(k - 1) * 4 + t] = from_m(g[t]);
        /* fold the D-side vectors with r_k: V' = V_0 + r_k (V_1 - V_0) */
        fe rk = to_m(r[k - 1]);
        #pragma omp parallel for schedule(static)
        for (int64_t y = 0; y < (int64_t)halfn; ++y) {
            Anx[y] = fadd(Acur[2 * y], fmul(rk, fsub(Acur[2 * y + 1], Acur[2 * y])));
            Snx[y] = fadd(Scur[2 * y], fmul(rk, fsub(Scur[2 * y + 1], Scur[2 * y])));
            Enx[y] = fadd(Ecur[2 * y], fmul(rk, fsub(Ecur[2 * y + 1], Ecur[2 * y])));
        }
        fe *t0 = Acur; Acur = Anx; Anx = t0;
        t0 = Scur; Scur = Snx; Snx = t0;
        t0 = Ecur; Ecur = Enx; Enx = t0;
        len = halfn;
    }
    free(part);
    finals[0] = from_m(Acur[0]);
    finals[1] = from_m(Scur[0]);
    finals[2] = from_m(B[0]);
    finals[3] = from_m(Tv[0]);
    finals[4] = from_m(Mv[0]);
done:
    free(m); free(A); free(Sv); free(E); free(B); free(Tv); free(Mv); free(E2); free(um); free(ks);
    free(A2); free(S2); free(Ed2);
    return status;
}

/* ------------------------------------------------------------------ streaming tier (pair inputs) */

/* canonical x + alpha_f y for int32 x, y (af_m: alpha_f in Montgomery form) -- as zko_pair_inputs */
static fe pair_value(int32_t x, int32_t y, const fe *af_m) {
    return fadd(fe_from_i64(x), from_m(fmul(*af_m, to_m(fe_from_i64(y)))));
}

/* the summand of Eq. tlookup-sumcheck at one point of the line, D side: A (alpha1 e (S + beta) + 1) */
static fe d_term(fe a, fe sv, fe e, fe a1, fe beta) { return fmul(a, fadd(fmul(fmul(a1, e), fadd(sv, beta)), ONE_M)); }

/* table side at one point of the line (PAPER variant / LOGUP variant) */
static fe t_term(fe b, fe t, fe m, fe e, fe a2, fe beta, int variant) {
    if (variant == 0) return fmul(b, fsub(fmul(fmul(a2, e), fadd(t, beta)), m));
    return fsub(fmul(fmul(a2, e), fsub(fmul(b, fadd(t, beta)), m)), b);
}

/* one round on `len` materialised elements of A, S, E: direct sums at t = 0..3 into g, fold with rk into the
 * first len/2 entries of the out arrays */
static void d_round(const fe *A, const fe *S, const fe *E, uint64_t len, fe *An, fe *Sn, fe *En, fe rk, fe a1,
                    fe beta, fe g[4]) {
    uint64_t halfn = len / 2;
    int nt = zko_num_threads();
    fe *part = (fe *)calloc((size_t)nt * 4, sizeof(fe));
    #pragma omp parallel
    {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        fe acc[4] = {fe_from_u64(0), fe_from_u64(0), fe_from_u64(0), fe_from_u64(0)};
        #pragma omp for schedule(static)
        for (int64_t y = 0; y < (int64_t)halfn; ++y) {
            fe a0 = A[2 * y], s0 = S[2 * y], e0 = E[2 * y];
            fe da = fsub(A[2 * y + 1], a0), ds = fsub(S[2 * y + 1], s0), de = fsub(E[2 * y + 1], e0);
            fe at = a0, st = s0, et = e0;
            for (int t = 0; t < 4; ++t) {
                if (t > 0) { at = fadd(at, da); st = fadd(st, ds); et = fadd(et, de); }
                acc[t] = fadd(acc[t], d_term(at, st, et, a1, beta));
            }
        }
        for (int t = 0; t < 4; ++t) part[tid * 4 + t] = acc[t];
    }
    for (int q = 0; q < nt; ++q) for (int t = 0; t < 4; ++t) g[t] = fadd(g[t], part[q * 4 + t]);
    free(part);
    #pragma omp parallel for schedule(static)
    for (int64_t y = 0; y < (int64_t)halfn; ++y) {
        An[y] = fadd(A[2 * y], fmul(rk, fsub(A[2 * y + 1], A[2 * y])));
        Sn[y] = fadd(S[2 * y], fmul(rk, fsub(S[2 * y + 1], S[2 * y])));
        En[y] = fadd(E[2 * y], fmul(rk, fsub(E[2 * y + 1], E[2 * y])));
    }
}

/*
 * x, y: D int32 (S_i = x_i + alpha_f y_i); tx, ty: N int32 (T_j = tx_j + alpha_f ty_j); alpha_f, chal canonical
 * (chal as in zko_tlookup).  s: rounds streamed block by block (0 <= s <= log2 D).  Outputs as zko_tlookup
 * (m_out, B_out may be NULL).  Errors: E_SHAPE, E_DUP_TABLE(j), E_NOT_IN_TABLE(smallest i), E_DIV_ZERO_T(j),
 * E_DIV_ZERO_S(smallest i), E_OOM.
 */
int zko_tlookup_pair_stream(uint64_t D, uint64_t N, const int32_t *x, const int32_t *y, const int32_t *tx,
                            const int32_t *ty, const fe *alpha_f, const fe *chal, int variant, int s,
                            uint32_t *m_out, fe *B_out, fe *evals, fe *finals, int64_t *err_index) {
    init();
    *err_index = -1;
    if (!is_pow2(D) || !is_pow2(N) || N > D) return ZKO_E_SHAPE;
    int d = log2u(D), n = log2u(N);
    if (s < 0 || s > d) return ZKO_E_SHAPE;
    fe beta = to_m(chal[0]), a1 = to_m(chal[1]), a2 = to_m(chal[2]);
    const fe *u = chal + 3, *r = chal + 3 + d;
    fe af = to_m(*alpha_f);
    int nt = zko_num_threads();
    int status = ZKO_OK;
    uint64_t Ds = D >> s;                       /* materialised length after the streamed rounds */
    fe *T = malloc(N * sizeof(fe)), *B = malloc(N * sizeof(fe)), *Tv = malloc(N * sizeof(fe));
    fe *Mv = malloc(N * sizeof(fe)), *E2 = malloc(N * sizeof(fe)), *um = malloc((d + 1) * sizeof(fe));
    keyed *ks = malloc(N * sizeof(keyed));
    uint32_t *m = calloc(N, sizeof(uint32_t)), *mth = calloc((size_t)nt * N, sizeof(uint32_t));
    fe *dg = calloc((size_t)d * 4, sizeof(fe)), *tg = calloc((size_t)d * 4, sizeof(fe));
    int h = d / 2;                              /* e~(u, x) = e~(u[0:d-h], x >> h) e~(u[d-h:], x mod 2^h) */
    fe *Ehi = malloc(((size_t)1 << (d - h)) * sizeof(fe)), *Elo = malloc(((size_t)1 << h) * sizeof(fe));
    fe *A3 = malloc(Ds * sizeof(fe)), *S3 = malloc(Ds * sizeof(fe)), *E3 = malloc(Ds * sizeof(fe));
    fe *A4 = malloc((Ds / 2 + 1) * sizeof(fe)), *S4 = malloc((Ds / 2 + 1) * sizeof(fe)), *E4 = malloc((Ds / 2 + 1) * sizeof(fe));
    int64_t *miss_th = malloc(nt * sizeof(int64_t)), *zero_th = malloc(nt * sizeof(int64_t));
    fe *gth = calloc((size_t)nt * (s + 1) * 4, sizeof(fe));
    if (!T || !B || !Tv || !Mv || !E2 || !um || !ks || !m || !mth || !dg || !tg || !Ehi || !Elo || !A3 || !S3 || !E3 ||
        !A4 || !S4 || !E4 || !miss_th || !zero_th || !gth) { status = ZKO_E_OOM; goto done; }

    /* T, distinctness (smallest later duplicate index), as zko_tlookup */
    for (uint64_t j = 0; j < N; ++j) { T[j] = pair_value(tx[j], ty[j], &af); ks[j].v = T[j]; ks[j].idx = (uint32_t)j; }
    qsort(ks, N, sizeof(keyed), cmp_keyed);
    {
        int64_t dup = -1;
        for (uint64_t j = 1; j < N; ++j)
            if (fe_eq(ks[j].v, ks[j - 1].v) && (dup < 0 || ks[j].idx < dup)) dup = ks[j].idx;
        if (dup >= 0) { *err_index = dup; status = ZKO_E_DUP_TABLE; goto done; }
    }
    /* m_j = #{i : S_i = T_j} (Eq. hab22-coefs), binary search in the sorted table; per-thread counts */
    for (int t = 0; t < nt; ++t) miss_th[t] = -1;
    #pragma omp parallel
    {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        uint32_t *mc = mth + (size_t)tid * N;
        #pragma omp for schedule(static)
        for (int64_t i = 0; i < (int64_t)D; ++i) {
            fe sv = pair_value(x[i], y[i], &af);
            uint64_t lo = 0, hi = N;
            while (lo < hi) {
                uint64_t mid = (lo + hi) / 2;
                if (cmp_fe(&ks[mid].v, &sv) < 0) lo = mid + 1; else hi = mid;
            }
            if (lo < N && fe_eq(ks[lo].v, sv)) mc[ks[lo].idx]++;
            else if (miss_th[tid] < 0) miss_th[tid] = i;   /* static schedule: increasing i per thread */
        }
    }
    {
        int64_t miss = -1;
        for (int t = 0; t < nt; ++t) if (miss_th[t] >= 0 && (miss < 0 || miss_th[t] < miss)) miss = miss_th[t];
        if (miss >= 0) { *err_index = miss; status = ZKO_E_NOT_IN_TABLE; goto done; }
    }
    for (int t = 0; t < nt; ++t) for (uint64_t j = 0; j < N; ++j) m[j] += mth[(size_t)t * N + j];
    if (m_out) memcpy(m_out, m, N * sizeof(uint32_t));
    /* B (Eq. hab22-invs); beta + T_j = 0 first */
    for (uint64_t j = 0; j < N; ++j) {
        Tv[j] = fadd(beta, to_m(T[j]));
        if (fe_is_zero(Tv[j])) { *err_index = (int64_t)j; status = ZKO_E_DIV_ZERO_T; goto done; }
    }
    batch_inverse(B, Tv, N);
    if (variant == 1) for (uint64_t j = 0; j < N; ++j) B[j] = fmul(B[j], to_m(fe_from_u64(m[j])));
    if (B_out) for (uint64_t j = 0; j < N; ++j) B_out[j] = from_m(B[j]);

    /* ---- table side, every round (N-sized vectors, weight rule of DESIGN.md §5 a8) */
    for (uint64_t j = 0; j < N; ++j) { Tv[j] = to_m(T[j]); Mv[j] = to_m(fe_from_u64(m[j])); }
    for (int c = 0; c < d; ++c) um[c] = to_m(u[c]);
    eq_table(E2, um + (d - n), n);
    {
        fe half = finv(to_m(fe_from_u64(2)));
        fe tau = fe_from_u64(0), tau_scale = ONE_M;
        uint64_t tlen = N;
        if (n == 0) tau = t_term(B[0], Tv[0], Mv[0], E2[0], a2, beta, variant);
        for (int k = 1; k <= d; ++k) {
            fe *g = tg + (size_t)(k - 1) * 4;
            if (k <= n) {
                uint64_t th = tlen / 2;
                for (uint64_t yy = 0; yy < th; ++yy) {
                    fe b0 = B[2 * yy], t0 = Tv[2 * yy], m0 = Mv[2 * yy], e0 = E2[2 * yy];
                    fe db = fsub(B[2 * yy + 1], b0), dt = fsub(Tv[2 * yy + 1], t0);
                    fe dm = fsub(Mv[2 * yy + 1], m0), de = fsub(E2[2 * yy + 1], e0);
                    fe bt = b0, ttv = t0, mt = m0, et = e0;
                    for (int t = 0; t < 4; ++t) {
                        if (t > 0) { bt = fadd(bt, db); ttv = fadd(ttv, dt); mt = fadd(mt, dm); et = fadd(et, de); }
                        g[t] = fadd(g[t], t_term(bt, ttv, mt, et, a2, beta, variant));
                    }
                }
                fe rk = to_m(r[k - 1]);
                for (uint64_t yy = 0; yy < th; ++yy) {
                    B[yy] = fadd(B[2 * yy], fmul(rk, fsub(B[2 * yy + 1], B[2 * yy])));
                    Tv[yy] = fadd(Tv[2 * yy], fmul(rk, fsub(Tv[2 * yy + 1], Tv[2 * yy])));
                    Mv[yy] = fadd(Mv[2 * yy], fmul(rk, fsub(Mv[2 * yy + 1], Mv[2 * yy])));
                    E2[yy] = fadd(E2[2 * yy], fmul(rk, fsub(E2[2 * yy + 1], E2[2 * yy])));
                }
                tlen = th;
                if (k == n) tau = t_term(B[0], Tv[0], Mv[0], E2[0], a2, beta, variant);
            } else {
                tau_scale = fmul(tau_scale, half);
                fe c = fmul(tau, tau_scale);
                for (int t = 0; t < 4; ++t) g[t] = c;
            }
        }
    }

    /* ---- D side: rounds 1..s block by block, A recomputed per batch of blocks */
    eq_table(Ehi, um, d - h);
    eq_table(Elo, um + (d - h), h);
    for (int t = 0; t < nt; ++t) zero_th[t] = -1;
    {
        const uint64_t bs = 1ULL << s;                                   /* block length */
        const uint64_t nb = Ds;                                          /* blocks */
        const uint64_t per = bs >= 4096 ? 1 : 4096 / bs;                 /* blocks per inversion batch */
        const uint64_t nbatch = (nb + per - 1) / per;
        fe rkm[64];
        for (int k = 1; k <= s; ++k) rkm[k] = to_m(r[k - 1]);
        #pragma omp parallel
        {
            int tid = 0;
#ifdef _OPENMP
            tid = omp_get_thread_num();
#endif
            fe *acc = gth + (size_t)tid * (s + 1) * 4;
            uint64_t blen = per * bs;
            fe *xs = malloc(blen * sizeof(fe)), *sv = malloc(blen * sizeof(fe)), *av = malloc(blen * sizeof(fe));
            fe *ev = malloc(bs * sizeof(fe));
            #pragma omp for schedule(static)
            for (int64_t q = 0; q < (int64_t)nbatch; ++q) {
                uint64_t b0 = (uint64_t)q * per, b1 = b0 + per < nb ? b0 + per : nb;
                uint64_t i0 = b0 * bs, cnt = (b1 - b0) * bs;
                for (uint64_t k = 0; k < cnt; ++k) {
                    sv[k] = to_m(pair_value(x[i0 + k], y[i0 + k], &af));
                    xs[k] = fadd(beta, sv[k]);
                    if (fe_is_zero(xs[k]) && zero_th[tid] < 0) zero_th[tid] = (int64_t)(i0 + k);
                }
                /* A = 1/(beta + S) for the batch: prefix products, one Fermat inversion, backward pass */
                fe p = ONE_M;
                for (uint64_t k = 0; k < cnt; ++k) { av[k] = p; if (!fe_is_zero(xs[k])) p = fmul(p, xs[k]); }
                fe iv = finv(p);
                for (uint64_t k = cnt; k-- > 0;) {
                    if (fe_is_zero(xs[k])) { av[k] = fe_from_u64(0); continue; }
                    av[k] = fmul(av[k], iv);
                    iv = fmul(iv, xs[k]);
                }
                for (uint64_t b = b0; b < b1; ++b) {
                    fe *ab = av + (b - b0) * bs, *sb = sv + (b - b0) * bs;
                    for (uint64_t k = 0; k < bs; ++k) {
                        uint64_t i = b * bs + k;
                        ev[k] = fmul(Ehi[i >> h], Elo[i & ((1ULL << h) - 1)]);
                    }
                    uint64_t len = bs;
                    for (int k = 1; k <= s; ++k) {
                        fe *g = acc + (size_t)k * 4;
                        for (uint64_t yy = 0; yy < len / 2; ++yy) {
                            fe a0 = ab[2 * yy], s0 = sb[2 * yy], e0 = ev[2 * yy];
                            fe da = fsub(ab[2 * yy + 1], a0), ds = fsub(sb[2 * yy + 1], s0), de = fsub(ev[2 * yy + 1], e0);
                            fe at = a0, st = s0, et = e0;
                            for (int t = 0; t < 4; ++t) {
                                if (t > 0) { at = fadd(at, da); st = fadd(st, ds); et = fadd(et, de); }
                                g[t] = fadd(g[t], d_term(at, st, et, a1, beta));
                            }
                        }
                        for (uint64_t yy = 0; yy < len / 2; ++yy) {
                            ab[yy] = fadd(ab[2 * yy], fmul(rkm[k], fsub(ab[2 * yy + 1], ab[2 * yy])));
                            sb[yy] = fadd(sb[2 * yy], fmul(rkm[k], fsub(sb[2 * yy + 1], sb[2 * yy])));
                            ev[yy] = fadd(ev[2 * yy], fmul(rkm[k], fsub(ev[2 * yy + 1], ev[2 * yy])));
                        }
                        len /= 2;
                    }
                    A3[b] = ab[0];
                    S3[b] = sb[0];
                    E3[b] = ev[0];
                }
            }
            free(xs); free(sv); free(av); free(ev);
        }
    }
    {
        int64_t z = -1;
        for (int t = 0; t < nt; ++t) if (zero_th[t] >= 0 && (z < 0 || zero_th[t] < z)) z = zero_th[t];
        if (z >= 0) { *err_index = z; status = ZKO_E_DIV_ZERO_S; goto done; }
    }
    for (int k = 1; k <= s; ++k)
        for (int t = 0; t < nt; ++t)
            for (int q = 0; q < 4; ++q) dg[(k - 1) * 4 + q] = fadd(dg[(k - 1) * 4 + q], gth[((size_t)t * (s + 1) + k) * 4 + q]);
    /* ---- rounds s+1..d on the materialised vectors */
    {
        fe *Ac = A3, *Sc = S3, *Ec = E3, *An = A4, *Sn = S4, *En = E4;
        uint64_t len = Ds;
        for (int k = s + 1; k <= d; ++k) {
            d_round(Ac, Sc, Ec, len, An, Sn, En, to_m(r[k - 1]), a1, beta, dg + (size_t)(k - 1) * 4);
            fe *t0 = Ac; Ac = An; An = t0;
            t0 = Sc; Sc = Sn; Sn = t0;
            t0 = Ec; Ec = En; En = t0;
            len /= 2;
        }
        finals[0] = from_m(Ac[0]);
        finals[1] = from_m(Sc[0]);
    }
    finals[2] = from_m(B[0]);
    finals[3] = from_m(Tv[0]);
    finals[4] = from_m(Mv[0]);
    for (int k = 0; k < d; ++k)
        for (int t = 0; t < 4; ++t) evals[k * 4 + t] = from_m(fadd(dg[k * 4 + t], tg[k * 4 + t]));
done:
    free(T); free(B); free(Tv); free(Mv); free(E2); free(um); free(ks); free(m); free(mth); free(dg); free(tg);
    free(Ehi); free(Elo); free(A3); free(S3); free(E3); free(A4); free(S4); free(E4); free(miss_th); free(zero_th);
    free(gth);
    return status;
}

// BLS12-381 G1 over F_q for the Hyrax/Pedersen commitments:
// y^2 = x^3 + 4.  F_q elements: 12 x 32-bit limbs, Montgomery form (R = 2^384), CIOS multiplication.
// Points: Jacobian (X, Y, Z) with x = X/Z^2, y = Y/Z^3, Z = 0 the point at infinity; tables and generators
// affine.  Constants were computed with Python big integers (q from the BLS12 family formula, pinned in
// tests/test_oracle_hyrax.py).
#pragma once
#include <stdint.h>

namespace zkl {

struct fq {
    uint32_t v[12];
};

__device__ __constant__ uint32_t kQ[12] = {0xffffaaabu, 0xb9feffffu, 0xb153ffffu, 0x1eabfffeu, 0xf6b0f624u, 0x6730d2a0u,
                                           0xf38512bfu, 0x64774b84u, 0x434bacd7u, 0x4b1ba7b6u, 0x397fe69au, 0x1a0111eau};
__device__ __constant__ uint32_t kQR1[12] = {0x0002fffdu, 0x76090000u, 0xc40c0002u, 0xebf4000bu, 0x53c758bau, 0x5f489857u,
                                             0x70525745u, 0x77ce5853u, 0xa256ec6du, 0x5c071a97u, 0xfa80e493u, 0x15f65ec3u};
__device__ __constant__ uint32_t kQR2[12] = {0x1c341746u, 0xf4df1f34u, 0x09d104f1u, 0x0a76e6a6u, 0x4c95b6d5u, 0x8de5476cu,
                                             0x939d83c0u, 0x67eb88a9u, 0xb519952du, 0x9a793e85u, 0x92cae3aau, 0x11988fe5u};
__device__ __constant__ uint32_t kQR3[12] = {0xd94ca1e0u, 0xed48ac6bu, 0x03a7adf8u, 0x315f831eu, 0x615e29ddu, 0x9a53352au,
                                             0x921e1761u, 0x34c04e5eu, 0x65724728u, 0x2512d435u, 0x91755d4du, 0x0aa63460u};
__device__ __constant__ uint32_t kQSqrtExp[12] = {0xffffeaabu, 0xee7fbfffu, 0xac54ffffu, 0x07aaffffu, 0x3dac3d89u,
                                                  0xd9cc34a8u, 0x3ce144afu, 0xd91dd2e1u, 0x90d2eb35u, 0x92c6e9edu,
                                                  0x8e5ff9a6u, 0x0680447au};
__device__ __constant__ uint32_t kQEulerExp[12] = {0xffffd555u, 0xdcff7fffu, 0x58a9ffffu, 0x0f55ffffu, 0x7b587b12u,
                                                   0xb3986950u, 0x79c2895fu, 0xb23ba5c2u, 0x21a5d66bu, 0x258dd3dbu,
                                                   0x1cbff34du, 0x0d0088f5u};
__device__ __constant__ uint32_t kQInvExp[12] = {0xffffaaa9u, 0xb9feffffu, 0xb153ffffu, 0x1eabfffeu, 0xf6b0f624u,
                                                 0x6730d2a0u, 0xf38512bfu, 0x64774b84u, 0x434bacd7u, 0x4b1ba7b6u,
                                                 0x397fe69au, 0x1a0111eau};
constexpr uint32_t kQPrime = 0xfffcfffdu;   // -q^{-1} mod 2^32
// the cofactor h = #E / r = 0x396c8c005555e1568c00aaab0000aaab
__device__ __constant__ uint32_t kH[4] = {0x0000aaabu, 0x8c00aaabu, 0x5555e156u, 0x396c8c00u};

__device__ __forceinline__ fq fq_const(const uint32_t* c) {
    fq x;
#pragma unroll
    for (int i = 0; i < 12; ++i) x.v[i] = c[i];
    return x;
}
__device__ __forceinline__ fq fq_zero() {
    fq x;
#pragma unroll
    for (int i = 0; i < 12; ++i) x.v[i] = 0;
    return x;
}
__device__ __forceinline__ fq fq_one() { return fq_const(kQR1); }
__device__ __forceinline__ bool fq_is_zero(const fq& a) {
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 12; ++i) x |= a.v[i];
    return x == 0;
}
__device__ __forceinline__ bool fq_eq(const fq& a, const fq& b) {
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 12; ++i) x |= a.v[i] ^ b.v[i];
    return x == 0;
}

// a >= q ?
__device__ __forceinline__ bool fq_geq_q(const fq& a) {
#pragma unroll
    for (int i = 11; i >= 0; --i)
        if (a.v[i] != kQ[i]) return a.v[i] > kQ[i];
    return true;
}

__device__ __forceinline__ void fq_sub_q(fq& a) {
    uint64_t br = 0;
#pragma unroll
    for (int i = 0; i < 12; ++i) {
        const uint64_t d = (uint64_t)a.v[i] - kQ[i] - br;
        a.v[i] = (uint32_t)d;
        br = (d >> 32) & 1;
    }
}

__device__ __forceinline__ fq fq_add(const fq& a, const fq& b) {
    fq s;
    uint64_t c = 0;
#pragma unroll
    for (int i = 0; i < 12; ++i) {
        c += (uint64_t)a.v[i] + b.v[i];
        s.v[i] = (uint32_t)c;
        c >>= 32;
    }
    if (c || fq_geq_q(s)) fq_sub_q(s);   // a + b < 2q < 2^384: c is always 0, kept for clarity
    return s;
}

__device__ __forceinline__ fq fq_sub(const fq& a, const fq& b) {
    fq d;
    uint64_t br = 0;
#pragma unroll
    for (int i = 0; i < 12; ++i) {
        const uint64_t t = (uint64_t)a.v[i] - b.v[i] - br;
        d.v[i] = (uint32_t)t;
        br = (t >> 32) & 1;
    }
    if (br) {   // add q back
        uint64_t c = 0;
#pragma unroll
        for (int i = 0; i < 12; ++i) {
            c += (uint64_t)d.v[i] + kQ[i];
            d.v[i] = (uint32_t)c;
            c >>= 32;
        }
    }
    return d;
}

__device__ __forceinline__ fq fq_neg(const fq& a) { return fq_is_zero(a) ? a : fq_sub(fq_zero(), a); }
__device__ __forceinline__ fq fq_dbl(const fq& a) { return fq_add(a, a); }

// Montgomery multiplication a b / 2^384 mod q (a, b < q), CIOS with aligned register pairs: the F_q analogue of
// fr_mul (csrc/fr.cuh).  The running value is X + Y 2^32, X = x0..x12 aligned at word 0 and Y = y0..y11 aligned at
// word 1; even products a_j b_i and m q_j go to X, odd ones to Y, so each lo/hi pair is one IMAD.WIDE.U32: 288
// of them plus 12 IMAD for m = x0 q' (q' = -q^{-1} mod 2^32).  The dropped carries are zero (checked word by word
// for random and extreme operands by tools/sim_fq_mul.py).
#define ZKQ_MP(dl, dh, a, b, al, ah) \
    "madc.lo.cc.u32 " dl ", " a ", " b ", " al ";\n\t" "madc.hi.cc.u32 " dh ", " a ", " b ", " ah ";\n\t"
#define ZKQ_REDUCE()                                                                                     \
    asm("{\n\t.reg .u32 m;\n\t" \
        "mul.lo.u32 m, %0, 0xfffcfffd;\n\t" \
        "mad.lo.cc.u32 %0, m, %25, %0;\n\t" \
        "madc.hi.cc.u32 %1, m, %25, %1;\n\t" \
        ZKQ_MP("%2", "%3", "m", "%27", "%2", "%3") \
        ZKQ_MP("%4", "%5", "m", "%29", "%4", "%5") \
        ZKQ_MP("%6", "%7", "m", "%31", "%6", "%7") \
        ZKQ_MP("%8", "%9", "m", "%33", "%8", "%9") \
        ZKQ_MP("%10", "%11", "m", "%35", "%10", "%11") \
        "addc.u32 %12, %12, 0;\n\t" \
        "mad.lo.cc.u32 %13, m, %26, %13;\n\t" \
        "madc.hi.cc.u32 %14, m, %26, %14;\n\t" \
        ZKQ_MP("%15", "%16", "m", "%28", "%15", "%16") \
        ZKQ_MP("%17", "%18", "m", "%30", "%17", "%18") \
        ZKQ_MP("%19", "%20", "m", "%32", "%19", "%20") \
        ZKQ_MP("%21", "%22", "m", "%34", "%21", "%22") \
        "madc.lo.cc.u32 %23, m, %36, %23;\n\t" \
        "madc.hi.u32 %24, m, %36, %24;\n\t}" \
        : "+r"(x[0]), "+r"(x[1]), "+r"(x[2]), "+r"(x[3]), "+r"(x[4]), "+r"(x[5]), "+r"(x[6]), "+r"(x[7]), "+r"(x[8]), "+r"(x[9]), "+r"(x[10]), "+r"(x[11]), "+r"(x[12]), "+r"(y[0]), "+r"(y[1]), "+r"(y[2]), "+r"(y[3]), "+r"(y[4]), "+r"(y[5]), "+r"(y[6]), "+r"(y[7]), "+r"(y[8]), "+r"(y[9]), "+r"(y[10]), "+r"(y[11]) \
        : "n"(0xffffaaab), "n"(0xb9feffff), "n"(0xb153ffff), "n"(0x1eabfffe), "n"(0xf6b0f624), "n"(0x6730d2a0), "n"(0xf38512bf), "n"(0x64774b84), "n"(0x434bacd7), "n"(0x4b1ba7b6), "n"(0x397fe69a), "n"(0x1a0111ea))

// One out-of-line copy by default: the group law inlines ~40 multiplications per kernel, and fully inlined
// (~33k SASS instructions) the MSM kernel is bound by instruction fetch.  ZKL_FQ_INLINE restores inlining.
#ifdef ZKL_FQ_INLINE
#define ZKL_FQ_MUL_ATTR __device__ __forceinline__
#else
#define ZKL_FQ_MUL_ATTR static __device__ __noinline__
#endif
ZKL_FQ_MUL_ATTR fq fq_mul(const fq a, const fq b) {
    uint32_t x[13], y[12];
    {   // iteration 0: plain products
        const uint32_t bi = b.v[0];
#pragma unroll
        for (int j = 0; j < 12; j += 2) {
            const uint64_t p = (uint64_t)a.v[j] * bi, o = (uint64_t)a.v[j + 1] * bi;
            x[j] = (uint32_t)p; x[j + 1] = (uint32_t)(p >> 32);
            y[j] = (uint32_t)o; y[j + 1] = (uint32_t)(o >> 32);
        }
        x[12] = 0;
    }
    ZKQ_REDUCE();
#pragma unroll
    for (int i = 1; i < 12; ++i) {
        const uint32_t bi = b.v[i];
        uint32_t X[13], Y[12], M0;
        asm("add.cc.u32 %0, %13, %14;\n\t"
            ZKQ_MP("%1", "%2", "%26", "%32", "%15", "%16")
            ZKQ_MP("%3", "%4", "%27", "%32", "%17", "%18")
            ZKQ_MP("%5", "%6", "%28", "%32", "%19", "%20")
            ZKQ_MP("%7", "%8", "%29", "%32", "%21", "%22")
            ZKQ_MP("%9", "%10", "%30", "%32", "%23", "%24")
            "madc.lo.cc.u32 %11, %31, %32, %25;\n\t"
            "madc.hi.u32 %12, %31, %32, 0;"
            : "=r"(M0), "=r"(Y[0]), "=r"(Y[1]), "=r"(Y[2]), "=r"(Y[3]), "=r"(Y[4]), "=r"(Y[5]), "=r"(Y[6]), "=r"(Y[7]), "=r"(Y[8]), "=r"(Y[9]), "=r"(Y[10]), "=r"(Y[11])
            : "r"(y[0]), "r"(x[1]), "r"(x[2]), "r"(x[3]), "r"(x[4]), "r"(x[5]), "r"(x[6]), "r"(x[7]), "r"(x[8]), "r"(x[9]), "r"(x[10]), "r"(x[11]), "r"(x[12]), "r"(a.v[1]), "r"(a.v[3]), "r"(a.v[5]), "r"(a.v[7]), "r"(a.v[9]), "r"(a.v[11]), "r"(bi));
        asm("mad.lo.cc.u32 %0, %25, %31, %13;\n\t"
            "madc.hi.cc.u32 %1, %25, %31, %14;\n\t"
            ZKQ_MP("%2", "%3", "%26", "%31", "%15", "%16")
            ZKQ_MP("%4", "%5", "%27", "%31", "%17", "%18")
            ZKQ_MP("%6", "%7", "%28", "%31", "%19", "%20")
            ZKQ_MP("%8", "%9", "%29", "%31", "%21", "%22")
            ZKQ_MP("%10", "%11", "%30", "%31", "%23", "%24")
            "addc.u32 %12, 0, 0;"
            : "=r"(X[0]), "=r"(X[1]), "=r"(X[2]), "=r"(X[3]), "=r"(X[4]), "=r"(X[5]), "=r"(X[6]), "=r"(X[7]), "=r"(X[8]), "=r"(X[9]), "=r"(X[10]), "=r"(X[11]), "=r"(X[12])
            : "r"(M0), "r"(y[1]), "r"(y[2]), "r"(y[3]), "r"(y[4]), "r"(y[5]), "r"(y[6]), "r"(y[7]), "r"(y[8]), "r"(y[9]), "r"(y[10]), "r"(y[11]), "r"(a.v[0]), "r"(a.v[2]), "r"(a.v[4]), "r"(a.v[6]), "r"(a.v[8]), "r"(a.v[10]), "r"(bi));
#pragma unroll
        for (int k = 0; k < 13; ++k) x[k] = X[k];
#pragma unroll
        for (int k = 0; k < 12; ++k) y[k] = Y[k];
        ZKQ_REDUCE();
    }
    // T = (x1..x12) + (y0..y11), both aligned at word 0; T < 2q
    fq r;
    asm("add.cc.u32 %0, %12, %24;\n\t"
        "addc.cc.u32 %1, %13, %25;\n\t"
        "addc.cc.u32 %2, %14, %26;\n\t"
        "addc.cc.u32 %3, %15, %27;\n\t"
        "addc.cc.u32 %4, %16, %28;\n\t"
        "addc.cc.u32 %5, %17, %29;\n\t"
        "addc.cc.u32 %6, %18, %30;\n\t"
        "addc.cc.u32 %7, %19, %31;\n\t"
        "addc.cc.u32 %8, %20, %32;\n\t"
        "addc.cc.u32 %9, %21, %33;\n\t"
        "addc.cc.u32 %10, %22, %34;\n\t"
        "addc.u32 %11, %23, %35;"
        : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]), "=r"(r.v[6]), "=r"(r.v[7]), "=r"(r.v[8]), "=r"(r.v[9]), "=r"(r.v[10]), "=r"(r.v[11])
        : "r"(x[1]), "r"(x[2]), "r"(x[3]), "r"(x[4]), "r"(x[5]), "r"(x[6]), "r"(x[7]), "r"(x[8]), "r"(x[9]), "r"(x[10]), "r"(x[11]), "r"(x[12]), "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]), "r"(y[4]), "r"(y[5]), "r"(y[6]), "r"(y[7]), "r"(y[8]), "r"(y[9]), "r"(y[10]), "r"(y[11]));
    if (fq_geq_q(r)) fq_sub_q(r);
    return r;
}
#undef ZKQ_REDUCE
#undef ZKQ_MP

// Portable CIOS (64-bit accumulation) for an unreduced left operand: a b / 2^384 mod q for any a < 2^384 and b < q
// (a b < R q).  Only the hash to the field uses it (a 384-bit digest times R^2); fq_mul needs a, b < q.
__device__ __forceinline__ fq fq_mul_wide_a(const fq& a, const fq& b) {
    uint32_t t[14];
#pragma unroll
    for (int i = 0; i < 14; ++i) t[i] = 0;
#pragma unroll
    for (int i = 0; i < 12; ++i) {
        uint64_t c = 0;
#pragma unroll
        for (int j = 0; j < 12; ++j) {
            c += (uint64_t)a.v[j] * b.v[i] + t[j];
            t[j] = (uint32_t)c;
            c >>= 32;
        }
        c += t[12];
        t[12] = (uint32_t)c;
        t[13] = (uint32_t)(c >> 32);
        const uint32_t m = t[0] * kQPrime;
        c = ((uint64_t)m * kQ[0] + t[0]) >> 32;
#pragma unroll
        for (int j = 1; j < 12; ++j) {
            c += (uint64_t)m * kQ[j] + t[j];
            t[j - 1] = (uint32_t)c;
            c >>= 32;
        }
        c += t[12];
        t[11] = (uint32_t)c;
        t[12] = t[13] + (uint32_t)(c >> 32);
    }
    fq r;
#pragma unroll
    for (int i = 0; i < 12; ++i) r.v[i] = t[i];
    if (t[12] || fq_geq_q(r)) fq_sub_q(r);
    return r;
}


__device__ __forceinline__ fq fq_sqr(const fq& a) { return fq_mul(a, a); }
__device__ __forceinline__ fq fq_to_mont(const fq& a) { return fq_mul(a, fq_const(kQR2)); }
__device__ __forceinline__ fq fq_from_mont(const fq& a) {
    fq one = fq_zero();
    one.v[0] = 1;
    return fq_mul(a, one);
}

// a^e, e given as 12 little-endian words (square-and-multiply, MSB first)
static __device__ __noinline__ fq fq_pow(const fq a, const uint32_t* e) {
    fq acc = fq_one();
    bool started = false;
    for (int i = 383; i >= 0; --i) {
        const uint32_t bit = (e[i >> 5] >> (i & 31)) & 1u;
        if (started) acc = fq_sqr(acc);
        if (bit) {
            acc = started ? fq_mul(acc, a) : a;
            started = true;
        }
    }
    return acc;
}

__device__ __forceinline__ fq fq_inv(const fq& a) { return fq_pow(a, kQInvExp); }   // 0 -> 0

// ---------------------------------------------------------------------------------- G1
struct g1j {   // Jacobian
    fq X, Y, Z;
};
struct g1a {   // affine (Montgomery coordinates); infinity flagged by inf
    fq x, y;
    uint32_t inf;
    uint32_t pad[3];
};

__device__ __forceinline__ g1j g1_infinity() {
    g1j p;
    p.X = fq_one();
    p.Y = fq_one();
    p.Z = fq_zero();
    return p;
}
__device__ __forceinline__ bool g1_is_inf(const g1j& p) { return fq_is_zero(p.Z); }

__device__ __forceinline__ g1j g1_from_affine(const g1a& a) {
    if (a.inf) return g1_infinity();
    g1j p;
    p.X = a.x;
    p.Y = a.y;
    p.Z = fq_one();
    return p;
}

// dbl-2009-l (a = 0): 2M + 5S
#ifdef ZKL_G1_NOINLINE
#define ZKL_G1_ATTR static __device__ __noinline__
#else
#define ZKL_G1_ATTR __device__ __forceinline__
#endif
ZKL_G1_ATTR g1j g1_dbl(const g1j& p) {
    if (g1_is_inf(p)) return p;
    const fq A = fq_sqr(p.X), B = fq_sqr(p.Y), C = fq_sqr(B);
    fq D = fq_sub(fq_sub(fq_sqr(fq_add(p.X, B)), A), C);
    D = fq_dbl(D);
    const fq E = fq_add(fq_dbl(A), A), F = fq_sqr(E);
    g1j r;
    r.X = fq_sub(F, fq_dbl(D));
    const fq C8 = fq_dbl(fq_dbl(fq_dbl(C)));
    r.Y = fq_sub(fq_mul(E, fq_sub(D, r.X)), C8);
    r.Z = fq_dbl(fq_mul(p.Y, p.Z));
    return r;
}

// madd-2007-bl: Jacobian + affine, 7M + 4S, with the exceptional cases (P = inf, Q = inf, P = Q, P = -Q)
ZKL_G1_ATTR g1j g1_add_affine(const g1j& p, const g1a& q) {
    if (q.inf) return p;
    if (g1_is_inf(p)) return g1_from_affine(q);
    const fq Z1Z1 = fq_sqr(p.Z);
    const fq U2 = fq_mul(q.x, Z1Z1);
    const fq S2 = fq_mul(q.y, fq_mul(p.Z, Z1Z1));
    const fq H = fq_sub(U2, p.X);
    const fq rr = fq_dbl(fq_sub(S2, p.Y));
    if (fq_is_zero(H)) {
        if (fq_is_zero(rr)) return g1_dbl(p);
        return g1_infinity();
    }
    const fq HH = fq_sqr(H);
    const fq I = fq_dbl(fq_dbl(HH));
    const fq J = fq_mul(H, I);
    const fq V = fq_mul(p.X, I);
    g1j r;
    r.X = fq_sub(fq_sub(fq_sqr(rr), J), fq_dbl(V));
    r.Y = fq_sub(fq_mul(rr, fq_sub(V, r.X)), fq_dbl(fq_mul(p.Y, J)));
    r.Z = fq_sub(fq_sub(fq_sqr(fq_add(p.Z, H)), Z1Z1), HH);
    return r;
}

// add-2007-bl: Jacobian + Jacobian, 11M + 5S, with the exceptional cases
__device__ __forceinline__ g1j g1_add(const g1j& p, const g1j& q) {
    if (g1_is_inf(p)) return q;
    if (g1_is_inf(q)) return p;
    const fq Z1Z1 = fq_sqr(p.Z), Z2Z2 = fq_sqr(q.Z);
    const fq U1 = fq_mul(p.X, Z2Z2), U2 = fq_mul(q.X, Z1Z1);
    const fq S1 = fq_mul(p.Y, fq_mul(q.Z, Z2Z2)), S2 = fq_mul(q.Y, fq_mul(p.Z, Z1Z1));
    const fq H = fq_sub(U2, U1);
    const fq rr = fq_dbl(fq_sub(S2, S1));
    if (fq_is_zero(H)) {
        if (fq_is_zero(rr)) return g1_dbl(p);
        return g1_infinity();
    }
    const fq I = fq_sqr(fq_dbl(H));
    const fq J = fq_mul(H, I);
    const fq V = fq_mul(U1, I);
    g1j r;
    r.X = fq_sub(fq_sub(fq_sqr(rr), J), fq_dbl(V));
    r.Y = fq_sub(fq_mul(rr, fq_sub(V, r.X)), fq_dbl(fq_mul(S1, J)));
    r.Z = fq_mul(fq_sub(fq_sub(fq_sqr(fq_add(p.Z, q.Z)), Z1Z1), Z2Z2), H);
    return r;
}

__device__ __forceinline__ g1a g1_to_affine(const g1j& p) {
    g1a a;
    a.pad[0] = a.pad[1] = a.pad[2] = 0;
    if (g1_is_inf(p)) {
        a.x = fq_zero();
        a.y = fq_zero();
        a.inf = 1;
        return a;
    }
    const fq zi = fq_inv(p.Z), zi2 = fq_sqr(zi);
    a.x = fq_mul(p.X, zi2);
    a.y = fq_mul(p.Y, fq_mul(zi2, zi));
    a.inf = 0;
    return a;
}

}  // namespace zkl

// Fr, the BLS12-381 scalar field, on sm_100a.
//
// Field: r = 0x73eda753299d7d483339d80809a1d80553bda402fffe5bfeffffffff00000001
// ("BLS12-381 ... |F| ~ 2^254", §7; value: DESIGN.md reading 1).
//
// Representation: 8 x 32-bit little-endian limbs in Montgomery form x*2^256 mod r, kept in
// [0, r).  In HBM field vectors are stored limb-interleaved (SoA): limb l of element i at
// limbs[l*n + i], so a warp reads 128 contiguous bytes per limb plane and 4 consecutive
// elements per thread with one 128-bit load per plane.
//
// Multiplication is CIOS Montgomery on the integer multiply-add pipe with PTX carry chains
// (mad.lo.cc / madc.hi.cc).  r = 1 (mod 2^32), so r' = -r^{-1} = -1 (mod 2^32) and the
// reduction quotient is q = -t0: no multiply.  Since 4r < 2^256, CIOS on inputs < r
// returns a value < 2r and one conditional subtraction restores [0, r).
#pragma once
#include <stdint.h>

namespace zkl {

struct fr {
    uint32_t v[8];
};

// r, little-endian 32-bit limbs
#define ZKL_R0 0x00000001u
#define ZKL_R1 0xffffffffu
#define ZKL_R2 0xfffe5bfeu
#define ZKL_R3 0x53bda402u
#define ZKL_R4 0x09a1d805u
#define ZKL_R5 0x3339d808u
#define ZKL_R6 0x299d7d48u
#define ZKL_R7 0x73eda753u

__device__ __forceinline__ fr fr_zero() {
    fr z;
#pragma unroll
    for (int i = 0; i < 8; ++i) z.v[i] = 0;
    return z;
}

// 1 in Montgomery form: 2^256 mod r
__device__ __forceinline__ fr fr_one() {
    fr o;
    o.v[0] = 0xfffffffeu; o.v[1] = 0x00000001u; o.v[2] = 0x00034802u; o.v[3] = 0x5884b7fau;
    o.v[4] = 0xecbc4ff5u; o.v[5] = 0x998c4fefu; o.v[6] = 0xacc5056fu; o.v[7] = 0x1824b159u;
    return o;
}

// R^2 mod r = 2^512 mod r (to-Montgomery multiplier)
__device__ __forceinline__ fr fr_r2() {
    fr o;
    o.v[0] = 0xf3f29c6du; o.v[1] = 0xc999e990u; o.v[2] = 0x87925c23u; o.v[3] = 0x2b6cedcbu;
    o.v[4] = 0x7254398fu; o.v[5] = 0x05d31496u; o.v[6] = 0x9f59ff11u; o.v[7] = 0x0748d9d9u;
    return o;
}

#define ZKL_FR_CONST(name, a0, a1, a2, a3, a4, a5, a6, a7)                                          \
    __device__ __forceinline__ fr name() {                                                          \
        fr o;                                                                                       \
        o.v[0] = a0; o.v[1] = a1; o.v[2] = a2; o.v[3] = a3; o.v[4] = a4; o.v[5] = a5; o.v[6] = a6;   \
        o.v[7] = a7;                                                                                \
        return o;                                                                                   \
    }
// Montgomery forms of small constants (x * 2^256 mod r)
ZKL_FR_CONST(fr_inv2_m, 0xffffffffu, 0x00000000u, 0x0001a401u, 0xac425bfdu, 0xf65e27fau, 0xccc627f7u, 0xd66282b7u, 0x0c1258acu)
ZKL_FR_CONST(fr_inv6_m, 0xaaaaaaabu, 0xffffffffu, 0x5554c954u, 0x1be9e156u, 0xade09d57u, 0x11134802u, 0x63347f18u, 0x514f37c6u)
ZKL_FR_CONST(fr_two_m, 0xfffffffcu, 0x00000003u, 0x00069004u, 0xb1096ff4u, 0xd9789feau, 0x33189fdfu, 0x598a0adfu, 0x304962b3u)
ZKL_FR_CONST(fr_three_m, 0xfffffffau, 0x00000005u, 0x0009d806u, 0x098e27eeu, 0xc634efe0u, 0xcca4efcfu, 0x064f104eu, 0x486e140du)
ZKL_FR_CONST(fr_five_m, 0xfffffff5u, 0x0000000au, 0x00120c0bu, 0x66d9f3dfu, 0x960bb7c5u, 0xcc83b7a7u, 0x363b9de5u, 0x04c9cf6du)
ZKL_FR_CONST(fr_six_m, 0xfffffff3u, 0x0000000cu, 0x0015540du, 0xbf5eabd9u, 0x82c807bau, 0x66100797u, 0xe300a355u, 0x1cee80c6u)

// 2^32 in Montgomery form (2^32 * 2^256 mod r) and its negation
ZKL_FR_CONST(fr_2p32_m, 0xcaaf6b13u, 0x355094eau, 0x69a568efu, 0xf6b10cb3u, 0x40cc3869u, 0xe2c926a6u, 0xed269aadu, 0x736a6d3bu)
ZKL_FR_CONST(fr_2p32_m_neg, 0x355094eeu, 0xcaaf6b14u, 0x9658f30fu, 0x5d0c974fu, 0xc8d59f9bu, 0x5070b161u, 0x3c76e29au, 0x00833a17u)

__device__ __forceinline__ bool fr_is_zero(const fr& a) {
    uint32_t x = a.v[0] | a.v[1] | a.v[2] | a.v[3] | a.v[4] | a.v[5] | a.v[6] | a.v[7];
    return x == 0;
}

__device__ __forceinline__ bool fr_eq(const fr& a, const fr& b) {
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) x |= a.v[i] ^ b.v[i];
    return x == 0;
}

// x in [0, 2r) -> [0, r): subtract r, keep the difference if no borrow.
__device__ __forceinline__ void fr_reduce_once(fr& x) {
    uint32_t d[8], borrow;
    asm("sub.cc.u32  %0, %9,  %17;\n\t"
        "subc.cc.u32 %1, %10, %18;\n\t"
        "subc.cc.u32 %2, %11, %19;\n\t"
        "subc.cc.u32 %3, %12, %20;\n\t"
        "subc.cc.u32 %4, %13, %21;\n\t"
        "subc.cc.u32 %5, %14, %22;\n\t"
        "subc.cc.u32 %6, %15, %23;\n\t"
        "subc.cc.u32 %7, %16, %24;\n\t"
        "subc.u32    %8, 0, 0;"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
          "=r"(borrow)
        : "r"(x.v[0]), "r"(x.v[1]), "r"(x.v[2]), "r"(x.v[3]), "r"(x.v[4]), "r"(x.v[5]), "r"(x.v[6]),
          "r"(x.v[7]), "n"(ZKL_R0), "n"(ZKL_R1), "n"(ZKL_R2), "n"(ZKL_R3), "n"(ZKL_R4), "n"(ZKL_R5),
          "n"(ZKL_R6), "n"(ZKL_R7));
    // borrow == 0xffffffff if x < r (keep x), 0 otherwise (take d)
#pragma unroll
    for (int i = 0; i < 8; ++i) x.v[i] = borrow ? x.v[i] : d[i];
}

__device__ __forceinline__ fr fr_add(const fr& a, const fr& b) {
    fr s;
    asm("add.cc.u32  %0, %8,  %16;\n\t"
        "addc.cc.u32 %1, %9,  %17;\n\t"
        "addc.cc.u32 %2, %10, %18;\n\t"
        "addc.cc.u32 %3, %11, %19;\n\t"
        "addc.cc.u32 %4, %12, %20;\n\t"
        "addc.cc.u32 %5, %13, %21;\n\t"
        "addc.cc.u32 %6, %14, %22;\n\t"
        "addc.u32    %7, %15, %23;"
        : "=r"(s.v[0]), "=r"(s.v[1]), "=r"(s.v[2]), "=r"(s.v[3]), "=r"(s.v[4]), "=r"(s.v[5]), "=r"(s.v[6]),
          "=r"(s.v[7])
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]), "r"(a.v[6]), "r"(a.v[7]),
          "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]), "r"(b.v[4]), "r"(b.v[5]), "r"(b.v[6]), "r"(b.v[7]));
    fr_reduce_once(s);   // a + b < 2r < 2^256
    return s;
}

// a - b mod r: compute a - b; on borrow add r.
__device__ __forceinline__ fr fr_sub(const fr& a, const fr& b) {
    fr d;
    uint32_t borrow;
    asm("sub.cc.u32  %0, %9,  %17;\n\t"
        "subc.cc.u32 %1, %10, %18;\n\t"
        "subc.cc.u32 %2, %11, %19;\n\t"
        "subc.cc.u32 %3, %12, %20;\n\t"
        "subc.cc.u32 %4, %13, %21;\n\t"
        "subc.cc.u32 %5, %14, %22;\n\t"
        "subc.cc.u32 %6, %15, %23;\n\t"
        "subc.cc.u32 %7, %16, %24;\n\t"
        "subc.u32    %8, 0, 0;"
        : "=r"(d.v[0]), "=r"(d.v[1]), "=r"(d.v[2]), "=r"(d.v[3]), "=r"(d.v[4]), "=r"(d.v[5]), "=r"(d.v[6]),
          "=r"(d.v[7]), "=r"(borrow)
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]), "r"(a.v[6]), "r"(a.v[7]),
          "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]), "r"(b.v[4]), "r"(b.v[5]), "r"(b.v[6]), "r"(b.v[7]));
    // add (r & borrow)
    asm("add.cc.u32  %0, %0, %8;\n\t"
        "addc.cc.u32 %1, %1, %9;\n\t"
        "addc.cc.u32 %2, %2, %10;\n\t"
        "addc.cc.u32 %3, %3, %11;\n\t"
        "addc.cc.u32 %4, %4, %12;\n\t"
        "addc.cc.u32 %5, %5, %13;\n\t"
        "addc.cc.u32 %6, %6, %14;\n\t"
        "addc.u32    %7, %7, %15;"
        : "+r"(d.v[0]), "+r"(d.v[1]), "+r"(d.v[2]), "+r"(d.v[3]), "+r"(d.v[4]), "+r"(d.v[5]), "+r"(d.v[6]),
          "+r"(d.v[7])
        : "r"(ZKL_R0 & borrow), "r"(ZKL_R1 & borrow), "r"(ZKL_R2 & borrow), "r"(ZKL_R3 & borrow),
          "r"(ZKL_R4 & borrow), "r"(ZKL_R5 & borrow), "r"(ZKL_R6 & borrow), "r"(ZKL_R7 & borrow));
    return d;
}

__device__ __forceinline__ fr fr_neg(const fr& a) { return fr_sub(fr_zero(), a); }

// ---------------------------------------------------------------------------------------
// Lazy forms.  fr_mul(a, b) needs a < r but accepts any b < 2^256 (the CIOS bound T < 2r only uses a < r and
// the 32-bit size of each limb of b), so a difference or sum feeding the b side need not be reduced.
// a - b as a + (r - b), in (0, 2r) for canonical a, b: two carry chains, no select.
__device__ __forceinline__ fr fr_sub_lazy(const fr& a, const fr& b) {
    fr d;
    asm("sub.cc.u32  %0, %8,  %16;\n\t"
        "subc.cc.u32 %1, %9,  %17;\n\t"
        "subc.cc.u32 %2, %10, %18;\n\t"
        "subc.cc.u32 %3, %11, %19;\n\t"
        "subc.cc.u32 %4, %12, %20;\n\t"
        "subc.cc.u32 %5, %13, %21;\n\t"
        "subc.cc.u32 %6, %14, %22;\n\t"
        "subc.u32    %7, %15, %23;"
        : "=r"(d.v[0]), "=r"(d.v[1]), "=r"(d.v[2]), "=r"(d.v[3]), "=r"(d.v[4]), "=r"(d.v[5]), "=r"(d.v[6]),
          "=r"(d.v[7])
        : "n"(ZKL_R0), "n"(ZKL_R1), "n"(ZKL_R2), "n"(ZKL_R3), "n"(ZKL_R4), "n"(ZKL_R5), "n"(ZKL_R6), "n"(ZKL_R7),
          "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]), "r"(b.v[4]), "r"(b.v[5]), "r"(b.v[6]), "r"(b.v[7]));
    fr s;
    asm("add.cc.u32  %0, %8,  %16;\n\t"
        "addc.cc.u32 %1, %9,  %17;\n\t"
        "addc.cc.u32 %2, %10, %18;\n\t"
        "addc.cc.u32 %3, %11, %19;\n\t"
        "addc.cc.u32 %4, %12, %20;\n\t"
        "addc.cc.u32 %5, %13, %21;\n\t"
        "addc.cc.u32 %6, %14, %22;\n\t"
        "addc.u32    %7, %15, %23;"
        : "=r"(s.v[0]), "=r"(s.v[1]), "=r"(s.v[2]), "=r"(s.v[3]), "=r"(s.v[4]), "=r"(s.v[5]), "=r"(s.v[6]),
          "=r"(s.v[7])
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]), "r"(a.v[6]), "r"(a.v[7]),
          "r"(d.v[0]), "r"(d.v[1]), "r"(d.v[2]), "r"(d.v[3]), "r"(d.v[4]), "r"(d.v[5]), "r"(d.v[6]), "r"(d.v[7]));
    return s;
}

// a + b without reduction, in [0, 2r) for canonical a, b
__device__ __forceinline__ fr fr_add_lazy(const fr& a, const fr& b) {
    fr s;
    asm("add.cc.u32  %0, %8,  %16;\n\t"
        "addc.cc.u32 %1, %9,  %17;\n\t"
        "addc.cc.u32 %2, %10, %18;\n\t"
        "addc.cc.u32 %3, %11, %19;\n\t"
        "addc.cc.u32 %4, %12, %20;\n\t"
        "addc.cc.u32 %5, %13, %21;\n\t"
        "addc.cc.u32 %6, %14, %22;\n\t"
        "addc.u32    %7, %15, %23;"
        : "=r"(s.v[0]), "=r"(s.v[1]), "=r"(s.v[2]), "=r"(s.v[3]), "=r"(s.v[4]), "=r"(s.v[5]), "=r"(s.v[6]),
          "=r"(s.v[7])
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]), "r"(a.v[6]), "r"(a.v[7]),
          "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]), "r"(b.v[4]), "r"(b.v[5]), "r"(b.v[6]), "r"(b.v[7]));
    return s;
}

// 288-bit accumulator of canonical values (no reduction per add); fr_acc_final reduces it mod r.
struct fr_acc {
    uint32_t v[9];
};

__device__ __forceinline__ fr_acc fr_acc_zero() {
    fr_acc a;
#pragma unroll
    for (int i = 0; i < 9; ++i) a.v[i] = 0;
    return a;
}

__device__ __forceinline__ void fr_acc_add(fr_acc& acc, const fr& x) {
    asm("add.cc.u32  %0, %0, %9;\n\t"
        "addc.cc.u32 %1, %1, %10;\n\t"
        "addc.cc.u32 %2, %2, %11;\n\t"
        "addc.cc.u32 %3, %3, %12;\n\t"
        "addc.cc.u32 %4, %4, %13;\n\t"
        "addc.cc.u32 %5, %5, %14;\n\t"
        "addc.cc.u32 %6, %6, %15;\n\t"
        "addc.cc.u32 %7, %7, %16;\n\t"
        "addc.u32    %8, %8, 0;"
        : "+r"(acc.v[0]), "+r"(acc.v[1]), "+r"(acc.v[2]), "+r"(acc.v[3]), "+r"(acc.v[4]), "+r"(acc.v[5]),
          "+r"(acc.v[6]), "+r"(acc.v[7]), "+r"(acc.v[8])
        : "r"(x.v[0]), "r"(x.v[1]), "r"(x.v[2]), "r"(x.v[3]), "r"(x.v[4]), "r"(x.v[5]), "r"(x.v[6]), "r"(x.v[7]));
}

__device__ __forceinline__ fr fr_mul(const fr& a, const fr& b);

// acc = hi 2^256 + lo  ->  (lo mod r) + hi (2^256 mod r); hi (2^256 mod r) = mont(R^2, hi)
__device__ __forceinline__ fr fr_acc_final(const fr_acc& acc) {
    fr lo;
#pragma unroll
    for (int i = 0; i < 8; ++i) lo.v[i] = acc.v[i];
    fr_reduce_once(lo);     // lo < 2^256 < 3r
    fr_reduce_once(lo);
    fr hi = fr_zero();
    hi.v[0] = acc.v[8];
    return fr_add(lo, fr_mul(fr_r2(), hi));
}

// ---------------------------------------------------------------------------------------
// Montgomery multiplication, CIOS with aligned register pairs.
//
// The running value T (< 2r) is held as X + Y*2^32: X = x0..x8 aligned at word 0, Y = y0..y7
// aligned at word 1.  Each iteration adds a_even*b_i and q*r_even to X (pairs (x_j, x_j+1), j
// even) and a_odd*b_i / 2^32 and q*r_odd / 2^32 to Y (pairs (y_j-1, y_j), j odd): every
// lo/hi product pair lands on an aligned register pair, so ptxas emits one IMAD.WIDE.U32(.X)
// per pair.  q = -x0 because r' = -1 (mod 2^32); r0 = 1 makes the j = 0 reduction pair an add.
// The division by 2^32 is a renaming: the next X is Y (with x1 merged into word 0) and the
// next Y is x2..x8 read as the addends of the next odd-product chain.  The Y chains never
// carry out: X >= 0 and T + a b_i + q r < 2r * 2^32 bound Y below 2^256 (checked word by word
// in tools/sim_fr_mul.py).
// ---------------------------------------------------------------------------------------
#define ZKL_MADPAIR(dl, dh, a, b, al, ah) \
    "madc.lo.cc.u32 " dl ", " a ", " b ", " al ";\n\t" "madc.hi.cc.u32 " dh ", " a ", " b ", " ah ";\n\t"

__device__ __forceinline__ fr fr_mul(const fr& a, const fr& b) {
    uint32_t x0, x1, x2, x3, x4, x5, x6, x7, x8;
    uint32_t y0, y1, y2, y3, y4, y5, y6, y7;
    // ---- iteration 0: plain products (T = 0)
    {
        const uint32_t bi = b.v[0];
        // one IMAD.WIDE.U32 per product (a lo/hi pair of mul.lo / mul.hi would cost an extra half-rate IMAD.HI)
        asm("{\n\t.reg .u64 p0, p1, p2, p3;\n\t"
            "mul.wide.u32 p0, %9, %13;\n\t"  "mul.wide.u32 p1, %10, %13;\n\t"
            "mul.wide.u32 p2, %11, %13;\n\t" "mul.wide.u32 p3, %12, %13;\n\t"
            "mov.b64 {%0, %1}, p0;\n\t" "mov.b64 {%2, %3}, p1;\n\t"
            "mov.b64 {%4, %5}, p2;\n\t" "mov.b64 {%6, %7}, p3;\n\t"
            "mov.u32 %8, 0;\n\t}"
            : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3), "=r"(x4), "=r"(x5), "=r"(x6), "=r"(x7), "=r"(x8)
            : "r"(a.v[0]), "r"(a.v[2]), "r"(a.v[4]), "r"(a.v[6]), "r"(bi));
        asm("{\n\t.reg .u64 p0, p1, p2, p3;\n\t"
            "mul.wide.u32 p0, %8, %12;\n\t"  "mul.wide.u32 p1, %9, %12;\n\t"
            "mul.wide.u32 p2, %10, %12;\n\t" "mul.wide.u32 p3, %11, %12;\n\t"
            "mov.b64 {%0, %1}, p0;\n\t" "mov.b64 {%2, %3}, p1;\n\t"
            "mov.b64 {%4, %5}, p2;\n\t" "mov.b64 {%6, %7}, p3;\n\t}"
            : "=r"(y0), "=r"(y1), "=r"(y2), "=r"(y3), "=r"(y4), "=r"(y5), "=r"(y6), "=r"(y7)
            : "r"(a.v[1]), "r"(a.v[3]), "r"(a.v[5]), "r"(a.v[7]), "r"(bi));
    }
// q r1 with r1 = 2^32 - 1 is not multiplied: q r1 = (q - 1) 2^32 + (2^32 - q) for q = -x0 != 0, so lo = x0 and
// hi = q - [x0 != 0] = ~x0 + [x0 == 0] (also right for q = 0): one borrow chain instead of a half-rate IMAD.HI
// (SURVEY.md §8(d) "224 slots"; tools/sim_fr_mul.py checks the chain).
#define ZKL_REDUCE_STEP()                                                                        \
    asm("{\n\t.reg .u32 q, xo, hi;\n\t"                                                          \
        "mov.u32 xo, %0;\n\t"                                                                    \
        "sub.cc.u32 q, 0, %0;\n\t"              /* borrow = [x0 != 0] */                         \
        "subc.u32 hi, q, 0;\n\t"                /* hi = q - [x0 != 0] = ~x0 + [x0 == 0] */       \
        "add.cc.u32 %0, %0, q;\n\t"                                                              \
        "addc.cc.u32 %1, %1, 0;\n\t"                                                             \
        ZKL_MADPAIR("%2", "%3", "q", "%18", "%2", "%3")                                          \
        ZKL_MADPAIR("%4", "%5", "q", "%20", "%4", "%5")                                          \
        ZKL_MADPAIR("%6", "%7", "q", "%22", "%6", "%7")                                          \
        "addc.u32 %8, %8, 0;\n\t"                                                                \
        "add.cc.u32  %9,  %9, xo;\n\t"                                                           \
        "addc.cc.u32 %10, %10, hi;\n\t"                                                          \
        ZKL_MADPAIR("%11", "%12", "q", "%19", "%11", "%12")                                      \
        ZKL_MADPAIR("%13", "%14", "q", "%21", "%13", "%14")                                      \
        "madc.lo.cc.u32 %15, q, %23, %15;\n\t"                                                   \
        "madc.hi.cc.u32 %16, q, %23, %16;\n\t}"    /* carry out is 0 (see header) */          \
        : "+r"(x0), "+r"(x1), "+r"(x2), "+r"(x3), "+r"(x4), "+r"(x5), "+r"(x6), "+r"(x7),          \
          "+r"(x8), "+r"(y0), "+r"(y1), "+r"(y2), "+r"(y3), "+r"(y4), "+r"(y5), "+r"(y6), "+r"(y7) \
        : "n"(ZKL_R1), "n"(ZKL_R2), "n"(ZKL_R3), "n"(ZKL_R4), "n"(ZKL_R5), "n"(ZKL_R6),           \
          "n"(ZKL_R7))
    ZKL_REDUCE_STEP();
#pragma unroll
    for (int i = 1; i < 8; ++i) {
        const uint32_t bi = b.v[i];
        uint32_t X0, X1, X2, X3, X4, X5, X6, X7, X8, Y0, Y1, Y2, Y3, Y4, Y5, Y6, Y7, M0;
        // merge x1 into word 0 of the new X (= old Y); odd products into the new Y, whose
        // addends are x2..x8 (the old X shifted down one word); the carry of the merge enters
        // the chain at word 1.
        //   outputs: %0 M0, %1..%8 Y0..Y7
        //   inputs : %9 y0, %10 x1, %11..%17 x2..x8, %18..%21 a1 a3 a5 a7, %22 bi
        asm("add.cc.u32 %0, %9, %10;\n\t"
            ZKL_MADPAIR("%1", "%2", "%18", "%22", "%11", "%12")
            ZKL_MADPAIR("%3", "%4", "%19", "%22", "%13", "%14")
            ZKL_MADPAIR("%5", "%6", "%20", "%22", "%15", "%16")
            "madc.lo.cc.u32 %7, %21, %22, %17;\n\t"
            "madc.hi.cc.u32 %8, %21, %22, 0;"
            : "=r"(M0), "=r"(Y0), "=r"(Y1), "=r"(Y2), "=r"(Y3), "=r"(Y4), "=r"(Y5), "=r"(Y6), "=r"(Y7)
            : "r"(y0), "r"(x1), "r"(x2), "r"(x3), "r"(x4), "r"(x5), "r"(x6), "r"(x7), "r"(x8),
              "r"(a.v[1]), "r"(a.v[3]), "r"(a.v[5]), "r"(a.v[7]), "r"(bi));
        // even products into the new X = (M0, y1..y7)
        //   outputs: %0..%8 X0..X8
        //   inputs : %9 M0, %10..%16 y1..y7, %17..%20 a0 a2 a4 a6, %21 bi
        asm("mad.lo.cc.u32  %0, %17, %21, %9;\n\t"
            "madc.hi.cc.u32 %1, %17, %21, %10;\n\t"
            ZKL_MADPAIR("%2", "%3", "%18", "%21", "%11", "%12")
            ZKL_MADPAIR("%4", "%5", "%19", "%21", "%13", "%14")
            ZKL_MADPAIR("%6", "%7", "%20", "%21", "%15", "%16")
            "addc.u32 %8, 0, 0;"
            : "=r"(X0), "=r"(X1), "=r"(X2), "=r"(X3), "=r"(X4), "=r"(X5), "=r"(X6), "=r"(X7), "=r"(X8)
            : "r"(M0), "r"(y1), "r"(y2), "r"(y3), "r"(y4), "r"(y5), "r"(y6), "r"(y7),
              "r"(a.v[0]), "r"(a.v[2]), "r"(a.v[4]), "r"(a.v[6]), "r"(bi));
        x0 = X0; x1 = X1; x2 = X2; x3 = X3; x4 = X4; x5 = X5; x6 = X6; x7 = X7; x8 = X8;
        y0 = Y0; y1 = Y1; y2 = Y2; y3 = Y3; y4 = Y4; y5 = Y5; y6 = Y6; y7 = Y7;
        ZKL_REDUCE_STEP();
    }
#undef ZKL_REDUCE_STEP
    // T = (x1..x8) + (y0..y7), both aligned at word 0; T < 2r.
    fr res;
    asm("add.cc.u32  %0, %8,  %16;\n\t"
        "addc.cc.u32 %1, %9,  %17;\n\t"
        "addc.cc.u32 %2, %10, %18;\n\t"
        "addc.cc.u32 %3, %11, %19;\n\t"
        "addc.cc.u32 %4, %12, %20;\n\t"
        "addc.cc.u32 %5, %13, %21;\n\t"
        "addc.cc.u32 %6, %14, %22;\n\t"
        "addc.u32    %7, %15, %23;"
        : "=r"(res.v[0]), "=r"(res.v[1]), "=r"(res.v[2]), "=r"(res.v[3]), "=r"(res.v[4]), "=r"(res.v[5]),
          "=r"(res.v[6]), "=r"(res.v[7])
        : "r"(x1), "r"(x2), "r"(x3), "r"(x4), "r"(x5), "r"(x6), "r"(x7), "r"(x8),
          "r"(y0), "r"(y1), "r"(y2), "r"(y3), "r"(y4), "r"(y5), "r"(y6), "r"(y7));
    fr_reduce_once(res);
    return res;
}

__device__ __forceinline__ fr fr_sqr(const fr& a) { return fr_mul(a, a); }

__device__ __forceinline__ fr fr_to_mont(const fr& a) { return fr_mul(a, fr_r2()); }

__device__ __forceinline__ fr fr_from_mont(const fr& a) {
    fr one = fr_zero();
    one.v[0] = 1;
    return fr_mul(a, one);
}

// R^3 mod r: fr_mul(y, R^3) = y R^2 turns y = (aR)^{-1} into the Montgomery form a^{-1} R
ZKL_FR_CONST(fr_r3, 0x439b73afu, 0xc62c1807u, 0x8cf06990u, 0x1b3e0d18u, 0xc7b5f418u, 0x73d13c71u, 0xc8db33e9u, 0x6e2a5bb9u)

__device__ __forceinline__ fr fr_modulus() {
    fr m;
    m.v[0] = ZKL_R0; m.v[1] = ZKL_R1; m.v[2] = ZKL_R2; m.v[3] = ZKL_R3;
    m.v[4] = ZKL_R4; m.v[5] = ZKL_R5; m.v[6] = ZKL_R6; m.v[7] = ZKL_R7;
    return m;
}

// x >>= s (0 < s < 32) on 256 bits
__device__ __forceinline__ void u256_shr(fr& x, uint32_t s) {
#pragma unroll
    for (int i = 0; i < 7; ++i) x.v[i] = __funnelshift_r(x.v[i], x.v[i + 1], s);
    x.v[7] >>= s;
}

// a - b on 256 bits (a >= b)
__device__ __forceinline__ fr u256_sub(const fr& a, const fr& b) {
    fr d;
    asm("sub.cc.u32  %0, %8,  %16;\n\t"
        "subc.cc.u32 %1, %9,  %17;\n\t"
        "subc.cc.u32 %2, %10, %18;\n\t"
        "subc.cc.u32 %3, %11, %19;\n\t"
        "subc.cc.u32 %4, %12, %20;\n\t"
        "subc.cc.u32 %5, %13, %21;\n\t"
        "subc.cc.u32 %6, %14, %22;\n\t"
        "subc.u32    %7, %15, %23;"
        : "=r"(d.v[0]), "=r"(d.v[1]), "=r"(d.v[2]), "=r"(d.v[3]), "=r"(d.v[4]), "=r"(d.v[5]), "=r"(d.v[6]),
          "=r"(d.v[7])
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]), "r"(a.v[6]), "r"(a.v[7]),
          "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]), "r"(b.v[4]), "r"(b.v[5]), "r"(b.v[6]), "r"(b.v[7]));
    return d;
}

__device__ __forceinline__ bool u256_geq(const fr& a, const fr& b) {
#pragma unroll
    for (int i = 7; i >= 0; --i)
        if (a.v[i] != b.v[i]) return a.v[i] > b.v[i];
    return true;
}

__device__ __forceinline__ bool u256_is_one(const fr& a) {
    return a.v[0] == 1 && (a.v[1] | a.v[2] | a.v[3] | a.v[4] | a.v[5] | a.v[6] | a.v[7]) == 0;
}

// x 2^{-s} mod r for canonical x, 0 < s <= 32: r = 1 (mod 2^32), so k = -x mod 2^s makes x + k r divisible
// by 2^s, and (x + k r) / 2^s < r / 2^s + r < 2r.
__device__ __forceinline__ fr fr_div_pow2(const fr& x, uint32_t s) {
    const uint32_t k = (0u - x.v[0]) & (s == 32 ? 0xffffffffu : ((1u << s) - 1u));
    uint32_t t[9];
    uint64_t c = 0;
    const fr m = fr_modulus();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        c += (uint64_t)k * m.v[i] + x.v[i];
        t[i] = (uint32_t)c;
        c >>= 32;
    }
    t[8] = (uint32_t)c;
    fr y;
    if (s == 32) {
#pragma unroll
        for (int i = 0; i < 8; ++i) y.v[i] = t[i + 1];
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) y.v[i] = __funnelshift_r(t[i], t[i + 1], s);
    }
    fr_reduce_once(y);
    return y;
}

// Strip the trailing zero bits of u (u != 0), dividing x by the same power of two mod r.
__device__ __forceinline__ void bgcd_strip(fr& u, fr& x) {
    while (u.v[0] == 0) {   // a whole zero word (rare)
#pragma unroll
        for (int i = 0; i < 7; ++i) u.v[i] = u.v[i + 1];
        u.v[7] = 0;
        x = fr_div_pow2(x, 32);
    }
    const uint32_t tz = __ffs(u.v[0]) - 1;
    if (tz) {
        u256_shr(u, tz);
        x = fr_div_pow2(x, tz);
    }
}

// Inverse in Montgomery form (0 -> 0): binary extended Euclid on the integer y = aR, then y^{-1} R^3 / R.
// Variable time (no secret-dependent timing concern on this path); about 5x lower latency than the
// 255-squaring Fermat chain it replaced, which matters because the top of every batched inversion is one thread.
static __device__ __noinline__ fr fr_inv(const fr a) {
    if (fr_is_zero(a)) return fr_zero();
    fr u = a, v = fr_modulus();
    fr x1 = fr_zero(), x2 = fr_zero();
    x1.v[0] = 1;
    // invariants: x1 a = u, x2 a = v (mod r) with a the integer aR; v odd after each strip
    bgcd_strip(u, x1);
#pragma unroll 1
    while (!u256_is_one(u) && !u256_is_one(v)) {
        if (u256_geq(u, v)) {
            u = u256_sub(u, v);
            x1 = fr_sub(x1, x2);
            bgcd_strip(u, x1);
        } else {
            v = u256_sub(v, u);
            x2 = fr_sub(x2, x1);
            bgcd_strip(v, x2);
        }
    }
    const fr y = u256_is_one(u) ? x1 : x2;
    return fr_mul(y, fr_r3());
}

// Fermat form a^(r-2) (4-bit fixed window: 252 squarings + at most 77 multiplications; 0 -> 0), kept as the
// cross-check of fr_inv in the microbenchmark.  Montgomery in, Montgomery out.
static __device__ __noinline__ fr fr_inv_fermat(const fr a) {
    // r - 2, little-endian 32-bit limbs
    const uint32_t e[8] = {0xffffffffu, 0xfffffffeu, 0xfffe5bfeu, 0x53bda402u,
                           0x09a1d805u, 0x3339d808u, 0x299d7d48u, 0x73eda753u};
    fr tab[16];
    tab[0] = fr_one();
    tab[1] = a;
#pragma unroll 1
    for (int i = 2; i < 16; ++i) tab[i] = fr_mul(tab[i - 1], a);
    fr acc = fr_one();
    bool started = false;
#pragma unroll 1
    for (int nib = 63; nib >= 0; --nib) {
        uint32_t w = (e[nib >> 3] >> ((nib & 7) * 4)) & 0xfu;
        if (started) {
            acc = fr_sqr(acc);
            acc = fr_sqr(acc);
            acc = fr_sqr(acc);
            acc = fr_sqr(acc);
        }
        if (w) {
            acc = started ? fr_mul(acc, tab[w]) : tab[w];
            started = true;
        }
    }
    return acc;
}

// ---------------------------------------------------------------------------------------
// Lazy (wide) accumulation of an eq-weighted sum  c = sum_y e_y X_y R^{-1} (mod r):
// the 512-bit products e_y X_y are summed without reduction (product scanning, 64 IMAD.WIDE and a carry word per
// column, against 112 IMAD.WIDE for a Montgomery product) and the sum is reduced once.  Bounds: e_y, X_y < 2r, so
// with at most 16 terms W < 64 r^2 < 2^516 fits 17 words; fr_wide_redc first brings the high half W_hi < 2^260
// below r by conditional subtractions of 16r, 8r, 4r, 2r, r (it changes W by multiples of r 2^256), then
// W < r 2^256 and one Montgomery reduction gives W R^{-1} mod r < 2r, made canonical.
struct fr_wide {
    uint32_t v[17];
};

__device__ __forceinline__ fr_wide fr_wide_zero() {
    fr_wide w;
#pragma unroll
    for (int i = 0; i < 17; ++i) w.v[i] = 0;
    return w;
}

// W += a * b
__device__ __forceinline__ void fr_wide_mac(fr_wide& W, const fr& a, const fr& b) {
    uint32_t t0 = 0, t1 = 0, t2 = 0;
#pragma unroll
    for (int c = 0; c < 16; ++c) {
        asm("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, 0;" : "+r"(t0), "+r"(t1) : "r"(W.v[c]));
#pragma unroll
        for (int j = (c > 7 ? c - 7 : 0); j <= (c < 7 ? c : 7); ++j)
            asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\tmadc.hi.cc.u32 %1, %3, %4, %1;\n\taddc.u32 %2, %2, 0;"
                : "+r"(t0), "+r"(t1), "+r"(t2) : "r"(a.v[j]), "r"(b.v[c - j]));
        W.v[c] = t0;
        t0 = t1;
        t1 = t2;
        t2 = 0;
    }
    W.v[16] += t0;   // t1 = 0: the sum stays below 2^544
}

// H = W[8..16] (9 words) -= m 2^s r  if  H >= m 2^s r
__device__ __forceinline__ void fr_wide_hi_sub_if(fr_wide& W, int s) {
    const uint32_t rl[8] = {ZKL_R0, ZKL_R1, ZKL_R2, ZKL_R3, ZKL_R4, ZKL_R5, ZKL_R6, ZKL_R7};
    uint32_t mr[9], d[9];
#pragma unroll
    for (int k = 0; k < 8; ++k) mr[k] = (rl[k] << s) | (k && s ? rl[k - 1] >> (32 - s) : 0u);
    mr[8] = s ? rl[7] >> (32 - s) : 0u;
    uint32_t borrow;
    asm("sub.cc.u32  %0, %10, %19;\n\t"
        "subc.cc.u32 %1, %11, %20;\n\t"
        "subc.cc.u32 %2, %12, %21;\n\t"
        "subc.cc.u32 %3, %13, %22;\n\t"
        "subc.cc.u32 %4, %14, %23;\n\t"
        "subc.cc.u32 %5, %15, %24;\n\t"
        "subc.cc.u32 %6, %16, %25;\n\t"
        "subc.cc.u32 %7, %17, %26;\n\t"
        "subc.cc.u32 %8, %18, %27;\n\t"
        "subc.u32    %9, 0, 0;"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]), "=r"(d[8]),
          "=r"(borrow)
        : "r"(W.v[8]), "r"(W.v[9]), "r"(W.v[10]), "r"(W.v[11]), "r"(W.v[12]), "r"(W.v[13]), "r"(W.v[14]),
          "r"(W.v[15]), "r"(W.v[16]), "r"(mr[0]), "r"(mr[1]), "r"(mr[2]), "r"(mr[3]), "r"(mr[4]), "r"(mr[5]),
          "r"(mr[6]), "r"(mr[7]), "r"(mr[8]));
#pragma unroll
    for (int k = 0; k < 9; ++k) W.v[8 + k] = borrow ? W.v[8 + k] : d[k];
}

// W R^{-1} mod r, canonical (W destroyed)
__device__ __forceinline__ fr fr_wide_redc(fr_wide& W) {
    fr_wide_hi_sub_if(W, 4);
    fr_wide_hi_sub_if(W, 3);
    fr_wide_hi_sub_if(W, 2);
    fr_wide_hi_sub_if(W, 1);
    fr_wide_hi_sub_if(W, 0);
    // W < r 2^256: eight Montgomery steps, q = -W[i] (r' = -1), W += q r 2^{32 i} (once per sum: plain 64-bit code)
    const uint32_t rl[8] = {ZKL_R0, ZKL_R1, ZKL_R2, ZKL_R3, ZKL_R4, ZKL_R5, ZKL_R6, ZKL_R7};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t q = 0u - W.v[i];
        uint64_t c = W.v[i] != 0;   // W[i] + q r0 = W[i] + q is 0 or 2^32
#pragma unroll
        for (int j = 1; j < 8; ++j) {
            c += (uint64_t)q * rl[j] + W.v[i + j];
            W.v[i + j] = (uint32_t)c;
            c >>= 32;
        }
#pragma unroll
        for (int k = i + 8; k < 17; ++k) {
            c += W.v[k];
            W.v[k] = (uint32_t)c;
            c >>= 32;
        }
    }
    fr o;
#pragma unroll
    for (int k = 0; k < 8; ++k) o.v[k] = W.v[8 + k];
    fr_reduce_once(o);
    return o;
}

// Canonical (non-Montgomery) a >= r ?
__device__ __forceinline__ bool fr_geq_modulus(const fr& x) {
    uint32_t borrow;
    asm("{\n\t.reg .u32 d;\n\t"
        "sub.cc.u32  d, %1, %9;\n\t"
        "subc.cc.u32 d, %2, %10;\n\t"
        "subc.cc.u32 d, %3, %11;\n\t"
        "subc.cc.u32 d, %4, %12;\n\t"
        "subc.cc.u32 d, %5, %13;\n\t"
        "subc.cc.u32 d, %6, %14;\n\t"
        "subc.cc.u32 d, %7, %15;\n\t"
        "subc.cc.u32 d, %8, %16;\n\t"
        "subc.u32    %0, 0, 0;\n\t}"
        : "=r"(borrow)
        : "r"(x.v[0]), "r"(x.v[1]), "r"(x.v[2]), "r"(x.v[3]), "r"(x.v[4]), "r"(x.v[5]), "r"(x.v[6]),
          "r"(x.v[7]), "n"(ZKL_R0), "n"(ZKL_R1), "n"(ZKL_R2), "n"(ZKL_R3), "n"(ZKL_R4), "n"(ZKL_R5),
          "n"(ZKL_R6), "n"(ZKL_R7));
    return borrow == 0;
}

}  // namespace zkl

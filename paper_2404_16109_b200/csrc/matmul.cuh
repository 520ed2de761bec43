// Matrix-multiplication sumcheck (Eq. matmul):
//     C~(u, v) = sum_{i in {0,1}^{log2 n}} A~(u, i) B~(i, v),   A in F^{m x n}, B in F^{n x p}.
// The prover's O(mn + np) part is the two restrictions a_i = A~(u, i) = sum_r e~(u, r) A[r][i] and
// b_i = B~(i, v) = sum_c B[i][c] e~(v, c).  The entries are quantised integers, so each term is
// an Fr eq weight times a 32-bit integer: it is accumulated as a plain 320-bit integer (8 IMAD.WIDE-class
// multiply-adds, no modular reduction) and reduced once per column chunk -- about 10x cheaper than an Fr
// multiplication, so the restrictions run near the HBM rate of reading A and B (4 B per entry).  The
// log2(n)-round degree-2 sumcheck on (a, b) reuses the chunked-round scheme of the tlookup path.
// Included by mm_api.cu.
#pragma once
#include "common.cuh"

namespace zkl {

constexpr int kMMThreads = 256;
constexpr int kMMChunkBits = 10;
constexpr int kMMChunk = 1 << kMMChunkBits;
constexpr int kMMChunkWarps = kMMChunk / 2 / 32;   // 512 threads, one pair each in the first chunk round
constexpr uint64_t kMMChunkMaxElems = (uint64_t)kMMChunk << 7;   // <= 128 chunks -> <= 128 values for the tail
constexpr int kMMRowChunk = 64;                    // rows of A per restriction block

struct MMRound {
    uint64_t base;    // partial rows of this round: [t][row], t = 0..2
    uint32_t rows;
};

// canonical -> Montgomery for the challenge vectors (u | v | r)
__global__ void k_mm_consts(const zkl_fr* __restrict__ in, int count, fr* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    fr x;
    for (int l = 0; l < 8; ++l) x.v[l] = in[i].w[l];
    out[i] = fr_to_mont(x);
}

// out[x] = e~(pt, bits(x)) = prod_j (bit_j ? pt_j : 1 - pt_j), coordinate 0 = MSB; CANONICAL (not Montgomery)
// AoS, since the restrictions multiply its integer value by the matrix entries
__global__ void k_mm_eq(const fr* __restrict__ pt, int bits, uint64_t count, fr* out) {
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < count; x += (uint64_t)gridDim.x * blockDim.x) {
        fr e = fr_one();
        for (int j = 0; j < bits; ++j) {
            const fr pj = pt[j];
            e = fr_mul(e, ((x >> (bits - 1 - j)) & 1) ? pj : fr_sub(fr_one(), pj));
        }
        out[x] = fr_from_mont(e);
    }
}

// 320-bit accumulator: acc += e * x (e < 2^256 canonical limbs, x < 2^32)
struct Wide {
    uint32_t w[10];
};

__device__ __forceinline__ void wide_zero(Wide& a) {
#pragma unroll
    for (int i = 0; i < 10; ++i) a.w[i] = 0;
}

__device__ __forceinline__ void wide_mad(Wide& a, const fr& e, uint32_t x) {
    asm("mad.lo.cc.u32  %0, %10, %18, %0;\n\t"
        "madc.lo.cc.u32 %1, %11, %18, %1;\n\t"
        "madc.lo.cc.u32 %2, %12, %18, %2;\n\t"
        "madc.lo.cc.u32 %3, %13, %18, %3;\n\t"
        "madc.lo.cc.u32 %4, %14, %18, %4;\n\t"
        "madc.lo.cc.u32 %5, %15, %18, %5;\n\t"
        "madc.lo.cc.u32 %6, %16, %18, %6;\n\t"
        "madc.lo.cc.u32 %7, %17, %18, %7;\n\t"
        "addc.cc.u32    %8, %8, 0;\n\t"
        "addc.u32       %9, %9, 0;\n\t"
        "mad.hi.cc.u32  %1, %10, %18, %1;\n\t"
        "madc.hi.cc.u32 %2, %11, %18, %2;\n\t"
        "madc.hi.cc.u32 %3, %12, %18, %3;\n\t"
        "madc.hi.cc.u32 %4, %13, %18, %4;\n\t"
        "madc.hi.cc.u32 %5, %14, %18, %5;\n\t"
        "madc.hi.cc.u32 %6, %15, %18, %6;\n\t"
        "madc.hi.cc.u32 %7, %16, %18, %7;\n\t"
        "madc.hi.cc.u32 %8, %17, %18, %8;\n\t"
        "addc.u32       %9, %9, 0;"
        : "+r"(a.w[0]), "+r"(a.w[1]), "+r"(a.w[2]), "+r"(a.w[3]), "+r"(a.w[4]), "+r"(a.w[5]), "+r"(a.w[6]),
          "+r"(a.w[7]), "+r"(a.w[8]), "+r"(a.w[9])
        : "r"(e.v[0]), "r"(e.v[1]), "r"(e.v[2]), "r"(e.v[3]), "r"(e.v[4]), "r"(e.v[5]), "r"(e.v[6]), "r"(e.v[7]),
          "r"(x));
}

// w mod r, canonical: w = hi 2^256 + lo, lo mod r by two conditional subtractions (lo < 2^256 < 3r) and
// hi 2^256 = hi R = mont(R^2, hi) mod r
__device__ __forceinline__ fr wide_reduce(const Wide& w) {
    fr lo;
#pragma unroll
    for (int i = 0; i < 8; ++i) lo.v[i] = w.w[i];
    fr_reduce_once(lo);
    fr_reduce_once(lo);
    fr hi = fr_zero();
    hi.v[0] = w.w[8];
    hi.v[1] = w.w[9];
    return fr_add(lo, fr_mul(fr_r2(), hi));
}

// sum_k e_k x_k with signed 32-bit x_k, from acc = sum e_k (x_k + 2^31) (unsigned) and esum = sum e_k:
// (acc - 2^31 esum) mod r, returned in Montgomery form
__device__ __forceinline__ fr wide_finish(const Wide& acc, const Wide& esum) {
    const fr es = wide_reduce(esum);
    Wide t;   // es 2^31 (< 2^286)
    t.w[0] = es.v[0] << 31;
#pragma unroll
    for (int i = 1; i < 8; ++i) t.w[i] = __funnelshift_l(es.v[i - 1], es.v[i], 31);
    t.w[8] = es.v[7] >> 1;
    t.w[9] = 0;
    const fr canon = fr_sub(wide_reduce(acc), wide_reduce(t));
    return fr_mul(canon, fr_r2());
}

__device__ __forceinline__ void wide_add_fr(Wide& a, const fr& e) {
    asm("add.cc.u32  %0, %0, %10;\n\t"
        "addc.cc.u32 %1, %1, %11;\n\t"
        "addc.cc.u32 %2, %2, %12;\n\t"
        "addc.cc.u32 %3, %3, %13;\n\t"
        "addc.cc.u32 %4, %4, %14;\n\t"
        "addc.cc.u32 %5, %5, %15;\n\t"
        "addc.cc.u32 %6, %6, %16;\n\t"
        "addc.cc.u32 %7, %7, %17;\n\t"
        "addc.cc.u32 %8, %8, 0;\n\t"
        "addc.u32    %9, %9, 0;"
        : "+r"(a.w[0]), "+r"(a.w[1]), "+r"(a.w[2]), "+r"(a.w[3]), "+r"(a.w[4]), "+r"(a.w[5]), "+r"(a.w[6]),
          "+r"(a.w[7]), "+r"(a.w[8]), "+r"(a.w[9])
        : "r"(e.v[0]), "r"(e.v[1]), "r"(e.v[2]), "r"(e.v[3]), "r"(e.v[4]), "r"(e.v[5]), "r"(e.v[6]), "r"(e.v[7]));
}

// a-restriction: partial[chunk][i] = sum_{r in chunk} e~(u, r) A[r][i] (Montgomery, AoS), one thread per column,
// a block per (256 columns, kMMRowChunk rows); the chunk's (canonical) eq weights staged in shared memory.
// 2^31 sum_k e_k mod r (canonical), the offset correction of a whole row chunk
__device__ __forceinline__ fr offset_correction(const Wide& esum) {
    const fr es = wide_reduce(esum);
    Wide t;
    t.w[0] = es.v[0] << 31;
#pragma unroll
    for (int i = 1; i < 8; ++i) t.w[i] = __funnelshift_l(es.v[i - 1], es.v[i], 31);
    t.w[8] = es.v[7] >> 1;
    t.w[9] = 0;
    return wide_reduce(t);
}

__global__ void __launch_bounds__(kMMThreads)
k_mm_restrict_rows(const int32_t* __restrict__ A, uint64_t m, uint64_t n, const fr* __restrict__ Eu, fr* partial) {
    __shared__ fr e[kMMRowChunk];
    __shared__ fr corr;
    const uint64_t r0 = (uint64_t)blockIdx.y * kMMRowChunk;
    const int rows = (int)(m - r0 < (uint64_t)kMMRowChunk ? m - r0 : (uint64_t)kMMRowChunk);
    for (int j = threadIdx.x; j < rows; j += blockDim.x) e[j] = Eu[r0 + j];
    __syncthreads();
    if (threadIdx.x == 0) {   // the chunk's sum of weights is the same for every column: once per CTA
        Wide es;
        wide_zero(es);
        for (int j = 0; j < rows; ++j) wide_add_fr(es, e[j]);
        corr = offset_correction(es);
    }
    __syncthreads();
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Wide acc;
    wide_zero(acc);
    const int32_t* col = A + r0 * n + i;
#pragma unroll 16
    for (int j = 0; j < rows; ++j) {
        const uint32_t x = (uint32_t)__ldg(col + (uint64_t)j * n) + 0x80000000u;   // x + 2^31
        wide_mad(acc, e[j], x);
    }
    partial[(uint64_t)blockIdx.y * n + i] = fr_mul(fr_sub(wide_reduce(acc), corr), fr_r2());
}

// a_i = sum over row chunks of partial[.][i]  (SoA Montgomery)
__global__ void k_mm_sum_chunks(const fr* __restrict__ partial, uint64_t nchunks, uint64_t n, uint32_t* a) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        fr s = fr_zero();
        for (uint64_t c = 0; c < nchunks; ++c) s = fr_add(s, partial[c * n + i]);
        st_fr(a, n, i, s);
    }
}

// b-restriction: b_i = sum_c B[i][c] e~(v, c): one warp per row (coalesced over c), per-lane wide sums,
// reduced to Fr per lane and summed over the warp.
__global__ void __launch_bounds__(kMMThreads)
k_mm_restrict_cols(const int32_t* __restrict__ B, uint64_t n, uint64_t p, const fr* __restrict__ Ev, uint32_t* b) {
    const uint64_t row = (uint64_t)blockIdx.x * (kMMThreads / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    Wide acc, es;
    wide_zero(acc);
    wide_zero(es);
    const int32_t* rp = B + row * p;
    for (uint64_t c = lane; c < p; c += 32) {
        const fr e = ld_fr_256(Ev + c);
        wide_mad(acc, e, (uint32_t)__ldg(rp + c) + 0x80000000u);
        wide_add_fr(es, e);
    }
    fr s = wide_finish(acc, es);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s = fr_add(s, shfl_down_fr(s, off));
    if (lane == 0) st_fr(b, n, row, s);
}

// b-restriction, tiled: a CTA owns kMMColRows consecutive rows of B; thread t walks the columns c = t, t + 256, ...
// holding e~(v, c) (canonical) in registers while it multiply-adds the kMMColRows entries B[i][c] into one
// 320-bit accumulator per row (each weight is loaded once per CTA instead of once per entry).  The accumulators
// are summed across the CTA as integers (shuffles, then shared memory) and reduced mod r once per row.
constexpr int kMMColRows = 4;

__device__ __forceinline__ void wide_add(Wide& a, const Wide& b) {
    asm("add.cc.u32  %0, %0, %10;\n\t"
        "addc.cc.u32 %1, %1, %11;\n\t"
        "addc.cc.u32 %2, %2, %12;\n\t"
        "addc.cc.u32 %3, %3, %13;\n\t"
        "addc.cc.u32 %4, %4, %14;\n\t"
        "addc.cc.u32 %5, %5, %15;\n\t"
        "addc.cc.u32 %6, %6, %16;\n\t"
        "addc.cc.u32 %7, %7, %17;\n\t"
        "addc.cc.u32 %8, %8, %18;\n\t"
        "addc.u32    %9, %9, %19;"
        : "+r"(a.w[0]), "+r"(a.w[1]), "+r"(a.w[2]), "+r"(a.w[3]), "+r"(a.w[4]), "+r"(a.w[5]), "+r"(a.w[6]),
          "+r"(a.w[7]), "+r"(a.w[8]), "+r"(a.w[9])
        : "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]), "r"(b.w[3]), "r"(b.w[4]), "r"(b.w[5]), "r"(b.w[6]), "r"(b.w[7]),
          "r"(b.w[8]), "r"(b.w[9]));
}

__device__ __forceinline__ void wide_warp_sum(Wide& a) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        Wide o;
#pragma unroll
        for (int i = 0; i < 10; ++i) o.w[i] = __shfl_down_sync(0xffffffffu, a.w[i], off);
        wide_add(a, o);
    }
}

__global__ void __launch_bounds__(kMMThreads, 3)
k_mm_restrict_cols_tiled(const int32_t* __restrict__ B, uint64_t n, uint64_t p, const fr* __restrict__ Ev,
                         uint32_t* b) {
    __shared__ Wide red[kMMColRows + 1][kMMThreads / 32];
    const uint64_t i0 = (uint64_t)blockIdx.x * kMMColRows;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    Wide acc[kMMColRows], es;
#pragma unroll
    for (int q = 0; q < kMMColRows; ++q) wide_zero(acc[q]);
    wide_zero(es);
#pragma unroll 2
    for (uint64_t c = t; c < p; c += kMMThreads) {
        const fr e = ld_fr_256(Ev + c);
        wide_add_fr(es, e);
#pragma unroll
        for (int q = 0; q < kMMColRows; ++q)
            wide_mad(acc[q], e, (uint32_t)__ldg(B + (i0 + q) * p + c) + 0x80000000u);
    }
#pragma unroll
    for (int q = 0; q < kMMColRows; ++q) wide_warp_sum(acc[q]);
    wide_warp_sum(es);
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < kMMColRows; ++q) red[q][warp] = acc[q];
        red[kMMColRows][warp] = es;
    }
    __syncthreads();
    if (t < kMMColRows) {
        Wide s = red[t][0], se = red[kMMColRows][0];
        for (int w = 1; w < kMMThreads / 32; ++w) {
            wide_add(s, red[t][w]);
            wide_add(se, red[kMMColRows][w]);
        }
        st_fr(b, n, i0 + t, wide_finish(s, se));
    }
}

// one degree-2 round pair: g(0) += a0 b0, g(1) += a1 b1, g(2) += (2 a1 - a0)(2 b1 - b0)
__device__ __forceinline__ void mm_pair(const fr& a0, const fr& a1, const fr& b0, const fr& b1, fr (&g)[3]) {
    g[0] = fr_add(g[0], fr_mul(a0, b0));
    g[1] = fr_add(g[1], fr_mul(a1, b1));
    const fr a2 = fr_sub(fr_add(a1, a1), a0), b2 = fr_sub(fr_add(b1, b1), b0);
    g[2] = fr_add(g[2], fr_mul(a2, b2));
}

// multi-block round k (only while the vectors are longer than kMMChunkMaxElems): fold with r_{k-1} on load
// (fold = 1) or not (k = 1), evaluate, write the folded vectors; one partial row per block
__global__ void __launch_bounds__(kMMThreads)
k_mm_round(const uint32_t* __restrict__ ain, const uint32_t* __restrict__ bin, uint64_t nin, int fold,
           const fr* __restrict__ rch, int k, uint32_t* aout, uint32_t* bout, fr* part, uint32_t rows) {
    const uint64_t len = fold ? nin / 2 : nin;   // elements of round k
    fr g[3] = {fr_zero(), fr_zero(), fr_zero()};
    const fr rp = fold ? rch[k - 2] : fr_zero();
    for (uint64_t y = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; y < len / 2; y += (uint64_t)gridDim.x * blockDim.x) {
        fr a0, a1, b0, b1;
        if (fold) {
            fr x[4], z[4];
            ld_fr4(ain, nin, 4 * y, x);
            ld_fr4(bin, nin, 4 * y, z);
            a0 = fr_add(x[0], fr_mul(rp, fr_sub_lazy(x[1], x[0])));
            a1 = fr_add(x[2], fr_mul(rp, fr_sub_lazy(x[3], x[2])));
            b0 = fr_add(z[0], fr_mul(rp, fr_sub_lazy(z[1], z[0])));
            b1 = fr_add(z[2], fr_mul(rp, fr_sub_lazy(z[3], z[2])));
            st_fr2(aout, len, 2 * y, a0, a1);
            st_fr2(bout, len, 2 * y, b0, b1);
        } else {
            fr x[2], z[2];
            ld_fr2(ain, nin, 2 * y, x);
            ld_fr2(bin, nin, 2 * y, z);
            a0 = x[0]; a1 = x[1]; b0 = z[0]; b1 = z[1];
        }
        mm_pair(a0, a1, b0, b1, g);
    }
    __shared__ fr scratch[3 * (kMMThreads / 32)];
    block_sum_fr<3>(g, scratch);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int t = 0; t < 3; ++t) part[(uint64_t)t * rows + blockIdx.x] = g[t];
    }
}

// chunked rounds kc .. kc + nr - 1: a CTA owns `chunk` consecutive round-(kc-1) pairs' worth of elements
// (folded on load with r_{kc-1} when fold, else the round-kc vectors themselves); one partial row per warp
__global__ void __launch_bounds__(kMMChunk / 2)
k_mm_chunk(const uint32_t* __restrict__ ain, const uint32_t* __restrict__ bin, uint64_t nin, int fold, int chunk,
           int nr, const fr* __restrict__ rch, int kc, const MMRound* __restrict__ rd, fr* parts, uint32_t* aout,
           uint32_t* bout) {
    extern __shared__ fr smem_fr[];
    fr* As = smem_fr;
    fr* Bs = smem_fr + kMMChunk;
    const int t = threadIdx.x;
    const uint64_t nchunks = gridDim.x;
    if (fold) {
        const fr rp = rch[kc - 2];
        const uint64_t base = 2 * (uint64_t)blockIdx.x * chunk;
        for (int i = t; i < chunk; i += blockDim.x) {
            fr x[2], z[2];
            ld_fr2(ain, nin, base + 2 * i, x);
            ld_fr2(bin, nin, base + 2 * i, z);
            As[i] = fr_add(x[0], fr_mul(rp, fr_sub_lazy(x[1], x[0])));
            Bs[i] = fr_add(z[0], fr_mul(rp, fr_sub_lazy(z[1], z[0])));
        }
    } else {
        const uint64_t base = (uint64_t)blockIdx.x * chunk;
        for (int i = t; i < chunk; i += blockDim.x) {
            As[i] = ld_fr(ain, nin, base + i);
            Bs[i] = ld_fr(bin, nin, base + i);
        }
    }
    __syncthreads();
    int len = chunk;
    for (int j = 0; j < nr; ++j) {
        const int k = kc + j;
        const int half = len / 2;
        fr g[3] = {fr_zero(), fr_zero(), fr_zero()};
        fr na, nb;
        if (t < half) {
            const fr a0 = As[2 * t], a1 = As[2 * t + 1], b0 = Bs[2 * t], b1 = Bs[2 * t + 1];
            mm_pair(a0, a1, b0, b1, g);
            const fr rk = rch[k - 1];
            na = fr_add(a0, fr_mul(rk, fr_sub_lazy(a1, a0)));
            nb = fr_add(b0, fr_mul(rk, fr_sub_lazy(b1, b0)));
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
            for (int q = 0; q < 3; ++q) g[q] = fr_add(g[q], shfl_down_fr(g[q], off));
        }
        if ((t & 31) == 0) {
            const MMRound r = rd[k - 1];
            const uint64_t row = (uint64_t)blockIdx.x * (blockDim.x / 32) + (t >> 5);
#pragma unroll
            for (int q = 0; q < 3; ++q) parts[r.base + (uint64_t)q * r.rows + row] = g[q];
        }
        __syncthreads();
        if (t < half) {
            As[t] = na;
            Bs[t] = nb;
        }
        __syncthreads();
        len = half;
    }
    if (t == 0) {
        st_fr(aout, nchunks, blockIdx.x, As[0]);
        st_fr(bout, nchunks, blockIdx.x, Bs[0]);
    }
}

// last rounds k0..L on n <= 128 elements in one warp; finals a~(w), b~(w)
__global__ void __launch_bounds__(32)
k_mm_tail(const uint32_t* __restrict__ ain, const uint32_t* __restrict__ bin, uint64_t n, const fr* __restrict__ rch,
          int k0, int L, const MMRound* __restrict__ rd, fr* parts, fr* fin) {
    __shared__ fr As[128], Bs[128];
    const int lane = threadIdx.x;
    for (int i = lane; i < (int)n; i += 32) {
        As[i] = ld_fr(ain, n, i);
        Bs[i] = ld_fr(bin, n, i);
    }
    __syncwarp();
    int len = (int)n;
    for (int k = k0; k <= L; ++k) {
        const int half = len / 2;
        const fr rk = rch[k - 1];
        fr g[3] = {fr_zero(), fr_zero(), fr_zero()};
        fr na[2], nb[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int y = lane + 32 * c;
            if (y < half) {
                const fr a0 = As[2 * y], a1 = As[2 * y + 1], b0 = Bs[2 * y], b1 = Bs[2 * y + 1];
                mm_pair(a0, a1, b0, b1, g);
                na[c] = fr_add(a0, fr_mul(rk, fr_sub_lazy(a1, a0)));
                nb[c] = fr_add(b0, fr_mul(rk, fr_sub_lazy(b1, b0)));
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
            for (int q = 0; q < 3; ++q) g[q] = fr_add(g[q], shfl_down_fr(g[q], off));
        }
        if (lane == 0) {
            const MMRound r = rd[k - 1];
#pragma unroll
            for (int q = 0; q < 3; ++q) parts[r.base + (uint64_t)q * r.rows] = g[q];
        }
        __syncwarp();
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int y = lane + 32 * c;
            if (y < half) {
                As[y] = na[c];
                Bs[y] = nb[c];
            }
        }
        __syncwarp();
        len = half;
    }
    if (lane == 0) {
        fin[0] = As[0];
        fin[1] = Bs[0];
    }
}

// per round: sum the partial rows -> g_k(0..2) canonical; claim (sum a_i b_i = g_1(0) + g_1(1), or a_0 b_0 when
// n = 1), finals canonical.  One block per round; block L (an extra one) writes claim and finals.
__global__ void k_mm_finish(const fr* __restrict__ parts, const MMRound* __restrict__ rd, int L,
                            const fr* __restrict__ fin, zkl_fr* out) {
    __shared__ fr scratch[3 * 8];
    const int k = blockIdx.x;   // 0-based round, or L
    if (k < L) {
        const MMRound r = rd[k];
        fr g[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            g[q] = fr_zero();
            for (uint32_t b = threadIdx.x; b < r.rows; b += blockDim.x) g[q] = fr_add(g[q], parts[r.base + (uint64_t)q * r.rows + b]);
        }
        block_sum_fr<3>(g, scratch);
        if (threadIdx.x == 0) {
#pragma unroll
            for (int q = 0; q < 3; ++q) out[3 + 3 * k + q] = to_canon(g[q]);
            if (k == 0) out[0] = to_canon(fr_add(g[0], g[1]));
        }
    } else if (threadIdx.x == 0) {
        out[1] = to_canon(fin[0]);
        out[2] = to_canon(fin[1]);
        if (L == 0) out[0] = to_canon(fr_mul(fin[0], fin[1]));
    }
}

}  // namespace zkl

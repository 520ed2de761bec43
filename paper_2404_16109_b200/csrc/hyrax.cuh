// Hyrax / Pedersen commitments (Protocol 1 lines 261, 267-269, 275).
// Readings as in oracle/hyrax.py: S (D = rows x cols, row-major) is committed row by row,
// C_j = sum_i S[j cols + i] G_i + rho_j H, with G_0..G_{cols-1}, H hashed to BLS12-381 G1 by try-and-increment
// (SHA-256, cofactor cleared): no trusted setup.  Commit = a batch of `rows` MSMs sharing their bases, computed by
// windowed Straus with 4-bit windows over precomputed affine tables {d G_i : d = 0..15} (L2-resident for
// cols <= 2^13): one thread per (row, slice of 16 columns, 32-bit scalar chunk) keeps one Jacobian accumulator,
// multiplies it by 16 per window and adds T_i[digit] for every column of its slice (64 mixed additions per scalar
// in all, no buckets, no sort, no atomics); the partial sums are tree-reduced per (row, chunk), the chunks combined
// by Horner (2^32 steps) and each row normalised once.  Included by hx_api.cu.
#pragma once
#include "g1.cuh"
#include "common.cuh"
#include "sha256.cuh"

namespace zkl {

// canonical -> Montgomery for the evaluation point
__global__ void k_hx_consts(const zkl_fr* __restrict__ in, int count, fr* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    fr x;
    for (int l = 0; l < 8; ++l) x.v[l] = in[i].w[l];
    out[i] = fr_to_mont(x);
}

constexpr int kHxThreads = 128;
constexpr int kHxSlice = 16;     // columns per thread in the commit kernel
constexpr int kHxGroups = 8;     // 32-bit scalar chunks (8 windows each) handled by separate threads
constexpr int kHxTab = 16;       // table entries per base (4-bit windows)

// try-and-increment hash to G1 for index i of the tag (oracle/hyrax.py hash_to_curve)
__device__ inline g1a hx_hash_to_curve(const uint8_t* tag, int tag_len, uint32_t i) {
    for (uint32_t ctr = 0;; ++ctr) {
        uint8_t msg[32 + 9];
        int p = 0;
        for (int k = 0; k < tag_len; ++k) msg[p++] = tag[k];
        for (int k = 0; k < 4; ++k) msg[p++] = (uint8_t)(i >> (8 * k));
        for (int k = 0; k < 4; ++k) msg[p++] = (uint8_t)(ctr >> (8 * k));
        uint8_t d0[32], d1[32];
        msg[p] = 0;
        sha256(msg, p + 1, d0);
        msg[p] = 1;
        sha256(msg, p + 1, d1);
        uint32_t w[16];
        for (int k = 0; k < 8; ++k) {
            w[k] = (uint32_t)d0[4 * k] | ((uint32_t)d0[4 * k + 1] << 8) | ((uint32_t)d0[4 * k + 2] << 16) |
                   ((uint32_t)d0[4 * k + 3] << 24);
            w[8 + k] = (uint32_t)d1[4 * k] | ((uint32_t)d1[4 * k + 1] << 8) | ((uint32_t)d1[4 * k + 2] << 16) |
                       ((uint32_t)d1[4 * k + 3] << 24);
        }
        // x = A + B 2^384 mod q, A = w[0..11], B = w[12..15]: Montgomery form = mont(A, R^2) + mont(B, R^3)
        fq A, Bq = fq_zero();
        for (int k = 0; k < 12; ++k) A.v[k] = w[k];
        for (int k = 0; k < 4; ++k) Bq.v[k] = w[12 + k];
        const fq x = fq_add(fq_mul_wide_a(A, fq_const(kQR2)), fq_mul(Bq, fq_const(kQR3)));   // A < 2^384 unreduced
        fq b4 = fq_zero();
        b4.v[0] = 4;
        const fq rhs = fq_add(fq_mul(fq_sqr(x), x), fq_to_mont(b4));
        if (fq_is_zero(rhs) || !fq_eq(fq_pow(rhs, kQEulerExp), fq_one())) continue;
        fq y = fq_pow(rhs, kQSqrtExp);
        // the smaller of y, q - y (canonical comparison)
        const fq yc = fq_from_mont(y), nyc = fq_from_mont(fq_neg(y));
        bool larger = false;
        for (int k = 11; k >= 0; --k)
            if (yc.v[k] != nyc.v[k]) {
                larger = yc.v[k] > nyc.v[k];
                break;
            }
        if (larger) y = fq_neg(y);
        g1a P;
        P.x = x;
        P.y = y;
        P.inf = 0;
        P.pad[0] = P.pad[1] = P.pad[2] = 0;
        g1j acc = g1_infinity();   // h P, MSB first
        for (int bit = 127; bit >= 0; --bit) {
            acc = g1_dbl(acc);
            if ((kH[bit >> 5] >> (bit & 31)) & 1u) acc = g1_add_affine(acc, P);
        }
        if (!g1_is_inf(acc)) return g1_to_affine(acc);
    }
}

// gens[0..cols-1] = G_i ("zkl-hyrax-G"), gens[cols] = H ("zkl-hyrax-H", 0)
__global__ void k_hx_gens(uint64_t cols, g1a* gens) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i > cols) return;
    const uint8_t tg[11] = {'z', 'k', 'l', '-', 'h', 'y', 'r', 'a', 'x', '-', 'G'};
    const uint8_t th[11] = {'z', 'k', 'l', '-', 'h', 'y', 'r', 'a', 'x', '-', 'H'};
    gens[i] = i < cols ? hx_hash_to_curve(tg, 11, (uint32_t)i) : hx_hash_to_curve(th, 11, 0);
}

// tab[g][i][d] = d 2^{32 g} gens[i], g = 0..7, d = 0..15 (affine; d = 0 the point at infinity): chunk g of a scalar
// adds from its own table, so the chunks' partial sums combine with additions only (no 32-doubling Horner per chunk)
__global__ void k_hx_tables(const g1a* __restrict__ gens, uint64_t count, g1a* tab) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= kHxGroups * count * kHxTab) return;
    const int g = (int)(k / (count * kHxTab));
    const uint64_t i = (k / kHxTab) % count;
    const int d = (int)(k % kHxTab);
    g1j acc = g1_infinity();
    for (int bit = 3; bit >= 0; --bit) {
        acc = g1_dbl(acc);
        if ((d >> bit) & 1) acc = g1_add_affine(acc, gens[i]);
    }
    if (!g1_is_inf(acc))
        for (int j = 0; j < 32 * g; ++j) acc = g1_dbl(acc);
    tab[k] = g1_to_affine(acc);
}

// hw[w][d] = d 16^w H, w = 0..63, d = 0..15 (affine): the blind rho H becomes 64 table additions, no doublings
__global__ void k_hx_htables(const g1a* __restrict__ H, g1a* hw) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= 64 * kHxTab) return;
    const int w = k / kHxTab, d = k % kHxTab;
    g1j acc = g1_infinity();
    for (int bit = 3; bit >= 0; --bit) {
        acc = g1_dbl(acc);
        if ((d >> bit) & 1) acc = g1_add_affine(acc, *H);
    }
    for (int i = 0; i < 4 * w; ++i) acc = g1_dbl(acc);
    hw[k] = g1_to_affine(acc);
}

// signed-magnitude canonical scalars: s in (r/2, r) is written as |s| = r - s with bit 255 set (s G = -(r - s) G),
// so small signed values (X, Y, the table columns) have zero limbs above the first and cost one 32-bit chunk
__global__ void k_hx_canon(const uint32_t* __restrict__ S, uint64_t n, uint32_t* out) {
    const fr half = [] {   // (r - 1) / 2
        fr h;
        h.v[0] = 0x80000000u; h.v[1] = 0x7fffffffu; h.v[2] = 0x7fff2dffu; h.v[3] = 0xa9ded201u;
        h.v[4] = 0x04d0ec02u; h.v[5] = 0x199cec04u; h.v[6] = 0x94cebea4u; h.v[7] = 0x39f6d3a9u;
        return h;
    }();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        fr c = fr_from_mont(ld_fr(S, n, i));
        bool neg = false;
        for (int l = 7; l >= 0; --l)
            if (c.v[l] != half.v[l]) {
                neg = c.v[l] > half.v[l];
                break;
            }
        if (neg) {
            c = fr_neg(c);
            c.v[7] |= 0x80000000u;
        }
        st_fr(out, n, i, c);
    }
}

// Work split: s = sum_g c_g 2^{32 g} (the 8 limbs of the canonical scalar), so
//   sum_i s_i G_i = sum_g 2^{32 g} Q_g,  Q_g = sum_i c_{i,g} G_i.
// k_hx_commit_partial: one thread per (row j, slice of kHxSlice columns, chunk g): windowed Straus over the 8
// 4-bit windows of c_g (MSB window first) -> partial[j][s][g].  Short dependent chains, D / 2 threads.
__global__ void __launch_bounds__(kHxThreads)
k_hx_commit_partial(const uint32_t* __restrict__ Sc, uint64_t D, uint64_t cols, const g1a* __restrict__ tab0,
                    uint64_t nslices, g1j* partial) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t rows = D / cols;
    if (t >= rows * nslices * kHxGroups) return;
    const int g = (int)(t % kHxGroups);
    const g1a* __restrict__ tab = tab0 + (uint64_t)g * (cols + 1) * kHxTab;   // d 2^{32 g} G_i
    const uint64_t js = t / kHxGroups;
    const uint64_t j = js / nslices, s = js % nslices;
    const uint64_t i0 = s * kHxSlice;
    const int len = (int)min((uint64_t)kHxSlice, cols - i0);
    const uint32_t* plane = Sc + (uint64_t)g * D + j * cols + i0;
    const uint32_t* top = Sc + (uint64_t)7 * D + j * cols + i0;   // limb 7: bit 31 is the sign (k_hx_canon)
    uint32_t c[kHxSlice], neg = 0;
#pragma unroll
    for (int k = 0; k < kHxSlice; ++k) {
        c[k] = k < len ? __ldg(plane + k) : 0u;
        const uint32_t t7 = k < len ? __ldg(top + k) : 0u;
        neg |= (t7 >> 31) << k;
        if (g == 7) c[k] &= 0x7fffffffu;
    }
    g1j acc = g1_infinity();
#pragma unroll 1
    for (int w = 7; w >= 0; --w) {
        if (!g1_is_inf(acc)) {
            acc = g1_dbl(acc);
            acc = g1_dbl(acc);
            acc = g1_dbl(acc);
            acc = g1_dbl(acc);
        }
#pragma unroll 1
        for (int k = 0; k < len; ++k) {
            const uint32_t d = (c[k] >> (4 * w)) & 15u;
            if (d) {
                g1a P = tab[(i0 + k) * kHxTab + d];
                if ((neg >> k) & 1u) P.y = fq_neg(P.y);
                acc = g1_add_affine(acc, P);
            }
        }
    }
    partial[t] = acc;
}

// Q[j][g] = sum_s partial[j][s][g]: one CTA per (row, chunk), a strided sum per thread then a tree in shared memory
constexpr int kHxRedThreads = 64;
__global__ void __launch_bounds__(kHxRedThreads)
k_hx_reduce_slices(const g1j* __restrict__ partial, uint64_t nslices, g1j* Qout) {
    __shared__ g1j sm[kHxRedThreads];
    const uint64_t jg = blockIdx.x;   // j * kHxGroups + g
    const uint64_t j = jg / kHxGroups;
    const int g = (int)(jg % kHxGroups);
    g1j acc = g1_infinity();
    for (uint64_t s = threadIdx.x; s < nslices; s += blockDim.x)
        acc = g1_add(acc, partial[(j * nslices + s) * kHxGroups + g]);
    sm[threadIdx.x] = acc;
    __syncthreads();
    for (int off = kHxRedThreads / 2; off > 0; off >>= 1) {
        if ((int)threadIdx.x < off) sm[threadIdx.x] = g1_add(sm[threadIdx.x], sm[threadIdx.x + off]);
        __syncthreads();
    }
    if (threadIdx.x == 0) Qout[jg] = sm[0];
}

// C_j = sum_g 2^{32 g} Q[j][g] (Horner, 32 doublings per chunk) + rho_j H, affine, canonical coordinates
__global__ void k_hx_commit_rows(const g1j* __restrict__ Q, uint64_t rows, const uint32_t* __restrict__ rho_canon,
                                 const g1a* __restrict__ htab, zkl_g1* out) {
    const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j >= rows) return;
    g1j acc = Q[j * kHxGroups + kHxGroups - 1];
    for (int g = kHxGroups - 2; g >= 0; --g) acc = g1_add(acc, Q[j * kHxGroups + g]);   // already 2^{32 g}-scaled
    if (rho_canon) {   // rho H = sum_w hw[w][digit_w] (htab: the 64 x 16 window table of H)
        for (int w = 0; w < 64; ++w) {
            const uint32_t d = (rho_canon[j * 8 + (w >> 3)] >> ((w & 7) * 4)) & 15u;
            if (d) acc = g1_add_affine(acc, htab[w * kHxTab + d]);
        }
    }
    const g1a a = g1_to_affine(acc);
    zkl_g1 o;
    const fq xc = fq_from_mont(a.x), yc = fq_from_mont(a.y);
    for (int k = 0; k < 12; ++k) {
        o.x[k] = a.inf ? 0u : xc.v[k];
        o.y[k] = a.inf ? 0u : yc.v[k];
    }
    o.infinity = a.inf;
    out[j] = o;
}

// affine generators -> canonical coordinates (export)
__global__ void k_hx_export(const g1a* __restrict__ g, uint64_t count, zkl_g1* out) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= count) return;
    const fq xc = fq_from_mont(g[i].x), yc = fq_from_mont(g[i].y);
    zkl_g1 o;
    for (int k = 0; k < 12; ++k) {
        o.x[k] = g[i].inf ? 0u : xc.v[k];
        o.y[k] = g[i].inf ? 0u : yc.v[k];
    }
    o.infinity = g[i].inf;
    out[i] = o;
}

// ProveEval (row-restriction form): w_i = sum_j e~(v_rows, j) S[j cols + i]; one thread per column
__global__ void k_hx_eval_w(const uint32_t* __restrict__ S, uint64_t D, uint64_t cols, const fr* __restrict__ Er,
                            uint32_t* w) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= cols) return;
    const uint64_t rows = D / cols;
    fr acc = fr_zero();
    for (uint64_t j = 0; j < rows; ++j) acc = fr_add(acc, fr_mul(ld_fr_256(Er + j), ld_fr(S, D, j * cols + i)));
    st_fr(w, cols, i, acc);
}

// y = sum_i w_i e~(v_cols, i): block partials, then one block sums them (canonical output)
__global__ void k_hx_eval_y(const uint32_t* __restrict__ w, uint64_t cols, const fr* __restrict__ Ec, fr* part) {
    fr v[1] = {fr_zero()};
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cols; i += (uint64_t)gridDim.x * blockDim.x)
        v[0] = fr_add(v[0], fr_mul(ld_fr(w, cols, i), Ec[i]));
    __shared__ fr scratch[8];
    block_sum_fr<1>(v, scratch);
    if (threadIdx.x == 0) part[blockIdx.x] = v[0];
}

__global__ void k_hx_eval_y_final(const fr* __restrict__ part, int nparts, zkl_fr* y) {
    fr v[1] = {fr_zero()};
    for (int b = threadIdx.x; b < nparts; b += blockDim.x) v[0] = fr_add(v[0], part[b]);
    __shared__ fr scratch[8];
    block_sum_fr<1>(v, scratch);
    if (threadIdx.x == 0) *y = to_canon(v[0]);
}

// Montgomery eq table e~(pt, bits(x)), coordinate 0 = MSB
__global__ void k_hx_eq(const fr* __restrict__ pt, int bits, uint64_t count, fr* out) {
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < count; x += (uint64_t)gridDim.x * blockDim.x) {
        fr e = fr_one();
        for (int j = 0; j < bits; ++j) e = fr_mul(e, ((x >> (bits - 1 - j)) & 1) ? pt[j] : fr_sub(fr_one(), pt[j]));
        out[x] = e;
    }
}

}  // namespace zkl

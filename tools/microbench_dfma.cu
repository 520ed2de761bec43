// Microbenchmark: the eq-weighted wide accumulation of k_round on the FP64 pipe ("what comes next").
// Per iteration a k_round-like mix: 4 fold multiplications and 2 Montgomery products (IMAD pipe), then two
// accumulations W += e * P, either (a) fr_wide_mac (64 IMAD.WIDE each) or (b) 52-bit limb products on the DFMA pipe:
//   a_i b_j = hi 2^52 + lo:  h = fma_rz(a, b, 2^104) = 2^104 + hi 2^52,  l = fma(a, b, (2^104 + 2^52) - h) = 2^52 + lo
// (both exact), the bit patterns minus the exponent bias summed in 64-bit integer columns (10 columns, each < 2^62
// after 64 terms), converted to the 17-word sum once and reduced by the same fr_wide_redc.  Checks (a) == (b) per
// thread, then reports each variant's time.  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_dfma tools/microbench_dfma.cu && ./mb_dfma
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2404_16109_b200/csrc/fr.cuh"

using namespace zkl;

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__);                       \
            return 1;                                                                          \
        }                                                                                      \
    } while (0)

struct fd5 {
    double l[5];
};
struct wide64 {
    unsigned long long c[10];
};

// 256-bit value (8 words) -> 5 limbs of 52 bits as exact doubles
__device__ __forceinline__ fd5 to_fd5(const fr& x) {
    fd5 o;
    const double two52 = 4503599627370496.0;
    const uint32_t w0 = x.v[0], w1 = x.v[1], w2 = x.v[2], w3 = x.v[3], w4 = x.v[4], w5 = x.v[5], w6 = x.v[6],
                   w7 = x.v[7];
    uint32_t lo, hi;
    lo = w0; hi = w1 & 0xfffffu;
    o.l[0] = __hiloint2double(0x43300000 | hi, lo) - two52;
    lo = __funnelshift_r(w1, w2, 20); hi = __funnelshift_r(w2, w3, 20) & 0xfffffu;
    o.l[1] = __hiloint2double(0x43300000 | hi, lo) - two52;
    lo = __funnelshift_r(w3, w4, 8); hi = __funnelshift_r(w4, w5, 8) & 0xfffffu;
    o.l[2] = __hiloint2double(0x43300000 | hi, lo) - two52;
    lo = __funnelshift_r(w4, w5, 28); hi = __funnelshift_r(w5, w6, 28) & 0xfffffu;
    o.l[3] = __hiloint2double(0x43300000 | hi, lo) - two52;
    lo = __funnelshift_r(w6, w7, 16); hi = w7 >> 16;
    o.l[4] = __hiloint2double(0x43300000 | hi, lo) - two52;
    return o;
}

__device__ __forceinline__ void col_add(unsigned long long& c, double v, uint32_t bias_hi) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    uint32_t lo = (uint32_t)c, hi = (uint32_t)(c >> 32);
    asm("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %3;" : "+r"(lo), "+r"(hi) : "r"((uint32_t)b), "r"((uint32_t)(b >> 32) - bias_hi));
    c = ((unsigned long long)hi << 32) | lo;
}

__device__ __forceinline__ void dmac(wide64& W, const fd5& a, const fd5& b) {
    const double c104 = 20282409603651670423947251286016.0;           // 2^104
    const double c104p52 = 20282409603651674927546878656512.0;        // 2^104 + 2^52
#pragma unroll
    for (int i = 0; i < 5; ++i)
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const double h = __fma_rz(a.l[i], b.l[j], c104);
            const double l = __fma_rn(a.l[i], b.l[j], c104p52 - h);
            col_add(W.c[i + j], l, 0x43300000u);
            col_add(W.c[i + j + 1 < 10 ? i + j + 1 : 9], h, 0x46700000u);
        }
}

// sum_c col_c 2^{52 c} -> 17 words
__device__ __forceinline__ fr_wide to_wide(const wide64& W) {
    fr_wide o = fr_wide_zero();
#pragma unroll
    for (int c = 0; c < 10; ++c) {
        const int s = 52 * c, wi = s >> 5, sh = s & 31;
        const unsigned long long v = W.c[c];
        uint32_t p0 = (uint32_t)(v << sh), p1 = (uint32_t)(v >> (32 - sh)), p2 = sh ? (uint32_t)(v >> (64 - sh)) : 0u;
        if (sh == 0) { p0 = (uint32_t)v; p1 = (uint32_t)(v >> 32); }
        unsigned long long cy = 0;
        const uint32_t add[3] = {p0, p1, p2};
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            if (wi + k < 17) {
                cy += (unsigned long long)o.v[wi + k] + add[k];
                o.v[wi + k] = (uint32_t)cy;
                cy >>= 32;
            }
        }
        for (int k = wi + 3; k < 17 && cy; ++k) {
            cy += o.v[k];
            o.v[k] = (uint32_t)cy;
            cy >>= 32;
        }
    }
    return o;
}

__device__ __forceinline__ fr gen(uint32_t seed, uint32_t y) {
    fr x = fr_r2();
    x.v[0] ^= seed * 2654435761u + y * 40503u;
    x.v[3] ^= seed + 7 * y;
    x.v[5] += y;
    return fr_mul(x, fr_one());
}

template <bool DF>
__global__ void __launch_bounds__(256, 2) k_mix(fr* out, int terms, int reps) {
    const uint32_t seed = blockIdx.x * blockDim.x + threadIdx.x;
    __shared__ fr e_s[64];
    if (threadIdx.x < 64) e_s[threadIdx.x] = gen(blockIdx.x, threadIdx.x);
    __syncthreads();
    fr a0 = gen(seed, 1), a1 = gen(seed, 2), s0 = gen(seed, 3), s1 = gen(seed, 4);
    const fr rk = gen(7, 9), beta = gen(8, 10);
    fr total = fr_zero();
    for (int rep = 0; rep < reps; ++rep) {
        fr_wide W0 = fr_wide_zero(), W1 = fr_wide_zero();
        wide64 D0, D1;
#pragma unroll
        for (int c = 0; c < 10; ++c) D0.c[c] = D1.c[c] = 0;
        for (int y = 0; y < terms; ++y) {
            // the fold of k_round (4 products) and its two evaluation products
            const fr A0 = fr_add(a0, fr_mul(rk, fr_sub_lazy(a1, a0)));
            const fr A1 = fr_add(a1, fr_mul(rk, fr_sub_lazy(a0, a1)));
            const fr S0 = fr_add(s0, fr_mul(rk, fr_sub_lazy(s1, s0)));
            const fr S1 = fr_add(s1, fr_mul(rk, fr_sub_lazy(s0, s1)));
            const fr P0 = fr_mul(A0, fr_add_lazy(S0, beta));
            const fr P1 = fr_mul(fr_sub(A1, A0), fr_sub_lazy(S1, S0));
            const fr e = e_s[y & 63];
            if (DF) {
                const fd5 ed = to_fd5(e);
                dmac(D0, ed, to_fd5(P0));
                dmac(D1, ed, to_fd5(P1));
            } else {
                fr_wide_mac(W0, e, P0);
                fr_wide_mac(W1, e, P1);
            }
            a0 = A1; a1 = A0; s0 = S1; s1 = S0;
        }
        if (DF) {
            W0 = to_wide(D0);
            W1 = to_wide(D1);
        }
        total = fr_add(total, fr_add(fr_wide_redc(W0), fr_wide_redc(W1)));
    }
    out[seed] = total;
}

int main() {
    const int blocks = 148 * 2 * 4, threads = 256, terms = 64, reps = 4;
    fr *o1, *o2;
    CK(cudaMalloc(&o1, sizeof(fr) * blocks * threads));
    CK(cudaMalloc(&o2, sizeof(fr) * blocks * threads));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best[2] = {1e9f, 1e9f};
    for (int t = 0; t < 3; ++t) {
        for (int v = 0; v < 2; ++v) {
            cudaEventRecord(e0);
            if (v == 0) k_mix<false><<<blocks, threads>>>(o1, terms, reps);
            else k_mix<true><<<blocks, threads>>>(o2, terms, reps);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best[v]) best[v] = ms;
        }
    }
    const size_t n = (size_t)blocks * threads;
    fr* h1 = new fr[n];
    fr* h2 = new fr[n];
    CK(cudaMemcpy(h1, o1, sizeof(fr) * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h2, o2, sizeof(fr) * n, cudaMemcpyDeviceToHost));
    size_t bad = 0;
    for (size_t i = 0; i < n; ++i)
        for (int l = 0; l < 8; ++l) bad += h1[i].v[l] != h2[i].v[l];
    const double pairs = (double)n * terms * reps;
    printf("{\"bench\": \"k_round mix, 64 terms\", \"imad_wide_ms\": %.3f, \"dfma_ms\": %.3f, \"speedup\": %.3f, "
           "\"imad_pairs_per_s\": %.3e, \"dfma_pairs_per_s\": %.3e, \"mismatched_words\": %zu}\n",
           best[0], best[1], best[0] / best[1], pairs / (best[0] * 1e-3), pairs / (best[1] * 1e-3), bad);
    return bad ? 2 : 0;
}

// Microbenchmark for the wide accumulation of k_round's eq-weighted sums: a sum of 16 terms,
// c = sum_y e_y X_y R^-1 (mod r), computed two ways on the same inputs:
//   (a) as in k_round today: 16 Montgomery multiplications fr_mul(e_y, X_y) and 16 modular additions;
//   (b) 16 schoolbook 256x256 products summed as one 544-bit value W, then the high half brought below r
//       (W < 16 r^2 < 7.3 r 2^256: conditional subtractions of 4r, 2r, r) and one Montgomery reduction.
// Checks (a) == (b) for every thread, then reports each variant's time.  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_wide tools/microbench_wideacc.cu && ./mb_wide
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2404_16109_b200/csrc/fr.cuh"

using namespace zkl;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int kTerms = 16;
__constant__ uint32_t c_r[8] = {ZKL_R0, ZKL_R1, ZKL_R2, ZKL_R3, ZKL_R4, ZKL_R5, ZKL_R6, ZKL_R7};

// W (17 limbs) += a * b
__device__ __forceinline__ void wide_mac(uint32_t* W, const fr& a, const fr& b) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        uint64_t carry = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint64_t t = (uint64_t)a.v[j] * b.v[i] + W[i + j] + carry;
            W[i + j] = (uint32_t)t;
            carry = t >> 32;
        }
#pragma unroll
        for (int k = i + 8; k < 17; ++k) {
            const uint64_t t = (uint64_t)W[k] + carry;
            W[k] = (uint32_t)t;
            carry = t >> 32;
        }
    }
}

// H (9 limbs, the high half W[8..16]) -= m r if H >= m r
__device__ __forceinline__ void hi_sub_if(uint32_t* H, int shift) {
    uint32_t mr[9];
    uint32_t prev = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        mr[k] = (c_r[k] << shift) | (shift ? prev >> (32 - shift) : 0u);
        prev = c_r[k];
    }
    mr[8] = shift ? prev >> (32 - shift) : 0u;
    uint32_t d[9];
    int64_t borrow = 0;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        const int64_t t = (int64_t)H[k] - mr[k] + borrow;
        d[k] = (uint32_t)t;
        borrow = t >> 32;
    }
    if (borrow == 0) {
#pragma unroll
        for (int k = 0; k < 9; ++k) H[k] = d[k];
    }
}

// W < r 2^256 -> W R^-1 mod r (R = 2^256); r' = -r^-1 = -1 mod 2^32 since r0 = 1
__device__ __forceinline__ fr wide_redc(uint32_t* W) {
    hi_sub_if(W + 8, 2);
    hi_sub_if(W + 8, 1);
    hi_sub_if(W + 8, 0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t q = 0u - W[i];
        uint64_t carry = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint64_t t = (uint64_t)q * c_r[j] + W[i + j] + carry;
            W[i + j] = (uint32_t)t;
            carry = t >> 32;
        }
#pragma unroll
        for (int k = i + 8; k < 17; ++k) {
            const uint64_t t = (uint64_t)W[k] + carry;
            W[k] = (uint32_t)t;
            carry = t >> 32;
        }
    }
    fr o;
#pragma unroll
    for (int k = 0; k < 8; ++k) o.v[k] = W[8 + k];
    fr_reduce_once(o);
    return o;
}

__device__ __forceinline__ fr term(int seed, int y) {
    fr x = fr_r2();
    x.v[0] ^= seed * 2654435761u + y * 40503u;
    x.v[3] ^= seed + 7 * y;
    return fr_mul(x, fr_one());   // canonical (< r) pseudo-random element
}

template <bool WIDE>
__global__ void k_sum(fr* out, int iters) {
    const int seed = blockIdx.x * blockDim.x + threadIdx.x;
    __shared__ fr e[kTerms];   // the eq weights, shared by the block (as E_lo in k_round)
    if (threadIdx.x < kTerms) e[threadIdx.x] = term(blockIdx.x, threadIdx.x);
    __syncthreads();
    fr x0 = term(seed + 1, 100);
    const fr step = term(seed + 2, 200);
    fr total = fr_zero();
    for (int it = 0; it < iters; ++it) {
        fr c, x = x0;
        if (WIDE) {
            uint32_t W[17] = {0};
#pragma unroll
            for (int y = 0; y < kTerms; ++y) { wide_mac(W, e[y], x); x = fr_add(x, step); }
            c = wide_redc(W);
        } else {
            c = fr_zero();
#pragma unroll
            for (int y = 0; y < kTerms; ++y) { c = fr_add(c, fr_mul(e[y], x)); x = fr_add(x, step); }
        }
        total = fr_add(total, c);
        x0.v[0] ^= c.v[0] & 1u;   // keep iterations dependent on the data
    }
    out[seed] = total;
}

int main() {
    const int blocks = 148 * 4, threads = 256, iters = 64, n = blocks * threads;
    fr *a, *b;
    CK(cudaMalloc(&a, n * sizeof(fr)));
    CK(cudaMalloc(&b, n * sizeof(fr)));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms[2];
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k_sum<false><<<blocks, threads>>>(a, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms[0], e0, e1);
        cudaEventRecord(e0);
        k_sum<true><<<blocks, threads>>>(b, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms[1], e0, e1);
    }
    CK(cudaGetLastError());
    fr* ha = new fr[n];
    fr* hb = new fr[n];
    CK(cudaMemcpy(ha, a, n * sizeof(fr), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hb, b, n * sizeof(fr), cudaMemcpyDeviceToHost));
    long bad = 0;
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < 8; ++k) bad += ha[i].v[k] != hb[i].v[k];
    const double terms = (double)n * iters * kTerms;
    printf("{\"terms_per_sum\": %d, \"mismatched_limbs\": %ld, \"fused_ms\": %.3f, \"wide_ms\": %.3f, "
           "\"fused_Gterm_s\": %.2f, \"wide_Gterm_s\": %.2f}\n",
           kTerms, bad, ms[0], ms[1], terms / ms[0] / 1e6, terms / ms[1] / 1e6);
    return bad != 0;
}

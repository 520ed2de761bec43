// Microbenchmark for the wide accumulation of the eq-weighted sums (csrc/fr.cuh fr_wide_*): 16 terms,
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
            fr_wide W = fr_wide_zero();
#pragma unroll
            for (int y = 0; y < kTerms; ++y) { fr_wide_mac(W, e[y], x); x = fr_add(x, step); }
            c = fr_wide_redc(W);
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

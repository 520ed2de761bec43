// Step-0 microbenchmark: integer-pipe throughput and Fr-mul throughput
// on the B200, plus device properties.  Standalone: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o microbench_fr tools/microbench_fr.cu && ./microbench_fr
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2404_16109_b200/csrc/fr.cuh"

using namespace zkl;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint64_t gtimer() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

// clock sampling: thread 0 of block 0 records (clock64, globaltimer) at start/end
__device__ unsigned long long g_clk[4];

template <int ILP>
__global__ void k_frmul(fr* out, int iters) {
    fr x[ILP];
    fr y = fr_one();
    y.v[0] ^= threadIdx.x;   // data-dependent operand
#pragma unroll
    for (int k = 0; k < ILP; ++k) { x[k] = fr_r2(); x[k].v[1] ^= blockIdx.x * 977 + k; }
    unsigned long long c0 = clock64(), t0 = gtimer();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < ILP; ++k) x[k] = fr_mul(x[k], y);
    }
    unsigned long long c1 = clock64(), t1 = gtimer();
    if (blockIdx.x == 0 && threadIdx.x == 0) { g_clk[0] = c0; g_clk[1] = c1; g_clk[2] = t0; g_clk[3] = t1; }
    fr acc = x[0];
#pragma unroll
    for (int k = 1; k < ILP; ++k) acc = fr_add(acc, x[k]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// raw IMAD (32-bit lo) throughput: 8 independent chains
__global__ void k_imad(uint32_t* out, int iters) {
    uint32_t a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x + k;
    uint32_t b = blockIdx.x | 1, c = 12345;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
    }
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// IMAD.WIDE.U32 throughput: 8 independent 64-bit accumulators acc = a*b + acc
__global__ void k_imadwide(unsigned long long* out, int iters) {
    unsigned long long acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = threadIdx.x + k;
    uint32_t b = blockIdx.x | 1;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            uint32_t lo = (uint32_t)acc[k];
            asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[k]) : "r"(lo), "r"(b));
        }
    }
    unsigned long long s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += acc[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// IADD3 throughput
__global__ void k_iadd(uint32_t* out, int iters) {
    uint32_t a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x + k;
    uint32_t b = blockIdx.x | 1, c = 7;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
    }
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s ^= a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// single-thread latency of a dependent chain of fr_mul, and of fr_inv
__global__ void k_lat(fr* out, int iters, unsigned long long* cyc) {
    fr x = fr_r2(), y = fr_one();
    y.v[0] ^= threadIdx.x;
    unsigned long long c0 = clock64();
    for (int i = 0; i < iters; ++i) x = fr_mul(x, y);
    unsigned long long c1 = clock64();
    fr z = fr_inv(x);
    unsigned long long c2 = clock64();
    fr w = fr_inv_fermat(x);
    unsigned long long c3 = clock64();
    out[0] = fr_add(x, z);
    cyc[0] = c1 - c0;
    cyc[1] = c2 - c1;
    cyc[2] = c3 - c2;
    cyc[3] = fr_eq(z, w) && fr_eq(fr_mul(x, z), fr_one());   // binary Euclid == Fermat, and x z = 1
}

static double mhz_from_clk() {
    unsigned long long h[4];
    cudaMemcpyFromSymbol(h, g_clk, sizeof(h));
    return double(h[1] - h[0]) / double(h[3] - h[2]) * 1e3;
}

template <typename K, typename T>
static int timeit(const char* name, K kern, T* buf, int blocks, int threads, int iters, double ops_per_iter_thread,
                  bool clk) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    kern<<<blocks, threads>>>(buf, iters / 10 + 1);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    kern<<<blocks, threads>>>(buf, iters);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double ops = ops_per_iter_thread * iters * (double)blocks * threads;
    double mhz = clk ? mhz_from_clk() : 0;
    printf("{\"bench\": \"%s\", \"blocks\": %d, \"threads\": %d, \"ms\": %.3f, \"Gops\": %.2f, \"sm_mhz_in_kernel\": %.0f}\n",
           name, blocks, threads, ms, ops / (ms * 1e6), mhz);
    return 0;
}

int main() {
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, 0));
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    printf("{\"device\": \"%s\", \"sm\": %d, \"cc\": \"%d.%d\", \"smem_per_block_optin\": %zu, \"l2\": %d, \"regs_per_sm\": %d, \"clock_khz\": %d}\n",
           p.name, p.multiProcessorCount, p.major, p.minor, p.sharedMemPerBlockOptin, p.l2CacheSize,
           p.regsPerMultiprocessor, clk_khz);
    int sms = p.multiProcessorCount;
    void* buf;
    CK(cudaMalloc(&buf, 64 << 20));
    timeit("imad_lo", k_imad, (uint32_t*)buf, sms * 8, 256, 20000, 8, false);
    timeit("imad_wide", k_imadwide, (unsigned long long*)buf, sms * 8, 256, 20000, 8, false);
    timeit("iadd", k_iadd, (uint32_t*)buf, sms * 8, 256, 20000, 16, false);
    {
        unsigned long long* cyc;
        CK(cudaMalloc(&cyc, 32));
        k_lat<<<1, 1>>>((fr*)buf, 1000, cyc);
        CK(cudaDeviceSynchronize());
        k_lat<<<1, 1>>>((fr*)buf, 1000, cyc);
        CK(cudaDeviceSynchronize());
        unsigned long long h[4];
        CK(cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost));
        printf("{\"bench\": \"latency\", \"frmul_cycles\": %.1f, \"frinv_cycles\": %llu, \"frinv_fermat_cycles\": %llu, "
               "\"inverses_agree\": %llu}\n", h[0] / 1000.0, h[1], h[2], h[3]);
    }
    for (int occ : {2, 4, 8}) {
        timeit("frmul_ilp1", k_frmul<1>, (fr*)buf, sms * occ, 256, 2000, 1, true);
        timeit("frmul_ilp2", k_frmul<2>, (fr*)buf, sms * occ, 256, 1000, 2, true);
        timeit("frmul_ilp4", k_frmul<4>, (fr*)buf, sms * occ, 128, 500, 4, true);
    }
    return 0;
}

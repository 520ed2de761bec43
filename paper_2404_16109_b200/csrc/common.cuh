// Shared device/host helpers of the zkl library (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/zkl.h"
#include "fr.cuh"

namespace zkl {

constexpr int kMaxRounds = 40;          // log2 D <= 40
constexpr int kSlots = 5;               // per-round D-side partial sums: H0, H1, Hinf, a0, a1
enum { SLOT_H0 = 0, SLOT_H1 = 1, SLOT_HINF = 2, SLOT_A0 = 3, SLOT_A1 = 4 };
constexpr int kMaxBlocks = 1184;        // partial-sum rows per round (148 SMs x 8)
constexpr int kTailMax = 2048;          // the single-CTA tail holds <= 2048 elements of A and S

// Debug builds (-DZKL_CHECK; tools/sanitize_cases.py --check): every SoA access and table gather is bounds-checked
// with a device assert (compute-sanitizer is not available on this GPU pool).
#ifdef ZKL_CHECK
#include <assert.h>
#define ZKL_ASSERT(c) assert(c)
#else
#define ZKL_ASSERT(c) ((void)0)
#endif

// ------------------------------------------------------------------ SoA access
__device__ __forceinline__ fr ld_fr(const uint32_t* __restrict__ base, uint64_t n, uint64_t i) {
    ZKL_ASSERT(i < n);
    fr x;
#pragma unroll
    for (int l = 0; l < 8; ++l) x.v[l] = base[(uint64_t)l * n + i];
    return x;
}

__device__ __forceinline__ void st_fr(uint32_t* __restrict__ base, uint64_t n, uint64_t i, const fr& x) {
    ZKL_ASSERT(i < n);
#pragma unroll
    for (int l = 0; l < 8; ++l) base[(uint64_t)l * n + i] = x.v[l];
}

// 4 consecutive elements i..i+3 (i % 4 == 0, n % 4 == 0): one 128-bit load per limb plane
__device__ __forceinline__ void ld_fr4(const uint32_t* __restrict__ base, uint64_t n, uint64_t i, fr (&x)[4]) {
    ZKL_ASSERT(i + 4 <= n && (i & 3) == 0);
#pragma unroll
    for (int l = 0; l < 8; ++l) {
        uint4 q = __ldg(reinterpret_cast<const uint4*>(base + (uint64_t)l * n + i));
        x[0].v[l] = q.x; x[1].v[l] = q.y; x[2].v[l] = q.z; x[3].v[l] = q.w;
    }
}

__device__ __forceinline__ void st_fr4(uint32_t* __restrict__ base, uint64_t n, uint64_t i, const fr (&x)[4]) {
    ZKL_ASSERT(i + 4 <= n && (i & 3) == 0);
#pragma unroll
    for (int l = 0; l < 8; ++l) {
        uint4 q = make_uint4(x[0].v[l], x[1].v[l], x[2].v[l], x[3].v[l]);
        *reinterpret_cast<uint4*>(base + (uint64_t)l * n + i) = q;
    }
}

// 2 consecutive elements (i even, n even): one 64-bit access per plane
__device__ __forceinline__ void ld_fr2(const uint32_t* __restrict__ base, uint64_t n, uint64_t i, fr (&x)[2]) {
    ZKL_ASSERT(i + 2 <= n && (i & 1) == 0);
#pragma unroll
    for (int l = 0; l < 8; ++l) {
        uint2 q = __ldg(reinterpret_cast<const uint2*>(base + (uint64_t)l * n + i));
        x[0].v[l] = q.x; x[1].v[l] = q.y;
    }
}

__device__ __forceinline__ void st_fr2(uint32_t* __restrict__ base, uint64_t n, uint64_t i, const fr& a,
                                       const fr& b) {
    ZKL_ASSERT(i + 2 <= n && (i & 1) == 0);
#pragma unroll
    for (int l = 0; l < 8; ++l)
        *reinterpret_cast<uint2*>(base + (uint64_t)l * n + i) = make_uint2(a.v[l], b.v[l]);
}

// AoS Fr in global/shared memory
__device__ __forceinline__ fr ld_aos(const fr* p) { return *p; }

// ------------------------------------------------------------------ reductions
__device__ __forceinline__ fr shfl_down_fr(const fr& x, int off) {
    fr y;
#pragma unroll
    for (int l = 0; l < 8; ++l) y.v[l] = __shfl_down_sync(0xffffffffu, x.v[l], off);
    return y;
}

// One 256-bit read-only global load (sm_100: LDG.E.ENL2.256): a whole Fr element at a 32-byte aligned
// address in one instruction -- half the L1 wavefronts of two 128-bit loads for scattered (gather) accesses.
__device__ __forceinline__ fr ld_fr_256(const void* p) {
    fr x;
    asm("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(x.v[0]), "=r"(x.v[1]), "=r"(x.v[2]), "=r"(x.v[3]), "=r"(x.v[4]), "=r"(x.v[5]), "=r"(x.v[6]),
          "=r"(x.v[7])
        : "l"(p));
    return x;
}

// Sum of NV Fr values over the block; result valid in thread 0.  `scratch` holds
// NV * (blockDim/32) fr.  Contains __syncthreads (all threads must call).
template <int NV>
__device__ __forceinline__ void block_sum_fr(fr (&v)[NV], fr* scratch) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
        for (int k = 0; k < NV; ++k) v[k] = fr_add(v[k], shfl_down_fr(v[k], off));
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) scratch[k * nw + warp] = v[k];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) v[k] = lane < nw ? scratch[k * nw + lane] : fr_zero();
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
            for (int k = 0; k < NV; ++k) v[k] = fr_add(v[k], shfl_down_fr(v[k], off));
        }
    }
    __syncthreads();
}

__device__ __forceinline__ void atomic_min_i64(unsigned long long* p, uint64_t v) {
    atomicMin(p, (unsigned long long)v);
}

__device__ __forceinline__ fr fr_small(uint32_t v) {
    fr x = fr_zero();
    x.v[0] = v;
    return fr_to_mont(x);
}

__device__ __forceinline__ zkl_fr to_canon(const fr& m) {
    fr c = fr_from_mont(m);
    zkl_fr z;
    for (int l = 0; l < 8; ++l) z.w[l] = c.v[l];
    return z;
}

// Sense-counting grid barrier for a cooperative launch (all CTAs co-resident, guaranteed by
// cudaLaunchCooperativeKernel).  count returns to 0 after each barrier; gen only increases.
struct GridBar {
    unsigned int count;
    unsigned int gen;
};

__device__ __forceinline__ void grid_sync(GridBar* b) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned int* vgen = &b->gen;
        const unsigned int g = *vgen;
        __threadfence();
        if (atomicAdd(&b->count, 1u) == gridDim.x - 1) {
            b->count = 0;
            __threadfence();
            atomicAdd(&b->gen, 1u);
        } else {
            while (*vgen == g) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

// ------------------------------------------------------------------ device-side proof state
// Scalars of one proof, Montgomery form, in the workspace.
struct RoundDesc {
    uint64_t elo_off, ehi_off;   // offsets (in fr) of E_lo / E_hi in the eq arena
    uint64_t part_base;          // offset (in fr) of this round's partial rows: [slot][row], row stride nblocks
    uint32_t gbits;              // log2 of the group size G (pairs sharing one E_hi entry)
    uint32_t nblocks;            // partial rows (blocks / tiles) written for this round
    uint32_t direct_h1;          // 1: H(1) summed directly (round 1 of sumcheck_prove, u_c = 0)
    uint32_t a1_derived;         // 1: the round's kernel (k_round<FOLD>) does not sum a(1) = sum_y A(y,1); folding
                                 // is linear, so a0_k + a1_k = a0_{k-1} + r_{k-1} (a1_{k-1} - a0_{k-1}) gives it
};

struct ProofScalars {
    fr beta, alpha1, alpha2;
    fr u[kMaxRounds];
    fr r[kMaxRounds];
    fr rank_eq;            // eq(u[0:log2 P], bits(rank)) — this rank's factor of e~(u, .)
    fr w;                  // N D^{-1}
};

struct ProofOut {
    zkl_fr evals[kMaxRounds][4];
    zkl_fr finals[5];
    unsigned long long err_index[3];   // host copies of the error words: S div0, T div0, gather miss
    int status;
    int pad;
};

}  // namespace zkl

// ------------------------------------------------------------------ opaque ABI objects
#include <condition_variable>
#include <mutex>

// loopback group: P virtual ranks (threads) of one process on one device
struct zkl_group {
    int nranks;
    int device;
    uint8_t* staging;            // device, nranks x max block
    size_t staging_bytes;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    int min_arrived = 0;
    unsigned long long min_acc = ~0ull;
};

struct zkl_ctx {
    int device;
    cudaStream_t stream;
    cudaStream_t side;             // table-side work overlapping the D side (high priority, one block)
    cudaStream_t aux;              // upper inversion levels (high priority, latency hidden behind the D side)
    cudaStream_t low;              // async-mode histogram (lowest priority: fills the gaps of the proof's critical path)
    cudaEvent_t ev_keys, ev_m;     // index keys written (main) / m written (low)
    cudaEvent_t ev_b;              // B = 1/(beta + T) written (main), for a table side moved to the side stream
    cudaEvent_t ev_eq;             // the eq tables written (side stream, beside the B inversion)
    int m_pending;                 // ev_m recorded: the next consumer of m on the ctx stream must wait for it
    int prio_lo, prio_hi;
    cudaEvent_t ev_fork, ev_join;
    cudaEvent_t ev_fwd[2], ev_mid[2];
    int rank, nranks;
    void* nccl_comm;               // ncclComm_t (loaded at run time) when nranks > 1
    zkl_group* group;              // loopback communicator (instead of NCCL), or null
    uint8_t* ws;
    size_t ws_bytes;
    void* host_out;                // pinned host copy of ProofOut + staging
    uint8_t* dscratch;             // 4 KiB device scratch (scalars, error words) owned by the ctx
    int poisoned;
    uint64_t launches;
    // keys of the last successful zkl_tlookup_prepare (in the workspace): valid for this S / table
    int prep_valid;                // the workspace keys belong to (prep_S, prep_n, prep_table)
    const uint32_t* prep_S;        // nullptr: S is virtual (prepare_pair without S_local_out; S_i = T_key)
    uint64_t prep_n;
    const zkl_table* prep_table;
    char last_error[512];
    // async mode (zkl_ctx_set_async): prepare / prove enqueue and return; their host-side completion (error
    // words, outputs, the gather fallback) runs in zkl_ctx_wait, in call order.  One of each kind in flight.
    int async_mode;
    int pend_prepare, pend_prove;
    void* pending;                 // std::vector<std::function<int()>>*
    // zkl_tlookup_prove_pair_host: device copies of the host inputs, the table and m (owned, grown on demand)
    struct HostStep {
        void* buf;           // x | y | tx | ty | T (SoA) | table memory | m
        size_t bytes;
        zkl_table* table;
    } hs;
    // zkl_tlookup_prove_p1: the field vectors, table and m it owns, and a separate workspace for the Hyrax steps
    struct P1Buf {
        void* buf;
        size_t bytes;
        void* hxws;
        size_t hxbytes;
        zkl_table* table;
    } p1;
    // optional per-kernel timing (zkl_ctx_set_profiling): events around every launch
    int profiling;
    int nprof;
    struct ProfRec {
        const char* name;
        cudaEvent_t a, b;
        cudaStream_t stream;
    } prof[256];
};

struct zkl_table {
    uint64_t N;
    uint32_t* T;        // SoA Montgomery copy, N entries
    uint4* Taos;        // AoS copy (32 B per entry) by table index
    uint32_t* slots;
    uint4* Skeys;       // AoS key per slot    // open-addressing hash: slot -> index+1 (0 = empty)
    uint32_t slot_mask;
    uint64_t nslots;
    int device;
    // function-lookup tables T_j = tx_j + alpha ty_j whose tx column is the contiguous range x0, x0+1, ...
    // (zkl_table_attach_pair): the index of a pair (x, y) is x - x0, checked by ty[x - x0] == y
    int has_pair;
    int32_t x0;
    int32_t* ty;        // device copy, N entries (in the table memory)
    zkl_fr alpha;       // canonical alpha_f of the attached pair form
};

// Device kernels of the tlookup hot path.  Included once, by api.cu.
#pragma once
#include <cub/block/block_radix_sort.cuh>

#include "common.cuh"

namespace zkl {

// One out-of-line copy of the Montgomery product for single-pass scalar kernels (k_derive, k_round_consts): inlined
// there dozens of times, their code streams through the instruction cache once per launch.
static __device__ __noinline__ fr fr_mul_s(const fr a, const fr b) { return fr_mul(a, b); }

// ====================================================================== a1: boundary encode
// canonical AoS (8 LE words per element) -> SoA Montgomery.  One Fr mul (x * R^2) per element.
__global__ void k_import_canon(const uint32_t* __restrict__ src, uint64_t n, uint32_t* __restrict__ dst,
                               unsigned long long* err) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4* p = reinterpret_cast<const uint4*>(src + 8 * i);
        uint4 a = p[0], b = p[1];
        fr x;
        x.v[0] = a.x; x.v[1] = a.y; x.v[2] = a.z; x.v[3] = a.w;
        x.v[4] = b.x; x.v[5] = b.y; x.v[6] = b.z; x.v[7] = b.w;
        if (fr_geq_modulus(x)) {
            if (err) atomic_min_i64(err, i);
            x = fr_zero();
        }
        st_fr(dst, n, i, fr_to_mont(x));
    }
}

// signed integer -> canonical Fr (x < 0 -> r - |x|)
__device__ __forceinline__ fr fr_from_i64(int64_t v) {
    fr x = fr_zero();
    uint64_t mag = v < 0 ? (uint64_t)0 - (uint64_t)v : (uint64_t)v;
    x.v[0] = (uint32_t)mag;
    x.v[1] = (uint32_t)(mag >> 32);
    return v < 0 ? fr_sub(fr_zero(), x) : x;
}

__global__ void k_import_i64(const int64_t* __restrict__ src, uint64_t n, uint32_t* __restrict__ dst) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        st_fr(dst, n, i, fr_to_mont(fr_from_i64(src[i])));
}

// 32-bit integers -> Montgomery SoA (is_unsigned: u32 counts such as m; else int32 with x < 0 -> r - |x|)
__global__ void k_import_i32(const int32_t* __restrict__ src, uint64_t n, int is_unsigned, uint32_t* __restrict__ dst) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const int64_t v = is_unsigned ? (int64_t)(uint32_t)src[i] : (int64_t)src[i];
        st_fr(dst, n, i, fr_to_mont(fr_from_i64(v)));
    }
}

// S_i = x_i + alpha_f y_i for 32-bit x, y, straight into Montgomery form without a full
// field multiplication: with Cx = +-2^32 R, Cy = +-alpha_f 2^32 R (mod r, sign of x / y),
//   U = |x| Cx + |y| Cy  (< 2^32 r, 9 words),  V = (U + q r) / 2^32 with q = -U mod 2^32 (r' = -1)
// is congruent to (x + alpha_f y) R and below 2r: one conditional subtraction makes it canonical.
// consts: [Cx+, Cx-, Cy+, Cy-] (Montgomery-domain words, canonical).
__device__ __forceinline__ fr fr_from_small_pair(int32_t x, int32_t y, const fr* __restrict__ c) {
    const uint32_t ax = x < 0 ? 0u - (uint32_t)x : (uint32_t)x;
    const uint32_t ay = y < 0 ? 0u - (uint32_t)y : (uint32_t)y;
    const fr& cx = c[x < 0 ? 1 : 0];
    const fr& cy = c[y < 0 ? 3 : 2];
    uint32_t u[9];
    uint64_t t = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        t = (uint64_t)ax * cx.v[j] + (uint64_t)ay * cy.v[j] + (t >> 32);
        u[j] = (uint32_t)t;
    }
    u[8] = (uint32_t)(t >> 32);
    const uint32_t q = 0u - u[0];
    const uint32_t rl[8] = {ZKL_R0, ZKL_R1, ZKL_R2, ZKL_R3, ZKL_R4, ZKL_R5, ZKL_R6, ZKL_R7};
    uint64_t cy64 = u[0] != 0;   // u0 + q * r0 = u0 + q = 0 (mod 2^32), carry iff u0 != 0
    fr v;
#pragma unroll
    for (int j = 1; j < 8; ++j) {
        const uint64_t w = (uint64_t)q * rl[j] + u[j] + cy64;
        v.v[j - 1] = (uint32_t)w;
        cy64 = w >> 32;
    }
    v.v[7] = (uint32_t)(u[8] + cy64);
    fr_reduce_once(v);
    return v;
}

__global__ void k_pair_consts(const fr* __restrict__ af_m, fr* c) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        c[0] = fr_2p32_m();
        c[1] = fr_2p32_m_neg();
        c[2] = fr_mul(*af_m, fr_2p32_m());
        c[3] = fr_neg(c[2]);
    }
}

__global__ void k_import_pair_dev(const int32_t* __restrict__ x, const int32_t* __restrict__ y, uint64_t n,
                                  const fr* __restrict__ consts, uint32_t* __restrict__ dst) {
    __shared__ fr c[4];
    if (threadIdx.x < 4) c[threadIdx.x] = consts[threadIdx.x];
    __syncthreads();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        st_fr(dst, n, i, fr_from_small_pair(x[i], y[i], c));
}

__global__ void k_export(const uint32_t* __restrict__ src, uint64_t n, uint32_t* __restrict__ dst) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        fr x = fr_from_mont(ld_fr(src, n, i));
        uint4* p = reinterpret_cast<uint4*>(dst + 8 * i);
        p[0] = make_uint4(x.v[0], x.v[1], x.v[2], x.v[3]);
        p[1] = make_uint4(x.v[4], x.v[5], x.v[6], x.v[7]);
    }
}

// ====================================================================== a2: table handle
// Open addressing over the Montgomery representation; slot holds index+1 (0 = empty).
__device__ __forceinline__ uint32_t hash_fr(const fr& x) {
    uint32_t h = x.v[0] * 0x9E3779B1u;
    h ^= x.v[1] + 0x7F4A7C15u + (h << 6) + (h >> 2);
    h ^= x.v[6] * 0x85EBCA6Bu;
    h ^= x.v[7];
    h ^= h >> 16;
    h *= 0x2C1B3C6Du;
    h ^= h >> 13;
    return h;
}

struct TableView {
    const uint32_t* T;       // SoA Montgomery
    const uint4* Taos;       // AoS copy (2 x uint4 per entry), indexed by table index
    const uint32_t* slots;   // index + 1, 0 = empty
    const uint4* Skeys;      // AoS key stored WITH each occupied slot: one probe = two independent loads
    uint64_t N;
    uint32_t mask;
};

__device__ __forceinline__ bool aos_eq(const uint4* p, const fr& x) {
    return fr_eq(ld_fr_256(p), x);
}

// index of x in T, or -1 (linear probing; slot index and slot key are loaded together)
__device__ __forceinline__ int64_t table_find(const TableView& tv, const fr& x) {
    uint32_t h = hash_fr(x) & tv.mask;
    for (;;) {
        const uint32_t s = __ldg(tv.slots + h);
        const bool eq = aos_eq(tv.Skeys + 2 * (uint64_t)h, x);
        if (s == 0) return -1;
        if (eq) return (int64_t)(s - 1);
        h = (h + 1) & tv.mask;
    }
}

// insert-time helper: the (final) key of every occupied slot
__global__ void k_table_fill_keys(const uint32_t* __restrict__ T, uint64_t N, const uint32_t* __restrict__ slots,
                                  uint64_t nslots, uint4* Skeys) {
    for (uint64_t h = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; h < nslots; h += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = slots[h];
        fr x = s ? ld_fr(T, N, s - 1) : fr_zero();
        Skeys[2 * h] = make_uint4(x.v[0], x.v[1], x.v[2], x.v[3]);
        Skeys[2 * h + 1] = make_uint4(x.v[4], x.v[5], x.v[6], x.v[7]);
    }
}

__global__ void k_table_copy(const uint32_t* __restrict__ src, uint64_t n, uint32_t* __restrict__ dst,
                             uint4* __restrict__ aos) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const fr x = ld_fr(src, n, i);
        st_fr(dst, n, i, x);
        aos[2 * i] = make_uint4(x.v[0], x.v[1], x.v[2], x.v[3]);
        aos[2 * i + 1] = make_uint4(x.v[4], x.v[5], x.v[6], x.v[7]);
    }
}

__global__ void k_table_insert(const uint32_t* __restrict__ T, uint64_t N, uint32_t* slots, uint32_t mask) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < N; j += (uint64_t)gridDim.x * blockDim.x) {
        fr x = ld_fr(T, N, j);
        uint32_t h = hash_fr(x) & mask;
        for (;;) {
            uint32_t old = atomicCAS(slots + h, 0u, (uint32_t)(j + 1));
            if (old == 0) break;
            if (fr_eq(ld_fr(T, N, old - 1), x)) {   // equal key: the slot keeps the smallest index
                atomicMin(slots + h, (uint32_t)(j + 1));
                break;
            }
            h = (h + 1) & mask;
        }
    }
}

// j is a duplicate iff its key's slot holds a smaller index; report the smallest such j.
__global__ void k_table_dups(const uint32_t* __restrict__ T, const uint4* __restrict__ aos, uint64_t N,
                             const uint32_t* slots, const uint4* skeys, uint32_t mask, unsigned long long* err) {
    TableView tv{T, aos, slots, skeys, N, mask};
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < N; j += (uint64_t)gridDim.x * blockDim.x) {
        int64_t f = table_find(tv, ld_fr(T, N, j));
        if (f != (int64_t)j) atomic_min_i64(err, j);
    }
}

// ====================================================================== a3: multiplicities
// Two passes, atomic-free:
//  (1) index map: one lookup per thread (high occupancy hides the two dependent L2 round trips of the
//      hash probe): key_i = j such that S_i = T_j (full 256-bit compare against the AoS key copy).  A
//      lookup not in T reports its index (atomicMin on the error word — the error path only) and gets
//      key 0 (m is discarded on error).
//  (2) count: per tile of 4096 keys, block radix sort, then per distinct key one read-modify-write of
//      the CTA-private row: heads subtract their sorted position, tails add theirs + 1 (two barrier-
//      separated phases, each touching one address per distinct key).  Keys beyond n (a partial tile,
//      n < 4096) take the sentinel N, which sorts last and is not counted.  A column sum gives m.
__global__ void __launch_bounds__(256)
k_index_map(const uint32_t* __restrict__ S, uint64_t n, uint64_t global_offset, TableView tv,
            uint32_t* __restrict__ keys, unsigned long long* err) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const fr x = ld_fr(S, n, i);
        const int64_t f = table_find(tv, x);
        uint32_t key = 0;
        if (f < 0) atomic_min_i64(err, global_offset + i);
        else key = (uint32_t)f;
        keys[i] = key;
    }
}

// Range fast path of the fused function-lookup prepare: for a table attached as a pair range (T_j = tx_j +
// alpha ty_j, tx_j = x0 + j), the index of (x, y) is j = x - x0, valid iff 0 <= j < N and ty[j] == y (then
// S = T_j exactly; T is duplicate-free).  No hash probe: a 4-byte gather from the L2-resident ty column.  A pair
// that fails this test may still equal another entry for a special alpha, so a miss only raises `miss`, and the
// caller redoes the prepare with the exact hash index.  dst == nullptr: S stays virtual (keys only; S_i = T_key,
// S is committed homomorphically as [X] + alpha [Y] and never needs to exist in HBM).
__global__ void __launch_bounds__(256, 4)
k_import_pair_range(const int32_t* __restrict__ x, const int32_t* __restrict__ y, uint64_t n,
                    const fr* __restrict__ consts, uint32_t* __restrict__ dst, int32_t x0,
                    const int32_t* __restrict__ ty, uint64_t N, uint32_t* __restrict__ keys,
                    unsigned long long* miss) {
    __shared__ fr c[4];
    if (threadIdx.x < 4) c[threadIdx.x] = consts[threadIdx.x];
    __syncthreads();
    bool missed = false;
    if ((n & 3) == 0) {
        // two groups of 4 lookups per step: both groups' x, y loads and ty gathers are in flight together
        const uint64_t stride = 4 * (uint64_t)gridDim.x * blockDim.x;
        for (uint64_t i = 4 * (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x); i < n; i += 2 * stride) {
            const uint64_t i2 = i + stride;
            const bool two = i2 < n;
            const int4 xv = __ldg(reinterpret_cast<const int4*>(x + i));
            const int4 yv = __ldg(reinterpret_cast<const int4*>(y + i));
            int4 xv2 = make_int4(0, 0, 0, 0), yv2 = make_int4(0, 0, 0, 0);
            if (two) {
                xv2 = __ldg(reinterpret_cast<const int4*>(x + i2));
                yv2 = __ldg(reinterpret_cast<const int4*>(y + i2));
            }
            const int xs[8] = {xv.x, xv.y, xv.z, xv.w, xv2.x, xv2.y, xv2.z, xv2.w};
            const int ys[8] = {yv.x, yv.y, yv.z, yv.w, yv2.x, yv2.y, yv2.z, yv2.w};
            int64_t jj[8];
            int32_t tyv[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                jj[q] = (int64_t)xs[q] - (int64_t)x0;
                const bool inr = jj[q] >= 0 && (uint64_t)jj[q] < N && (q < 4 || two);
                tyv[q] = inr ? __ldg(ty + jj[q]) : ~ys[q];
            }
            uint32_t kk[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const bool ok = tyv[q] == ys[q];
                if (q < 4 || two) missed |= !ok;
                kk[q] = ok ? (uint32_t)jj[q] : 0u;
            }
            if (dst) {
                fr s4[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) s4[q] = fr_from_small_pair(xs[q], ys[q], c);
                st_fr4(dst, n, i, s4);
                if (two) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) s4[q] = fr_from_small_pair(xs[4 + q], ys[4 + q], c);
                    st_fr4(dst, n, i2, s4);
                }
            }
            *reinterpret_cast<uint4*>(keys + i) = make_uint4(kk[0], kk[1], kk[2], kk[3]);
            if (two) *reinterpret_cast<uint4*>(keys + i2) = make_uint4(kk[4], kk[5], kk[6], kk[7]);
        }
    } else {
        for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
            const int64_t j = (int64_t)x[i] - (int64_t)x0;
            const bool ok = j >= 0 && (uint64_t)j < N && __ldg(ty + j) == y[i];
            missed |= !ok;
            keys[i] = ok ? (uint32_t)j : 0u;
            if (dst) st_fr(dst, n, i, fr_from_small_pair(x[i], y[i], c));
        }
    }
    if (__any_sync(0xffffffffu, missed) && (threadIdx.x & 31) == 0) atomicMin(miss, 0ull);
}

// zkl_table_attach_pair: tx is the range x0 + j and T_j = tx_j + alpha ty_j for every j; copy ty
__global__ void k_table_check_pair(const int32_t* __restrict__ tx, const int32_t* __restrict__ ty, uint64_t N,
                                   const fr* __restrict__ consts, const uint32_t* __restrict__ T, int32_t* ty_out,
                                   unsigned long long* bad) {
    __shared__ fr c[4];
    if (threadIdx.x < 4) c[threadIdx.x] = consts[threadIdx.x];
    __syncthreads();
    const int64_t x0 = tx[0];
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < N; j += (uint64_t)gridDim.x * blockDim.x) {
        const bool range = (int64_t)tx[j] == x0 + (int64_t)j;
        const bool same = fr_eq(fr_from_small_pair(tx[j], ty[j], c), ld_fr(T, N, j));
        if (!range || !same) atomicMin(bad, (unsigned long long)j);
        ty_out[j] = ty[j];
    }
}

// a1 + a3(1) fused for function lookups: S = x + alpha_f y straight into Montgomery form,
// stored, and its table index computed while it is still in registers.
__global__ void __launch_bounds__(256, 4)
k_import_pair_index(const int32_t* __restrict__ x, const int32_t* __restrict__ y, uint64_t n,
                    const fr* __restrict__ consts, uint32_t* __restrict__ dst, uint64_t global_offset, TableView tv,
                    uint32_t* __restrict__ keys, unsigned long long* err) {
    __shared__ fr c[4];
    if (threadIdx.x < 4) c[threadIdx.x] = consts[threadIdx.x];
    __syncthreads();
    if ((n & 3) == 0) {
        // 4 consecutive elements per thread: 128-bit loads of x, y; 128-bit stores per limb plane; 4 hash
        // probes in flight together
        const uint64_t stride = 4 * (uint64_t)gridDim.x * blockDim.x;
        uint64_t i = 4 * (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x);
        int4 xn = make_int4(0, 0, 0, 0), yn = make_int4(0, 0, 0, 0);
        if (i < n) {
            xn = __ldg(reinterpret_cast<const int4*>(x + i));
            yn = __ldg(reinterpret_cast<const int4*>(y + i));
        }
        for (; i < n; i += stride) {
            const int4 xv = xn, yv = yn;
            if (i + stride < n) {   // prefetch the next iteration's inputs
                xn = __ldg(reinterpret_cast<const int4*>(x + i + stride));
                yn = __ldg(reinterpret_cast<const int4*>(y + i + stride));
            }
            fr s[4];
            s[0] = fr_from_small_pair(xv.x, yv.x, c);
            s[1] = fr_from_small_pair(xv.y, yv.y, c);
            s[2] = fr_from_small_pair(xv.z, yv.z, c);
            s[3] = fr_from_small_pair(xv.w, yv.w, c);
            if (dst) st_fr4(dst, n, i, s);
            uint32_t h[4], slot[4], kk[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) h[q] = hash_fr(s[q]) & tv.mask;
#pragma unroll
            for (int q = 0; q < 4; ++q) slot[q] = __ldg(tv.slots + h[q]);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                bool ok = slot[q] != 0 && aos_eq(tv.Skeys + 2 * (uint64_t)h[q], s[q]);
                uint32_t key = slot[q] - 1;
                if (!ok && slot[q] != 0) {                 // collision: keep probing
                    const int64_t f = table_find(tv, s[q]);
                    ok = f >= 0;
                    key = (uint32_t)f;
                }
                if (!ok) {
                    atomic_min_i64(err, global_offset + i + q);
                    key = 0;
                }
                kk[q] = key;
            }
            *reinterpret_cast<uint4*>(keys + i) = make_uint4(kk[0], kk[1], kk[2], kk[3]);
        }
        return;
    }
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const fr s = fr_from_small_pair(x[i], y[i], c);
        if (dst) st_fr(dst, n, i, s);
        const int64_t f = table_find(tv, s);
        uint32_t key = 0;
        if (f < 0) atomic_min_i64(err, global_offset + i);
        else key = (uint32_t)f;
        keys[i] = key;
    }
}

constexpr int kHistThreads = 512;
constexpr int kHistItems = 8;
constexpr int kHistTile = kHistThreads * kHistItems;   // 4096

__global__ void __launch_bounds__(kHistThreads, 2)
k_hist_count(const uint32_t* __restrict__ keys_in, uint64_t n, uint32_t N, uint32_t* rows, int key_bits) {
    typedef cub::BlockRadixSort<uint32_t, kHistThreads, kHistItems> Sort;
    __shared__ union {
        typename Sort::TempStorage sort;
        uint32_t keys[kHistTile];
    } sm;
    uint32_t* row = rows + (uint64_t)blockIdx.x * N;
    for (uint32_t j = threadIdx.x; j < N; j += blockDim.x) row[j] = 0;
    __syncthreads();
    const uint64_t ntiles = (n + kHistTile - 1) / kHistTile;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t base = tile * kHistTile;
        uint32_t keys[kHistItems];
#pragma unroll
        for (int g = 0; g < kHistItems / 4; ++g) {
            const uint64_t i0 = base + 4 * kHistThreads * g + 4 * threadIdx.x;
            if (i0 + 3 < n) {
                const uint4 q = __ldg(reinterpret_cast<const uint4*>(keys_in + i0));
                keys[4 * g] = q.x; keys[4 * g + 1] = q.y; keys[4 * g + 2] = q.z; keys[4 * g + 3] = q.w;
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) keys[4 * g + j] = i0 + j < n ? keys_in[i0 + j] : N;
            }
        }
        __syncthreads();   // smem union reuse across tiles
        Sort(sm.sort).Sort(keys, 0, key_bits);
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kHistItems; ++q) sm.keys[threadIdx.x * kHistItems + q] = keys[q];
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kHistItems; ++q) {
            const int p = threadIdx.x * kHistItems + q;
            const uint32_t k = sm.keys[p];
            if (k < N && (p == 0 || sm.keys[p - 1] != k)) row[k] -= (uint32_t)p;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kHistItems; ++q) {
            const int p = threadIdx.x * kHistItems + q;
            const uint32_t k = sm.keys[p];
            if (k < N && (p == kHistTile - 1 || sm.keys[p + 1] != k)) row[k] += (uint32_t)(p + 1);
        }
        __syncthreads();
    }
}

__global__ void k_hist_colsum(const uint32_t* __restrict__ rows, int nrows, uint64_t N, uint32_t* __restrict__ m) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < N; j += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t s = 0;
        for (int b = 0; b < nrows; ++b) s += rows[(uint64_t)b * N + j];
        m[j] = s;
    }
}

// ====================================================================== a4: batched inversion
// Block product tree over one value per thread (heap layout in smem: leaves at [nt, 2nt)).
// Given the inverse of the root, returns the inverse of this thread's value.
// tree, inv: 2*nt fr each.  All threads must call.  Thread 0 supplies root_inv via *root_inv_src
// (global) or, if root_inv_src == nullptr, computes it by Fermat.
__device__ void block_tree_up(fr* tree, const fr& v) {
    const int nt = blockDim.x, t = threadIdx.x;
    tree[nt + t] = v;
    __syncthreads();
    for (int width = nt >> 1; width >= 1; width >>= 1) {
        if (t < width) tree[width + t] = fr_mul(tree[2 * (width + t)], tree[2 * (width + t) + 1]);
        __syncthreads();
    }
}

// after block_tree_up; inv[1] must be set (and synced) by the caller
__device__ fr block_tree_down(const fr* tree, fr* inv) {
    const int nt = blockDim.x, t = threadIdx.x;
    for (int width = 1; width < nt; width <<= 1) {
        if (t < width) {
            const int node = width + t;
            const fr iv = inv[node];
            inv[2 * node] = fr_mul(iv, tree[2 * node + 1]);
            inv[2 * node + 1] = fr_mul(iv, tree[2 * node]);
        }
        __syncthreads();
    }
    return inv[nt + t];
}

constexpr int kInvThreads = 256;
constexpr int kInvPer = 16;                         // elements per thread
constexpr int kInvTile = kInvThreads * kInvPer;     // 4096 elements
// Hierarchical (barrier-free) batched inversion.  Level 0 holds the D_local values x = beta + S; level L+1
// holds the per-thread chain products of level L (one per 16 elements).  Thread t of tile b owns the
// chain of elements e = 2g + j (g in 0..7, j in 0..1) at tile offset 512 g + 2 t + j: each step is one
// coalesced 64-bit access per limb plane, and both elements of a round-1 pair (2y, 2y+1), y = 256 g + t
// within the tile, sit in the same thread.  Its chain product goes to next[256 b + t].
//   forward : slot(e) = p_{e-1} = x_0 ... x_{e-1} for e >= 1 (slot(0) unused), next = p_15
//   backward: given I = 1/p_15 (inverse of the next-level element), A_e = I p_{e-1}; I <- I x_e
// The top level (<= 8192 values) is inverted by one block (k_batch_invert, one Fermat).
template <bool LEVEL0>
__global__ void __launch_bounds__(kInvThreads, 2)
k_inv_fwd(const uint32_t* __restrict__ X, uint64_t n, const ProofScalars* __restrict__ sc, uint32_t* slots,
          uint32_t* next, uint64_t nnext, uint64_t t0, uint64_t t1, uint64_t err_offset, unsigned long long* err) {
    const fr beta = LEVEL0 ? sc->beta : fr_zero();
    for (uint64_t tile = t0 + blockIdx.x; tile < t1; tile += gridDim.x) {
        const uint64_t base = tile * kInvTile + 2 * threadIdx.x;
        fr p = fr_zero();
        fr xn[2];
        ld_fr2(X, n, base, xn);
#pragma unroll 1
        for (int g = 0; g < 8; ++g) {
            const uint64_t i0 = base + 512 * g;
            fr x[2] = {xn[0], xn[1]};
            if (g < 7) ld_fr2(X, n, i0 + 512, xn);   // prefetch the next step
            if (LEVEL0) {
                x[0] = fr_add(x[0], beta);
                x[1] = fr_add(x[1], beta);
                if (fr_is_zero(x[0])) atomic_min_i64(err, err_offset + i0);
                if (fr_is_zero(x[1])) atomic_min_i64(err, err_offset + i0 + 1);
            }
            const fr prev = p;                       // p_{2g-1}
            p = (g == 0) ? x[0] : fr_mul(p, x[0]);   // p_{2g}
            st_fr2(slots, n, i0, g == 0 ? p : prev, p);
            p = fr_mul(p, x[1]);                     // p_{2g+1}
        }
        st_fr(next, nnext, (tile - t0) * kInvThreads + threadIdx.x, p);
    }
}

// Inverts elements [i0, i1) of the SoA vector `vals` (stride `count`) into `out` (same layout): one
// block, chains of ceil((i1 - i0) / blockDim) per thread, one Fermat for the whole batch.
__global__ void __launch_bounds__(1024)
k_batch_invert(const uint32_t* __restrict__ vals, uint64_t count, uint64_t i0, uint64_t i1, uint32_t* out) {
    extern __shared__ fr smem_fr[];
    fr* tree = smem_fr;
    fr* inv = smem_fr + 2 * blockDim.x;
    const uint64_t len = i1 - i0;
    const uint64_t per = (len + blockDim.x - 1) / blockDim.x;
    const uint64_t lo = i0 + threadIdx.x * per, hi = min(lo + per, i1);
    fr p = fr_one();
    for (uint64_t i = lo; i < hi; ++i) {
        st_fr(out, count, i, p);                    // exclusive prefix
        p = fr_mul(p, ld_fr(vals, count, i));
    }
    block_tree_up(tree, p);
    if (threadIdx.x == 0) inv[1] = fr_inv(tree[1]);
    __syncthreads();
    fr iv = block_tree_down(tree, inv);
    for (uint64_t i = hi; i-- > lo;) {
        st_fr(out, count, i, fr_mul(ld_fr(out, count, i), iv));
        iv = fr_mul(iv, ld_fr(vals, count, i));
    }
}

// Backward pass over tiles [t0, t1): slots (prefixes) -> inverses, in place.  Level 0 writes A = 1/(beta+S)
// and fuses the round-1 evaluation (a5):
//   Hinf += W[y] (A_1 - A_0)(S_1 - S_0),  a0 += A_0,  a1 += A_1   per pair y = (2y, 2y+1);
// H0 = H1 = sum_y W[y] A_t (S_t + beta) = sum W = 1 globally (A (S + beta) = 1), no work.
// W[y] = E_hi[tile] * E_lo[y mod 2048] (a tile is one group of 2048 pairs).  Partial rows go to
// row0 + blockIdx.x.
template <bool LEVEL0>
__global__ void __launch_bounds__(kInvThreads, 2)
k_inv_bwd(const uint32_t* __restrict__ X, uint64_t n, const ProofScalars* __restrict__ sc, uint32_t* slots,
          const uint32_t* __restrict__ next_inv, uint64_t nnext, uint64_t t0, uint64_t t1,
          const fr* __restrict__ elo, const fr* __restrict__ ehi, fr* partials, int row0, int rows) {
    const fr beta = LEVEL0 ? sc->beta : fr_zero();
    const bool eval = LEVEL0 && partials != nullptr;
    fr hinf = fr_zero(), a0 = fr_zero(), a1 = fr_zero();
    for (uint64_t tile = t0 + blockIdx.x; tile < t1; tile += gridDim.x) {
        const uint64_t base = tile * kInvTile + 2 * threadIdx.x;
        fr iv = ld_fr(next_inv, nnext, (tile - t0) * kInvThreads + threadIdx.x);
        fr acc = fr_zero();
#pragma unroll 1
        for (int g = 7; g >= 0; --g) {
            const uint64_t i0 = base + 512 * g;
            fr slot[2], x[2], A0, A1;
            ld_fr2(slots, n, i0, slot);
            ld_fr2(X, n, i0, x);
            A1 = fr_mul(iv, slot[1]);
            iv = fr_mul(iv, LEVEL0 ? fr_add(x[1], beta) : x[1]);
            if (g == 0) {
                A0 = iv;
            } else {
                A0 = fr_mul(iv, slot[0]);
                iv = fr_mul(iv, LEVEL0 ? fr_add(x[0], beta) : x[0]);
            }
            st_fr2(slots, n, i0, A0, A1);
            if (eval) {
                const fr dA = fr_sub(A1, A0), dS = fr_sub(x[1], x[0]);
                acc = fr_add(acc, fr_mul(ld_fr_256(elo + 256 * g + threadIdx.x), fr_mul(dA, dS)));
                a0 = fr_add(a0, A0);
                a1 = fr_add(a1, A1);
            }
        }
        if (eval) hinf = fr_add(hinf, fr_mul(ehi[tile], acc));
    }
    if (eval) {
        __shared__ fr scratch[3 * (kInvThreads / 32)];
        fr v[3] = {hinf, a0, a1};
        block_sum_fr<3>(v, scratch);
        if (threadIdx.x == 0) {
            const int row = row0 + blockIdx.x;
            partials[SLOT_HINF * rows + row] = v[0];
            partials[SLOT_A0 * rows + row] = v[1];
            partials[SLOT_A1 * rows + row] = v[2];
        }
    }
}

// ---------------------------------------------------------------------- a4 via the table (gather path)
// Every S_i is a table entry T_j (a3 checked it), so A_i = 1/(beta + S_i) = 1/(beta + T_j) = B_j: the D-sized
// batch inversion is replaced by N inversions (B, computed first) and a gather through the hash index.
// Same tile / thread layout as k_inv_bwd<true>, and the same fused round-1 evaluation (a5).  An S_i with
// no table entry (possible only when prove is called on an S that was not prepared, e.g. a tamper trial)
// sets *miss; the host then redoes the proof with the inversion path (bit-identical A by definition).
__device__ __forceinline__ fr ld_aos_fr(const uint4* p) { return ld_fr_256(p); }

__global__ void __launch_bounds__(kInvThreads)
k_gather_round1(const uint32_t* __restrict__ S, uint64_t n, TableView tv, const uint4* __restrict__ TB,
                uint32_t* __restrict__ Aout, const fr* __restrict__ elo, const fr* __restrict__ ehi, fr* partials,
                int rows, unsigned long long* miss) {
    fr acc = fr_zero(), a0 = fr_zero(), a1 = fr_zero();
    const uint64_t tile = blockIdx.x;
    const uint64_t base = tile * kInvTile + 2 * threadIdx.x;
#pragma unroll 1
    for (int g = 0; g < 8; ++g) {
        const uint64_t i0 = base + 512 * g;
        fr x[2];
        ld_fr2(S, n, i0, x);
        uint32_t h0 = hash_fr(x[0]) & tv.mask, h1 = hash_fr(x[1]) & tv.mask;
        uint32_t s0 = __ldg(tv.slots + h0), s1 = __ldg(tv.slots + h1);
        int64_t j0 = (s0 != 0 && aos_eq(tv.Skeys + 2 * (uint64_t)h0, x[0])) ? (int64_t)(s0 - 1) : -2;
        int64_t j1 = (s1 != 0 && aos_eq(tv.Skeys + 2 * (uint64_t)h1, x[1])) ? (int64_t)(s1 - 1) : -2;
        if (j0 == -2) j0 = s0 ? table_find(tv, x[0]) : -1;
        if (j1 == -2) j1 = s1 ? table_find(tv, x[1]) : -1;
        if (j0 < 0 || j1 < 0) {
            atomic_min_i64(miss, i0);
            j0 = j0 < 0 ? 0 : j0;
            j1 = j1 < 0 ? 0 : j1;
        }
        const fr A0 = ld_aos_fr(TB + 4 * j0), A1 = ld_aos_fr(TB + 4 * j1);
        st_fr2(Aout, n, i0, A0, A1);
        const fr dA = fr_sub(A1, A0), dS = fr_sub(x[1], x[0]);
        acc = fr_add(acc, fr_mul(ld_fr_256(elo + 256 * g + threadIdx.x), fr_mul(dA, dS)));
        a0 = fr_add(a0, A0);
        a1 = fr_add(a1, A1);
    }
    fr v[3] = {fr_mul(ehi[tile], acc), a0, a1};
    __shared__ fr scratch[3 * (kInvThreads / 32)];
    block_sum_fr<3>(v, scratch);
    if (threadIdx.x == 0) {
        partials[SLOT_HINF * rows + tile] = v[0];
        partials[SLOT_A0 * rows + tile] = v[1];
        partials[SLOT_A1 * rows + tile] = v[2];
    }
}

// Same as k_gather_round1, but the table index of every S_i comes from the keys of the preceding
// zkl_tlookup_prepare on this S (ctx-cached): each key is still verified (S_i == T_key, one sector of the
// AoS table copy, loaded in parallel with B_key), so a stale or foreign S only costs the fallback.
// 3 CTAs per SM (80 registers, a few spills) hide the L2 latency of the gathers better than 2 (measured -11%).
__global__ void __launch_bounds__(kInvThreads, 3)
k_gather_keys_round1(const uint32_t* __restrict__ S, uint64_t n, const uint32_t* __restrict__ keys,
                     uint64_t N, const uint4* __restrict__ TB,
                     uint32_t* __restrict__ Aout, const fr* __restrict__ elo, const fr* __restrict__ ehi,
                     fr* partials, int rows, unsigned long long* miss) {
    fr acc = fr_zero(), a0 = fr_zero(), a1 = fr_zero();
    const uint64_t tile = blockIdx.x;
    const uint64_t base = tile * kInvTile + 2 * threadIdx.x;
#pragma unroll 1
    for (int g = 0; g < 8; ++g) {
        const uint64_t i0 = base + 512 * g;
        uint2 k = __ldg(reinterpret_cast<const uint2*>(keys + i0));
        if (k.x >= N || k.y >= N) {
            atomic_min_i64(miss, i0);
            k.x = k.x >= N ? 0 : k.x;
            k.y = k.y >= N ? 0 : k.y;
        }
        const uint4* r0 = TB + 4 * (uint64_t)k.x;
        const uint4* r1 = TB + 4 * (uint64_t)k.y;
        const fr A0 = ld_aos_fr(r0), A1 = ld_aos_fr(r1);
        fr x[2];
        ld_fr2(S, n, i0, x);
        if (!aos_eq(r0 + 2, x[0]) || !aos_eq(r1 + 2, x[1]))
            atomic_min_i64(miss, i0);
        st_fr2(Aout, n, i0, A0, A1);
        const fr dA = fr_sub(A1, A0), dS = fr_sub_lazy(x[1], x[0]);
        acc = fr_add(acc, fr_mul(ld_fr_256(elo + 256 * g + threadIdx.x), fr_mul(dA, dS)));
        a0 = fr_add(a0, A0);
        a1 = fr_add(a1, A1);
    }
    fr v[3] = {fr_mul(ehi[tile], acc), a0, a1};
    __shared__ fr scratch[3 * (kInvThreads / 32)];
    block_sum_fr<3>(v, scratch);
    if (threadIdx.x == 0) {
        partials[SLOT_HINF * rows + tile] = v[0];
        partials[SLOT_A0 * rows + tile] = v[1];
        partials[SLOT_A1 * rows + tile] = v[2];
    }
}

// Round 1 from the keys of the preceding prepare (a4 + a5 through the table, no D-sized inversion and no D-sized
// read of S): A_i = B_key(i) and S_i = T_key(i) both come from the 64-byte (B, T) record of the key, so the kernel
// reads 4 B per lookup from HBM and gathers the records from L2.  VERIFY: S was materialised and may have been
// rewritten since the prepare -- each S_i is compared with T_key (a mismatch sets *miss, the host redoes the proof
// by inversion).  WRITE_A: A is written for the caller (A is an output of Prove); otherwise A is
// never materialised: round 2 gathers it again (k_round<..., GATHER>).  Same tile / pair layout and partial rows as
// k_inv_bwd<true>: tile = 2048 pairs, thread t owns pairs 256 g + t (g = 0..7), W = E_hi[tile] E_lo[256 g + t].
#ifndef ZKL_R1_ACC_SMEM
#define ZKL_R1_ACC_SMEM 1
#endif
#ifndef ZKL_R1_CTAS
#define ZKL_R1_CTAS 3   // 24 warps per SM hide the gathers' latency better than 16 without spills (measured -7%)
#endif
template <bool VERIFY, bool WRITE_A>
__global__ void __launch_bounds__(kInvThreads, ZKL_R1_CTAS)
k_round1_keys(const uint32_t* __restrict__ S, uint64_t n, const uint32_t* __restrict__ keys, uint64_t N,
              const uint4* __restrict__ TB, uint32_t* __restrict__ Aout, const fr* __restrict__ elo,
              const fr* __restrict__ ehi, fr* partials, int rows, unsigned long long* miss, int tpc) {
    // tpc consecutive tiles per CTA (CTA b: tiles b tpc .. b tpc + tpc - 1): per tile the E_lo-weighted sum of dA dS
    // over the thread's 8 pairs is accumulated wide and scaled by that tile's E_hi; the sums of A and the block
    // reduction are paid once per CTA.  The CTA's row is row b; rows b + gridDim.x j (j >= 1) are zeroed, so the
    // round still has one row per tile.
    fr hinf = fr_zero();
#if ZKL_R1_ACC_SMEM
    // the sums of A(., 0) and A(., 1) in shared memory (18 words per thread): fewer live registers at 80
    __shared__ fr_acc sh_a[2][kInvThreads];
    sh_a[0][threadIdx.x] = fr_acc_zero();
    sh_a[1][threadIdx.x] = fr_acc_zero();
    fr_acc& a0 = sh_a[0][threadIdx.x];
    fr_acc& a1 = sh_a[1][threadIdx.x];
#else
    fr_acc a0 = fr_acc_zero(), a1 = fr_acc_zero();
#endif
#pragma unroll 1
    for (int q = 0; q < tpc; ++q) {
        fr_wide acc = fr_wide_zero();
        const uint64_t tile = (uint64_t)blockIdx.x * tpc + q;
        const uint64_t base = tile * kInvTile + 2 * threadIdx.x;
        uint2 kn = __ldg(reinterpret_cast<const uint2*>(keys + base));
#pragma unroll 1
        for (int g = 0; g < 8; ++g) {
            const uint64_t i0 = base + 512 * g;
            uint2 k = kn;
            if (g < 7) kn = __ldg(reinterpret_cast<const uint2*>(keys + i0 + 512));   // the next pair's keys
            if (k.x >= N || k.y >= N) {
                atomic_min_i64(miss, i0);
                k.x = k.x >= N ? 0 : k.x;
                k.y = k.y >= N ? 0 : k.y;
            }
            ZKL_ASSERT(k.x < N && k.y < N);
            const uint4* r0 = TB + 4 * (uint64_t)k.x;
            const uint4* r1 = TB + 4 * (uint64_t)k.y;
            const fr A0 = ld_fr_256(r0), A1 = ld_fr_256(r1);
            const fr S0 = ld_fr_256(r0 + 2), S1 = ld_fr_256(r1 + 2);
            if (VERIFY) {
                fr x[2];
                ld_fr2(S, n, i0, x);
                if (!fr_eq(x[0], S0) || !fr_eq(x[1], S1)) atomic_min_i64(miss, i0);
            }
            if (WRITE_A) st_fr2(Aout, n, i0, A0, A1);
            const fr dA = fr_sub(A1, A0), dS = fr_sub_lazy(S1, S0);
            fr_wide_mac(acc, ld_fr_256(elo + 256 * g + threadIdx.x), fr_mul(dA, dS));
            fr_acc_add(a0, A0);
            fr_acc_add(a1, A1);
        }
        hinf = fr_add(hinf, fr_mul(ehi[tile], fr_wide_redc(acc)));
    }
    fr v[3] = {hinf, fr_acc_final(a0), fr_acc_final(a1)};
    __shared__ fr scratch[3 * (kInvThreads / 32)];
    block_sum_fr<3>(v, scratch);
    if (threadIdx.x == 0) {
        partials[SLOT_HINF * rows + blockIdx.x] = v[0];
        partials[SLOT_A0 * rows + blockIdx.x] = v[1];
        partials[SLOT_A1 * rows + blockIdx.x] = v[2];
    }
    if (threadIdx.x < 3 * (tpc - 1)) {
        const int slot = threadIdx.x % 3 == 0 ? SLOT_HINF : (threadIdx.x % 3 == 1 ? SLOT_A0 : SLOT_A1);
        partials[slot * rows + blockIdx.x + gridDim.x * (1 + threadIdx.x / 3)] = fr_zero();
    }
}

// a virtual S materialised where a kernel needs the vector itself: S_i = T_key(i) (AoS table copy -> SoA)
__global__ void k_s_from_keys(const uint32_t* __restrict__ keys, uint64_t n, uint64_t N, const uint4* __restrict__ Taos,
                              uint32_t* __restrict__ dst) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t k = keys[i];
        st_fr(dst, n, i, ld_fr_256(Taos + 2 * (uint64_t)(k < N ? k : 0)));
    }
}

// (B_j, T_j) packed as one 64-byte record per entry: the gather reads both from one L2 line
__global__ void k_pack_tb(const uint32_t* __restrict__ T, const uint32_t* __restrict__ B, uint64_t n,
                          uint4* __restrict__ dst) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const fr b = ld_fr(B, n, i), t = ld_fr(T, n, i);
        dst[4 * i] = make_uint4(b.v[0], b.v[1], b.v[2], b.v[3]);
        dst[4 * i + 1] = make_uint4(b.v[4], b.v[5], b.v[6], b.v[7]);
        dst[4 * i + 2] = make_uint4(t.v[0], t.v[1], t.v[2], t.v[3]);
        dst[4 * i + 3] = make_uint4(t.v[4], t.v[5], t.v[6], t.v[7]);
    }
}

// ====================================================================== a6/a7: sumcheck rounds
// Round k >= 2 fused with the fold of round k-1 (FOLD = true), or round 1 on given vectors
// (FOLD = false, sumcheck_prove).  Pairs y of the round are split y = (y_hi, y_lo), y_lo the low
// gbits bits; W[y] = E_hi[y_hi] E_lo[y_lo]; a block processes whole groups of G = 2^gbits pairs,
// each thread G/256 of them, accumulating E_lo-weighted sums that are scaled by E_hi once per group.
constexpr int kRoundThreads = 256;
#ifndef ZKL_ROUND_PREFETCH
#define ZKL_ROUND_PREFETCH 1
#endif

#ifndef ZKL_ROUND_A0_SMEM
#define ZKL_ROUND_A0_SMEM 1
#endif
#ifndef ZKL_ROUND_STAGE
#define ZKL_ROUND_STAGE 1
#endif
// plain fold rounds: the next iteration's 4 old A and 4 old S of each thread (16 x 16 B, one per limb plane) are
// copied to shared memory with cp.async while the current pair is computed, [plane][thread] so the 16-byte reads
// are bank-conflict free; thread-private slots, so only cp.async.wait_all orders them (no block barrier)
constexpr size_t kRoundStageSmem = (ZKL_ROUND_STAGE ? 16 * kRoundThreads * 16 : 0);

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// bulk prefetch of [p, p + bytes) into L2 (cp.async.bulk.prefetch; p 16-byte aligned, bytes a multiple of 16)
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// GATHER (round 2 after k_round1_keys): the four old elements of A and S are the (B, T) records of keys[4y..4y+3]
// (A_i = B_key, S_i = T_key): 16 B of keys from HBM and four 64-byte records from L2 replace 256 B of A and S.
#ifndef ZKL_ROUND_CTAS
#define ZKL_ROUND_CTAS 2
#endif
template <bool FOLD, bool DIRECT, bool GATHER = false>
__global__ void __launch_bounds__(kRoundThreads, ZKL_ROUND_CTAS)
k_round(const uint32_t* __restrict__ Aold, const uint32_t* __restrict__ Sold, uint64_t nold,
        uint32_t* __restrict__ Anew, uint32_t* __restrict__ Snew, const ProofScalars* __restrict__ sc, int k,
        const fr* __restrict__ elo, const fr* __restrict__ ehi, int gbits, fr* partials,
        const uint32_t* __restrict__ keys = nullptr, const uint4* __restrict__ TB = nullptr) {
    constexpr bool direct_h1 = DIRECT;
#ifdef ZKL_ROUND_SCALARS_IN_REGS
    const fr beta = sc->beta;
    const fr rk = FOLD ? sc->r[k - 2] : fr_zero();
#else
    // beta and r_{k-1} are read from shared memory where they are used: 16 fewer live registers in the pair loop
    __shared__ fr sh_beta, sh_rk;
    if (threadIdx.x == 0) {
        sh_beta = sc->beta;
        sh_rk = FOLD ? sc->r[k - 2] : fr_zero();
    }
    __syncthreads();
    const fr& beta = sh_beta;
    const fr& rk = sh_rk;
#endif
    const uint64_t nnew = nold / 2;
    const uint32_t G = 1u << gbits;
    // one group of G pairs per CTA (grid = #groups): each thread accumulates its G/256 <= 64 E_lo-weighted terms
    // unreduced (fr_wide_*) and scales the reduced sums by E_hi once
    const uint64_t grp = blockIdx.x;
    fr_wide c0 = fr_wide_zero(), cinf = fr_wide_zero();
    fr c1 = fr_zero();
#if ZKL_ROUND_A0_SMEM
    // the fold rounds' sum of A(., 0) in shared memory (9 words per thread): 9 fewer live registers in the pair loop
    __shared__ fr_acc sh_a0[kRoundThreads];
    sh_a0[threadIdx.x] = fr_acc_zero();
    fr_acc a1 = fr_acc_zero();
#else
    fr_acc a0 = fr_acc_zero(), a1 = fr_acc_zero();
#endif
    constexpr bool kStage = FOLD && !GATHER && ZKL_ROUND_STAGE;
    extern __shared__ uint4 rstage[];   // [16 planes][kRoundThreads] (kStage)
    auto stage_issue = [&](uint64_t yy) {
#pragma unroll
        for (int l = 0; l < 8; ++l) {
            cp_async16(&rstage[l * kRoundThreads + threadIdx.x], Aold + (uint64_t)l * nold + 4 * yy);
            cp_async16(&rstage[(8 + l) * kRoundThreads + threadIdx.x], Sold + (uint64_t)l * nold + 4 * yy);
        }
        cp_async_commit();
    };
    if (kStage && threadIdx.x < G) stage_issue((grp << gbits) + threadIdx.x);
    for (uint32_t yl = threadIdx.x; yl < G; yl += blockDim.x) {
        const uint64_t y = (grp << gbits) + yl;
#if ZKL_ROUND_PREFETCH > 0
        // GATHER: the CTA's keys ZKL_ROUND_PREFETCH iterations ahead into L2 (one bulk prefetch), so the key load
        // at the top of the next iteration waits on L2, not HBM (-2% on round 2).  The same prefetch of the A and S
        // limb planes in the plain fold rounds measured +5% (timeline), so they load directly.
        if (FOLD && GATHER && threadIdx.x == 0) {
            const uint32_t ynext = (yl & ~(kRoundThreads - 1u)) + ZKL_ROUND_PREFETCH * kRoundThreads;
            if (ynext < G) prefetch_l2_bulk(keys + 4 * ((grp << gbits) + ynext), 16u * kRoundThreads);
        }
#endif
        fr A0, A1, S0, S1;
        if (FOLD && GATHER) {
            const uint4 kq = __ldg(reinterpret_cast<const uint4*>(keys + 4 * y));
            const uint4 *p0 = TB + 4 * (uint64_t)kq.x, *p1 = TB + 4 * (uint64_t)kq.y;
            const uint4 *p2 = TB + 4 * (uint64_t)kq.z, *p3 = TB + 4 * (uint64_t)kq.w;
            {
                const fr a0v = ld_fr_256(p0), a1v = ld_fr_256(p1), a2v = ld_fr_256(p2), a3v = ld_fr_256(p3);
                A0 = fr_add(a0v, fr_mul(rk, fr_sub_lazy(a1v, a0v)));
                A1 = fr_add(a2v, fr_mul(rk, fr_sub_lazy(a3v, a2v)));
            }
            st_fr2(Anew, nnew, 2 * y, A0, A1);
            {
                const fr s0 = ld_fr_256(p0 + 2), s1 = ld_fr_256(p1 + 2), s2 = ld_fr_256(p2 + 2),
                         s3 = ld_fr_256(p3 + 2);
                S0 = fr_add(s0, fr_mul(rk, fr_sub_lazy(s1, s0)));
                S1 = fr_add(s2, fr_mul(rk, fr_sub_lazy(s3, s2)));
            }
            st_fr2(Snew, nnew, 2 * y, S0, S1);
        } else if (kStage) {
            cp_async_wait_all();
            {   // A first, then S: half the loaded words live at a time
                fr a[4];
#pragma unroll
                for (int l = 0; l < 8; ++l) {
                    const uint4 qa = rstage[l * kRoundThreads + threadIdx.x];
                    a[0].v[l] = qa.x; a[1].v[l] = qa.y; a[2].v[l] = qa.z; a[3].v[l] = qa.w;
                }
                A0 = fr_add(a[0], fr_mul(rk, fr_sub_lazy(a[1], a[0])));
                A1 = fr_add(a[2], fr_mul(rk, fr_sub_lazy(a[3], a[2])));
            }
            {
                fr sv[4];
#pragma unroll
                for (int l = 0; l < 8; ++l) {
                    const uint4 qs = rstage[(8 + l) * kRoundThreads + threadIdx.x];
                    sv[0].v[l] = qs.x; sv[1].v[l] = qs.y; sv[2].v[l] = qs.z; sv[3].v[l] = qs.w;
                }
                S0 = fr_add(sv[0], fr_mul(rk, fr_sub_lazy(sv[1], sv[0])));
                S1 = fr_add(sv[2], fr_mul(rk, fr_sub_lazy(sv[3], sv[2])));
            }
            // the slot is reused only after the folds consumed every word read from it (in-order issue: the copies
            // cannot start before those reads returned); the copies then overlap the rest of this pair's work
            if (yl + blockDim.x < G) stage_issue(y + blockDim.x);
            st_fr2(Anew, nnew, 2 * y, A0, A1);
            st_fr2(Snew, nnew, 2 * y, S0, S1);
        } else if (FOLD) {
            {
                fr a[4];
                ld_fr4(Aold, nold, 4 * y, a);
                A0 = fr_add(a[0], fr_mul(rk, fr_sub_lazy(a[1], a[0])));
                A1 = fr_add(a[2], fr_mul(rk, fr_sub_lazy(a[3], a[2])));
            }
            st_fr2(Anew, nnew, 2 * y, A0, A1);
            {
                fr sv[4];
                ld_fr4(Sold, nold, 4 * y, sv);
                S0 = fr_add(sv[0], fr_mul(rk, fr_sub_lazy(sv[1], sv[0])));
                S1 = fr_add(sv[2], fr_mul(rk, fr_sub_lazy(sv[3], sv[2])));
            }
            st_fr2(Snew, nnew, 2 * y, S0, S1);
        } else {
            fr av[2], sv[2];
            ld_fr2(Aold, nold, 2 * y, av);
            ld_fr2(Sold, nold, 2 * y, sv);
            A0 = av[0]; A1 = av[1]; S0 = sv[0]; S1 = sv[1];
        }
        const fr e = ld_fr_256(elo + yl);
        fr_wide_mac(c0, e, fr_mul(A0, fr_add_lazy(S0, beta)));
        fr_wide_mac(cinf, e, fr_mul(fr_sub(A1, A0), fr_sub_lazy(S1, S0)));
        if (direct_h1) c1 = fr_add(c1, fr_mul(e, fr_mul(A1, fr_add_lazy(S1, beta))));
#if ZKL_ROUND_A0_SMEM
        fr_acc_add(sh_a0[threadIdx.x], A0);
#else
        fr_acc_add(a0, A0);
#endif
        if (!FOLD) fr_acc_add(a1, A1);   // FOLD rounds: a(1) follows from round k-1 (RoundDesc::a1_derived)
    }
    const fr eh = ehi[grp];
    fr H0 = fr_mul(eh, fr_wide_redc(c0));
    fr Hinf = fr_mul(eh, fr_wide_redc(cinf));
    fr H1 = direct_h1 ? fr_mul(eh, c1) : fr_zero();
    __shared__ fr scratch[5 * (kRoundThreads / 32)];
#if ZKL_ROUND_A0_SMEM
    const fr_acc a0 = sh_a0[threadIdx.x];
#endif
    fr v[5] = {H0, H1, Hinf, fr_acc_final(a0), FOLD ? fr_zero() : fr_acc_final(a1)};
    block_sum_fr<5>(v, scratch);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < 5; ++s) partials[s * gridDim.x + blockIdx.x] = v[s];
    }
}

// ====================================================================== a9: tail rounds (one CTA)
// Rounds k0..kend on <= kTailMax elements held in shared memory.  Input: either the round-(k0-1)
// vectors (2n elements, folded with r_{k0-1} on load), or the round-k0 vectors (n elements).
// mode_invert: S only is given; A = 1/(beta + S) is computed here (block batch inversion) and
// written to Aout (the whole prove for D_local < 4096).  All partial sums are direct (H0, H1, Hinf).
// After round kend the vectors are folded with r_kend; A(v), S(v) go to fin[0], fin[1].
constexpr int kTailThreads = 512;

__global__ void __launch_bounds__(kTailThreads)
k_tail(const uint32_t* __restrict__ Ain, const uint32_t* __restrict__ Sin, uint64_t nin, int fold_in,
       int mode_invert, uint32_t* Aout, uint64_t err_offset, unsigned long long* err,
       const ProofScalars* __restrict__ sc, int k0, int kend, const RoundDesc* __restrict__ rounds,
       const fr* __restrict__ arena, fr* partials_base, fr* fin) {
    extern __shared__ fr smem_fr[];
    const int nt = blockDim.x, t = threadIdx.x;
    const uint64_t n = fold_in ? nin / 2 : nin;
    fr* As = smem_fr;              // n
    fr* Ss = smem_fr + kTailMax;   // n
    fr* tree = smem_fr + 2 * kTailMax;        // 2 nt
    fr* inv = tree + 2 * nt;                  // 2 nt
    const fr beta = sc->beta;
    if (fold_in) {
        const fr r = sc->r[k0 - 2];
        for (uint64_t i = t; i < n; i += nt) {
            fr a0 = ld_fr(Ain, nin, 2 * i), a1 = ld_fr(Ain, nin, 2 * i + 1);
            fr s0 = ld_fr(Sin, nin, 2 * i), s1 = ld_fr(Sin, nin, 2 * i + 1);
            As[i] = fr_add(a0, fr_mul(r, fr_sub(a1, a0)));
            Ss[i] = fr_add(s0, fr_mul(r, fr_sub(s1, s0)));
        }
    } else {
        for (uint64_t i = t; i < n; i += nt) {
            Ss[i] = ld_fr(Sin, nin, i);
            if (!mode_invert) As[i] = ld_fr(Ain, nin, i);
        }
    }
    __syncthreads();
    if (mode_invert) {
        // chain of ceil(n / nt) consecutive elements per thread
        const uint64_t per = (n + nt - 1) / nt, lo = t * per, hi = min(lo + per, n);
        fr p = fr_one();
        for (uint64_t i = lo; i < hi; ++i) {
            fr x = fr_add(Ss[i], beta);
            if (fr_is_zero(x)) atomic_min_i64(err, err_offset + i);
            As[i] = p;
            p = fr_mul(p, x);
        }
        block_tree_up(tree, p);
        if (t == 0) inv[1] = fr_inv(tree[1]);
        __syncthreads();
        fr iv = block_tree_down(tree, inv);
        for (uint64_t i = hi; i-- > lo;) {
            fr x = fr_add(Ss[i], beta);
            As[i] = fr_mul(As[i], iv);
            iv = fr_mul(iv, x);
        }
        __syncthreads();
        for (uint64_t i = t; i < n; i += nt) st_fr(Aout, n, i, As[i]);
    }
    uint64_t len = n;
    for (int k = k0; k <= kend; ++k) {
        const RoundDesc rd = rounds[k - 1];
        const fr* elo = arena + rd.elo_off;
        const fr eh = arena[rd.ehi_off];
        fr v[5] = {fr_zero(), fr_zero(), fr_zero(), fr_zero(), fr_zero()};
        for (uint64_t y = t; y < len / 2; y += nt) {
            const fr A0 = As[2 * y], A1 = As[2 * y + 1], S0 = Ss[2 * y], S1 = Ss[2 * y + 1];
            const fr e = fr_mul(eh, elo[y]);
            v[0] = fr_add(v[0], fr_mul(e, fr_mul(A0, fr_add(S0, beta))));
            v[1] = fr_add(v[1], fr_mul(e, fr_mul(A1, fr_add(S1, beta))));
            v[2] = fr_add(v[2], fr_mul(e, fr_mul(fr_sub(A1, A0), fr_sub(S1, S0))));
            v[3] = fr_add(v[3], A0);
            v[4] = fr_add(v[4], A1);
        }
        // warp sums -> one partial row per warp (kTailThreads / 32 rows; no block-wide reduction per round)
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
            for (int q = 0; q < 5; ++q) v[q] = fr_add(v[q], shfl_down_fr(v[q], off));
        }
        if ((t & 31) == 0) {
            fr* part = partials_base + rd.part_base;
            const int nw = nt >> 5;
#pragma unroll
            for (int q = 0; q < 5; ++q) part[q * nw + (t >> 5)] = v[q];
        }
        // fold with r_k
        const fr r = sc->r[k - 1];
        fr na[4], ns[4];
        int cnt = 0;
        for (uint64_t y = t; y < len / 2; y += nt, ++cnt) {
            na[cnt] = fr_add(As[2 * y], fr_mul(r, fr_sub(As[2 * y + 1], As[2 * y])));
            ns[cnt] = fr_add(Ss[2 * y], fr_mul(r, fr_sub(Ss[2 * y + 1], Ss[2 * y])));
        }
        __syncthreads();
        cnt = 0;
        for (uint64_t y = t; y < len / 2; y += nt, ++cnt) {
            As[y] = na[cnt];
            Ss[y] = ns[cnt];
        }
        __syncthreads();
        len /= 2;
    }
    if (t == 0) {
        fin[0] = As[0];
        fin[1] = Ss[0];
    }
}

// Rounds k0..kend on n <= kTailWarpMax round-k0 elements in ONE warp: the same sums and folds as k_tail
// without block barriers (each round costs a few dependent Fr multiplications and a shuffle reduction).
constexpr int kTailWarpMax = 128;

__global__ void __launch_bounds__(32)
k_tail_warp(const uint32_t* __restrict__ Ain, const uint32_t* __restrict__ Sin, uint64_t n,
            const ProofScalars* __restrict__ sc, int k0, int kend, const RoundDesc* __restrict__ rounds,
            const fr* __restrict__ arena, fr* partials_base, fr* fin) {
    __shared__ fr As[kTailWarpMax], Ss[kTailWarpMax];
    const int lane = threadIdx.x;
    const fr beta = sc->beta;
    for (int i = lane; i < (int)n; i += 32) {
        As[i] = ld_fr(Ain, n, i);
        Ss[i] = ld_fr(Sin, n, i);
    }
    __syncwarp();
    int len = (int)n;
    for (int k = k0; k <= kend; ++k) {
        const RoundDesc rd = rounds[k - 1];
        const fr* elo = arena + rd.elo_off;
        const fr eh = arena[rd.ehi_off];
        const fr rk = sc->r[k - 1];
        const int half = len / 2;
        fr v[5] = {fr_zero(), fr_zero(), fr_zero(), fr_zero(), fr_zero()};
        constexpr int kPer = kTailWarpMax / 2 / 32;
        fr na[kPer], ns[kPer];
#pragma unroll
        for (int c = 0; c < kPer; ++c) {
            const int y = lane + 32 * c;
            if (y < half) {
                const fr e = fr_mul(eh, elo[y]);
                const fr A0 = As[2 * y], A1 = As[2 * y + 1], S0 = Ss[2 * y], S1 = Ss[2 * y + 1];
                v[SLOT_H0] = fr_add(v[SLOT_H0], fr_mul(e, fr_mul(A0, fr_add_lazy(S0, beta))));
                v[SLOT_H1] = fr_add(v[SLOT_H1], fr_mul(e, fr_mul(A1, fr_add_lazy(S1, beta))));
                v[SLOT_HINF] = fr_add(v[SLOT_HINF], fr_mul(e, fr_mul(fr_sub(A1, A0), fr_sub_lazy(S1, S0))));
                v[SLOT_A0] = fr_add(v[SLOT_A0], A0);
                v[SLOT_A1] = fr_add(v[SLOT_A1], A1);
                na[c] = fr_add(A0, fr_mul(rk, fr_sub_lazy(A1, A0)));
                ns[c] = fr_add(S0, fr_mul(rk, fr_sub_lazy(S1, S0)));
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
            for (int q = 0; q < 5; ++q) v[q] = fr_add(v[q], shfl_down_fr(v[q], off));
        }
        if (lane == 0) {
            fr* part = partials_base + rd.part_base;   // one row (nblocks = 1)
#pragma unroll
            for (int q = 0; q < 5; ++q) part[q] = v[q];
        }
        __syncwarp();
#pragma unroll
        for (int c = 0; c < kPer; ++c) {
            const int y = lane + 32 * c;
            if (y < half) {
                As[y] = na[c];
                Ss[y] = ns[c];
            }
        }
        __syncwarp();
        len = half;
    }
    if (lane == 0) {
        fin[0] = As[0];
        fin[1] = Ss[0];
    }
}

// ====================================================================== a6/a9: chunked rounds
// The pairs of round k are (2y, 2y+1), so an aligned chunk of 2^c consecutive elements folds into an aligned
// chunk of the next round: a block that owns one chunk runs c rounds on it in shared memory with no
// inter-block exchange (the challenges r_k are inputs; each round's sums leave as one partial row per block,
// reduced later).  Used once the vectors are small (<= kChunkMaxElems), where one launch per round would be
// launch- and latency-bound: rounds kc .. kc + kChunkBits - 1 in one launch, leaving one element per chunk
// for k_tail.  Input: the round-(kc-1) vectors (2 kChunk elements per block, folded with r_{kc-1} on load).
constexpr int kChunkBits = 10;
constexpr int kChunk = 1 << kChunkBits;
constexpr int kChunkThreads = 256;
constexpr uint64_t kChunkMaxElems = 1ull << 17;   // chunk rounds start at the first round with <= 2^17 elements
constexpr int kChunkWarps = kChunkThreads / 32;   // partial rows per chunk and round: one per warp

// Causal: the chunks are synchronised by a grid barrier (cooperative launch) between writing a round's partial rows
// and folding with its challenge, so r_k is never used before every CTA has finished its share of g_k (SURVEY.md
// §8(a6); the challenges being explicit inputs does not change the order the prover commits to).
__device__ __forceinline__ void
chunk_rounds_body(const uint32_t* __restrict__ Ain, const uint32_t* __restrict__ Sin, uint64_t nin,
                  const ProofScalars* __restrict__ sc, int kc, int nrounds, const RoundDesc* __restrict__ rounds,
                  const fr* __restrict__ arena, fr* partials_base, uint32_t* __restrict__ Aout,
                  uint32_t* __restrict__ Sout, GridBar* bar) {
    extern __shared__ fr smem_fr[];
    fr* As = smem_fr;
    fr* Ss = smem_fr + kChunk;
    const int t = threadIdx.x, nt = blockDim.x;
    const uint64_t nchunks = gridDim.x;
    const fr beta = sc->beta;
    {
        const fr r = sc->r[kc - 2];
        const uint64_t base = 2 * (uint64_t)blockIdx.x * kChunk;
        for (int i = t; i < kChunk; i += nt) {
            fr a[2], s2[2];
            ld_fr2(Ain, nin, base + 2 * i, a);
            ld_fr2(Sin, nin, base + 2 * i, s2);
            As[i] = fr_add(a[0], fr_mul(r, fr_sub_lazy(a[1], a[0])));
            Ss[i] = fr_add(s2[0], fr_mul(r, fr_sub_lazy(s2[1], s2[0])));
        }
    }
    __syncthreads();
    int len = kChunk;
    for (int j = 0; j < nrounds; ++j) {
        const int k = kc + j;
        const RoundDesc rd = rounds[k - 1];
        const fr* elo = arena + rd.elo_off;
        const fr* ehi = arena + rd.ehi_off;
        const uint32_t gmask = (1u << rd.gbits) - 1u;
        const int half = len / 2;
        const fr rk = sc->r[k - 1];
        fr v[5] = {fr_zero(), fr_zero(), fr_zero(), fr_zero(), fr_zero()};
        constexpr int kPer = kChunk / 2 / kChunkThreads;   // pairs per thread in the first chunk round
        fr na[kPer], ns[kPer];
#pragma unroll
        for (int c = 0; c < kPer; ++c) {
            const int yl = t + c * nt;
            if (yl < half) {
                const uint64_t y = (uint64_t)blockIdx.x * half + yl;   // pair index of round k (this rank)
                const fr e = fr_mul(ehi[y >> rd.gbits], elo[y & gmask]);
                const fr A0 = As[2 * yl], A1 = As[2 * yl + 1], S0 = Ss[2 * yl], S1 = Ss[2 * yl + 1];
                v[SLOT_H0] = fr_add(v[SLOT_H0], fr_mul(e, fr_mul(A0, fr_add_lazy(S0, beta))));
                if (rd.direct_h1) v[SLOT_H1] = fr_add(v[SLOT_H1], fr_mul(e, fr_mul(A1, fr_add_lazy(S1, beta))));
                v[SLOT_HINF] = fr_add(v[SLOT_HINF], fr_mul(e, fr_mul(fr_sub(A1, A0), fr_sub_lazy(S1, S0))));
                v[SLOT_A0] = fr_add(v[SLOT_A0], A0);
                v[SLOT_A1] = fr_add(v[SLOT_A1], A1);
                na[c] = fr_add(A0, fr_mul(rk, fr_sub_lazy(A1, A0)));
                ns[c] = fr_add(S0, fr_mul(rk, fr_sub_lazy(S1, S0)));
            }
        }
        // warp sums -> one partial row per warp (no block-wide reduction on this latency-bound path)
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
            for (int q = 0; q < 5; ++q) v[q] = fr_add(v[q], shfl_down_fr(v[q], off));
        }
        if ((t & 31) == 0) {
            fr* part = partials_base + rd.part_base;
            const uint64_t rows = nchunks * kChunkWarps, row = (uint64_t)blockIdx.x * kChunkWarps + (t >> 5);
#pragma unroll
            for (int q = 0; q < 5; ++q) part[(uint64_t)q * rows + row] = v[q];
            __threadfence();
        }
        grid_sync(bar);   // every chunk's share of g_k is written before any chunk folds with r_k
#pragma unroll
        for (int c = 0; c < kPer; ++c) {
            const int yl = t + c * nt;
            if (yl < half) {
                As[yl] = na[c];
                Ss[yl] = ns[c];
            }
        }
        __syncthreads();
        len = half;
    }
    if (t == 0) {
        st_fr(Aout, nchunks, blockIdx.x, As[0]);
        st_fr(Sout, nchunks, blockIdx.x, Ss[0]);
    }
}

struct ChunkArgs {
    const uint32_t* Ain;
    const uint32_t* Sin;
    uint64_t nin;
    const ProofScalars* sc;
    int kc, nrounds;
    const RoundDesc* rounds;
    const fr* arena;
    fr* partials_base;
    uint32_t* Aout;
    uint32_t* Sout;
    GridBar* bar;
};

// cooperative launch (the grid barrier needs every chunk CTA resident)
__global__ void __launch_bounds__(kChunkThreads, 2) k_chunk_rounds_coop(ChunkArgs a) {
    chunk_rounds_body(a.Ain, a.Sin, a.nin, a.sc, a.kc, a.nrounds, a.rounds, a.arena, a.partials_base, a.Aout, a.Sout,
                      a.bar);
}

// ====================================================================== a8: table side
// The N-sized table term, all in ONE block on the low-priority side stream (it overlaps the D side and
// occupies a single SM): build the working vectors B (LOGUP: m B), T, m, e~(u[d-n:], .) (eq table by the
// doubling construction), then for rounds k = 1..n evaluate sum_y B_t (alpha2 e_t (T_t + beta) - m_t)
// (LOGUP: -B_t + alpha2 e_t (B_t (T_t + beta) - m_t)) directly at t = 0..3 and fold with r_k.  The
// D-repeated weight N/D cancels against the D/N repetitions (a8).  tab_sums[k-1][t];
// tfin = the fully folded B, T, m, e.  wk: 8 N fr of scratch (two AoS buffers of 4 N).
__device__ __forceinline__ fr tab_term(const fr& b, const fr& t, const fr& m, const fr& e, const fr& beta,
                                       const fr& alpha2, int variant) {
    if (variant == ZKL_VARIANT_PAPER) return fr_mul(b, fr_sub(fr_mul(fr_mul(alpha2, e), fr_add(t, beta)), m));
    return fr_sub(fr_mul(fr_mul(alpha2, e), fr_sub(fr_mul(b, fr_add(t, beta)), m)), b);
}

// Big table rounds run multi-block on the main stream (pairs > kTabTailPairs), the rest in one block on the
// side stream.  Working vectors are AoS: [B | T | M | E] with stride len.
constexpr uint64_t kTabTailPairs = 4096;

__global__ void k_tab_init(const uint32_t* __restrict__ Bin, const uint32_t* __restrict__ Tin,
                           const uint32_t* __restrict__ m_u32, const uint32_t* __restrict__ Mfin, uint64_t N,
                           const ProofScalars* __restrict__ sc, int d, int nbits, int variant, fr* cur,
                           uint32_t* Bout) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < N; j += (uint64_t)gridDim.x * blockDim.x) {
        fr mv;
        if (m_u32) {
            mv = fr_zero();
            mv.v[0] = m_u32[j];
            mv = fr_to_mont(mv);
        } else {
            mv = ld_fr(Mfin, N, j);
        }
        fr b = ld_fr(Bin, N, j);
        if (m_u32 && variant == ZKL_VARIANT_LOGUP) b = fr_mul(b, mv);
        if (Bout) st_fr(Bout, N, j, b);   // the variant's B, for the caller
        cur[j] = b;
        cur[N + j] = ld_fr(Tin, N, j);
        cur[2 * N + j] = mv;
        // e~(u[d-n:], j): coordinate d-n+b at bit position n-1-b of j
        fr e = fr_one();
        for (int c = 0; c < nbits; ++c) {
            const fr u = sc->u[d - nbits + c];
            e = fr_mul(e, ((j >> (nbits - 1 - c)) & 1) ? u : fr_sub(fr_one(), u));
        }
        cur[3 * N + j] = e;
    }
}

// one table round over `len` entries: direct evaluation at t = 0..3 and fold with r_k; per-block partials
__device__ __forceinline__ void tab_pair(const fr* cur, uint64_t len, uint64_t y, fr* nxt, const fr& r, const fr& beta,
                                         const fr& alpha2, int variant, fr (&g)[4]) {
    const uint64_t np = len / 2;
    const fr b0 = cur[2 * y], b1 = cur[2 * y + 1];
    const fr t0 = cur[len + 2 * y], t1 = cur[len + 2 * y + 1];
    const fr m0 = cur[2 * len + 2 * y], m1 = cur[2 * len + 2 * y + 1];
    const fr e0 = cur[3 * len + 2 * y], e1 = cur[3 * len + 2 * y + 1];
    const fr db = fr_sub(b1, b0), dt = fr_sub(t1, t0), dm = fr_sub(m1, m0), de = fr_sub(e1, e0);
    fr bt = b0, tt = t0, mt = m0, et = e0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (q > 0) { bt = fr_add(bt, db); tt = fr_add(tt, dt); mt = fr_add(mt, dm); et = fr_add(et, de); }
        g[q] = fr_add(g[q], tab_term(bt, tt, mt, et, beta, alpha2, variant));
    }
    nxt[y] = fr_add(b0, fr_mul(r, db));
    nxt[np + y] = fr_add(t0, fr_mul(r, dt));
    nxt[2 * np + y] = fr_add(m0, fr_mul(r, dm));
    nxt[3 * np + y] = fr_add(e0, fr_mul(r, de));
}

__global__ void __launch_bounds__(256)
k_tab_round(const fr* __restrict__ cur, uint64_t len, fr* nxt, const ProofScalars* __restrict__ sc, int k, int variant,
            fr* tpart, int rows_max) {
    const fr beta = sc->beta, alpha2 = sc->alpha2, r = sc->r[k - 1];
    fr g[4] = {fr_zero(), fr_zero(), fr_zero(), fr_zero()};
    for (uint64_t y = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; y < len / 2; y += (uint64_t)gridDim.x * blockDim.x)
        tab_pair(cur, len, y, nxt, r, beta, alpha2, variant, g);
    __shared__ fr scratch[4 * 8];
    block_sum_fr<4>(g, scratch);
    if (threadIdx.x == 0) {
        for (int q = 0; q < 4; ++q) tpart[q * rows_max + blockIdx.x] = g[q];   // row stride rows_max
    }
}

// Chunked table rounds (as k_chunk_rounds on the D side): a block owns kTabChunk consecutive entries of the
// four working vectors and runs kTabChunkBits rounds on them in shared memory; partial rows per warp.
// out: the chunks' last entries, AoS [B | T | M | E] with stride nchunks (= gridDim.x).
constexpr int kTabChunkBits = 9;
constexpr int kTabChunk = 1 << kTabChunkBits;
constexpr int kTabChunkThreads = kTabChunk / 2;
constexpr int kTabChunkWarps = kTabChunkThreads / 32;
constexpr uint64_t kTabChunkMaxElems = (uint64_t)kTabChunk << 8;   // <= 256 chunks; bigger rounds multi-block
constexpr int kTabRowsMax = 256 * kTabChunkWarps;                  // partial-row stride per round and slot

__global__ void __launch_bounds__(kTabChunkThreads)
k_tab_chunk(const fr* __restrict__ cur, uint64_t len, fr* __restrict__ out, const ProofScalars* __restrict__ sc,
            int k0, int variant, fr* tpart) {
    extern __shared__ fr smem_fr[];
    fr* V = smem_fr;   // [4][kTabChunk]
    const int t = threadIdx.x;
    const uint64_t nchunks = gridDim.x, base = (uint64_t)blockIdx.x * kTabChunk;
    for (int i = t; i < kTabChunk; i += blockDim.x) {
#pragma unroll
        for (int q = 0; q < 4; ++q) V[q * kTabChunk + i] = cur[q * len + base + i];
    }
    __syncthreads();
    const fr beta = sc->beta, alpha2 = sc->alpha2;
    int l = kTabChunk;
    for (int j = 0; j < kTabChunkBits; ++j) {
        const int k = k0 + j;
        const int half = l / 2;
        const fr r = sc->r[k - 1];
        fr g[4] = {fr_zero(), fr_zero(), fr_zero(), fr_zero()};
        fr nv[4];
        if (t < half) {
            fr a0[4], d[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                a0[q] = V[q * kTabChunk + 2 * t];
                d[q] = fr_sub(V[q * kTabChunk + 2 * t + 1], a0[q]);
            }
            fr bt = a0[0], tt = a0[1], mt = a0[2], et = a0[3];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (q > 0) { bt = fr_add(bt, d[0]); tt = fr_add(tt, d[1]); mt = fr_add(mt, d[2]); et = fr_add(et, d[3]); }
                g[q] = tab_term(bt, tt, mt, et, beta, alpha2, variant);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) nv[q] = fr_add(a0[q], fr_mul(r, d[q]));
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
            for (int q = 0; q < 4; ++q) g[q] = fr_add(g[q], shfl_down_fr(g[q], off));
        }
        if ((t & 31) == 0) {
            const uint64_t row = (uint64_t)blockIdx.x * kTabChunkWarps + (t >> 5);
#pragma unroll
            for (int q = 0; q < 4; ++q) tpart[((uint64_t)(k - 1) * 4 + q) * kTabRowsMax + row] = g[q];
        }
        __syncthreads();
        if (t < half) {
#pragma unroll
            for (int q = 0; q < 4; ++q) V[q * kTabChunk + t] = nv[q];
        }
        __syncthreads();
        l = half;
    }
    if (t == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) out[q * nchunks + blockIdx.x] = V[q * kTabChunk];
    }
}

// The remaining table rounds k0..n in one block; also reduces the partial rows of the big rounds.
// tpart: rounds 1..k0-1, round k at tpart + (k-1) * 4 * rows_max, [q][blk], tnb[k-1] blocks.
__global__ void __launch_bounds__(256)
k_tab_tail(fr* cur, fr* nxt, uint64_t len, int k0, int nbits, const ProofScalars* __restrict__ sc, int variant,
           const fr* __restrict__ tpart, int rows_max, const uint32_t* __restrict__ tnb, fr* tab_sums, fr* tfin) {
    __shared__ fr scratch[4 * 8];
    const int t = threadIdx.x, nt = blockDim.x;
    for (int k = 1; k < k0; ++k) {
        fr g[4];
        for (int q = 0; q < 4; ++q) {
            g[q] = fr_zero();
            for (uint32_t b = t; b < tnb[k - 1]; b += nt) g[q] = fr_add(g[q], tpart[((uint64_t)(k - 1) * 4 + q) * rows_max + b]);
        }
        block_sum_fr<4>(g, scratch);
        if (t == 0)
            for (int q = 0; q < 4; ++q) tab_sums[(k - 1) * 4 + q] = g[q];
    }
    const fr beta = sc->beta, alpha2 = sc->alpha2;
    for (int k = k0; k <= nbits; ++k) {
        const uint64_t np = len / 2;
        fr g[4] = {fr_zero(), fr_zero(), fr_zero(), fr_zero()};
        for (uint64_t y = t; y < np; y += nt) tab_pair(cur, len, y, nxt, sc->r[k - 1], beta, alpha2, variant, g);
        block_sum_fr<4>(g, scratch);
        if (t == 0)
            for (int q = 0; q < 4; ++q) tab_sums[(k - 1) * 4 + q] = g[q];
        __syncthreads();
        fr* tmp = cur; cur = nxt; nxt = tmp;
        len = np;
    }
    if (t == 0) {
        tfin[0] = cur[0];
        tfin[1] = cur[len];
        tfin[2] = cur[2 * len];
        tfin[3] = cur[3 * len];
    }
}

// ====================================================================== setup / derivation
// eq tables for every round: job list (offset, ncoords, first coordinate, times rank_eq)
struct EqJob {
    uint64_t off;
    uint32_t nbits;
    uint32_t c0;
    uint32_t scale;
    uint32_t pad;
};

__global__ void k_eq_fill(const EqJob* __restrict__ jobs, int njobs, uint64_t total, const ProofScalars* __restrict__ sc,
                          fr* arena) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        int jb = 0;
        while (jb + 1 < njobs && jobs[jb + 1].off <= i) ++jb;
        const EqJob J = jobs[jb];
        const uint64_t y = i - J.off;
        fr e = J.scale ? sc->rank_eq : fr_one();
        for (uint32_t b = 0; b < J.nbits; ++b) {
            const fr u = sc->u[J.c0 + b];
            const bool bit = (y >> (J.nbits - 1 - b)) & 1;
            e = fr_mul(e, bit ? u : fr_sub(fr_one(), u));
        }
        arena[i] = e;
    }
}

// Canonical challenges -> Montgomery scalars; rank factor eq(u[0:p], rank); w = N / D.
__global__ void k_setup(const zkl_fr* __restrict__ host_chal, int d, int pbits, int rank, uint64_t N, uint64_t D,
                        ProofScalars* sc) {
    // one thread per challenge (3 + 2d <= 83 Montgomery conversions in parallel, launched with 128 threads), then
    // this rank's eq factor on thread 0
    const int i = threadIdx.x;
    if (blockIdx.x != 0) return;
    if (i < 3 + 2 * d) {
        fr x;
        for (int l = 0; l < 8; ++l) x.v[l] = host_chal[i].w[l];
        x = fr_to_mont(x);
        if (i == 0) sc->beta = x;
        else if (i == 1) sc->alpha1 = x;
        else if (i == 2) sc->alpha2 = x;
        else if (i < 3 + d) sc->u[i - 3] = x;
        else sc->r[i - 3 - d] = x;
    }
    __syncthreads();
    if (i != 0) return;
    fr re = fr_one();
    for (int b = 0; b < pbits; ++b) {
        const bool bit = (rank >> (pbits - 1 - b)) & 1;
        re = fr_mul(re, bit ? sc->u[b] : fr_sub(fr_one(), sc->u[b]));
    }
    sc->rank_eq = re;
    (void)N; (void)D;
}

// Sum of each round's per-block partial rows -> rank_sums[k][slot] (this rank's contribution).
__global__ void k_reduce_rounds(const fr* __restrict__ partials, const RoundDesc* __restrict__ rounds, int nrounds,
                                fr* rank_sums) {
    __shared__ fr scratch[5 * 32];
    const int k = blockIdx.x;   // 0-based round (relative to `rounds`)
    if (k >= nrounds) return;
    const uint32_t nb = rounds[k].nblocks;
    fr v[5];
#pragma unroll
    for (int s = 0; s < 5; ++s) {
        v[s] = fr_zero();
        for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x)
            v[s] = fr_add(v[s], partials[rounds[k].part_base + (uint64_t)s * nb + b]);
    }
    block_sum_fr<5>(v, scratch);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < 5; ++s) rank_sums[k * kSlots + s] = v[s];
    }
}

// Per-round constants that depend only on the challenges (a7), computed on the side stream at the start
// of a proof: C_k = prod_{j<k} l_{d-j}(r_j), cl_t = alpha1 C_k l_c(t) (c = d - k), the inverse of
// cl_1 = alpha1 C_k u_c (one batch inversion, one Fermat), the Lagrange basis L_t(r_k) on {0,1,2,3},
// and 2^{-(k-n)} for the rounds after the table coordinates are bound.
struct RoundConst {
    fr cl[4];
    fr inv_cl1;   // 0 when cl_1 = 0
    fr L[4];
    fr tscale;
};

__global__ void k_round_consts(const ProofScalars* __restrict__ sc, int d, int n, RoundConst* rc) {
    __shared__ fr C[kMaxRounds + 1];
    const int k = threadIdx.x + 1;   // one thread per round
    if (threadIdx.x == 0) {
        fr c = fr_one();
        for (int j = 1; j <= d; ++j) {
            C[j] = c;
            const fr u = sc->u[d - j];
            const fr l0 = fr_sub(fr_one(), u);
            c = fr_mul_s(c, fr_add(l0, fr_mul_s(sc->r[j - 1], fr_sub(u, l0))));
        }
    }
    __syncthreads();
    if (k <= d) {
        const fr one = fr_one(), two = fr_two_m(), three = fr_three_m();
        const fr u = sc->u[d - k];
        const fr coef = fr_mul_s(sc->alpha1, C[k]);
        RoundConst& q = rc[k - 1];
        q.cl[0] = fr_mul_s(coef, fr_sub(one, u));
        q.cl[1] = fr_mul_s(coef, u);
        q.cl[2] = fr_mul_s(coef, fr_sub(fr_mul_s(three, u), one));
        q.cl[3] = fr_mul_s(coef, fr_sub(fr_mul_s(fr_five_m(), u), two));
        const fr x = sc->r[k - 1];
        const fr xm1 = fr_sub(x, one), xm2 = fr_sub(x, two), xm3 = fr_sub(x, three);
        const fr inv2 = fr_inv2_m(), inv6 = fr_inv6_m();
        q.L[0] = fr_neg(fr_mul_s(fr_mul_s(fr_mul_s(xm1, xm2), xm3), inv6));
        q.L[1] = fr_mul_s(fr_mul_s(fr_mul_s(x, xm2), xm3), inv2);
        q.L[2] = fr_neg(fr_mul_s(fr_mul_s(fr_mul_s(x, xm1), xm3), inv2));
        q.L[3] = fr_mul_s(fr_mul_s(fr_mul_s(x, xm1), xm2), inv6);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // batch inversion of the nonzero cl_1 (one Fermat) and the 2^{-(k-n)} scales
        fr pre[kMaxRounds], acc = fr_one();
        for (int j = 0; j < d; ++j) {
            pre[j] = acc;
            if (!fr_is_zero(rc[j].cl[1])) acc = fr_mul_s(acc, rc[j].cl[1]);
        }
        fr iv = fr_inv(acc);
        for (int j = d - 1; j >= 0; --j) {
            if (fr_is_zero(rc[j].cl[1])) {
                rc[j].inv_cl1 = fr_zero();
            } else {
                rc[j].inv_cl1 = fr_mul_s(iv, pre[j]);
                iv = fr_mul_s(iv, rc[j].cl[1]);
            }
        }
        fr ts = fr_one();
        for (int j = 1; j <= d; ++j) {
            if (j > n) ts = fr_mul_s(ts, fr_inv2_m());
            rc[j - 1].tscale = ts;
        }
    }
}

// Round derivation (a7): g_k(t) = cl_t H(t) + a(t) + tab_k(t).  H(1) is derived from
// g_k(0) + g_k(1) = g_{k-1}(r_{k-1}) when the round did not sum it directly, H(2) = -H0 + 2 H1 + 2 Hinf,
// H(3) = -2 H0 + 3 H1 + 6 Hinf.  Every quantity is affine in the running claim c_{k-1}: each thread
// builds its round's affine forms in parallel, thread 0 runs the chain c_k = alpha_k c_{k-1} + beta_k
// (one multiplication per round), then the threads finish their rounds.
// D-side sums of local rounds are summed over the `nranks` rows of `gathered`; rounds > dl use
// `repl_sums` (replicated, already global).  fin_loc: A(v), S(v); tfin: B, T, M, E2 at v'.
struct Affine {
    fr a, b;   // a * c + b
};

__global__ void k_derive(const fr* __restrict__ gathered, int nranks, int dl, const fr* __restrict__ repl_sums,
                         const RoundDesc* __restrict__ rounds, const fr* __restrict__ tab_sums,
                         const ProofScalars* __restrict__ sc, const RoundConst* __restrict__ rc, int d, int n,
                         int variant, int prove_mode, const fr* __restrict__ fin_loc, const fr* __restrict__ tfin,
                         ProofOut* out) {
    __shared__ Affine form[kMaxRounds][4];    // g_k(t) as affine functions of c_{k-1}
    __shared__ Affine step[kMaxRounds];
    __shared__ fr claim[kMaxRounds + 1];
    __shared__ fr sums[kMaxRounds][kSlots];
    const int k = threadIdx.x + 1;
    const fr one = fr_one(), zero = fr_zero();
    if (k <= d) {
        for (int q = 0; q < 5; ++q) {
            fr v = zero;
            if (k <= dl) {
                for (int p = 0; p < nranks; ++p)
                    v = fr_add(v, gathered[((uint64_t)p * dl + (k - 1)) * kSlots + q]);
            } else {
                v = repl_sums[(k - dl - 1) * kSlots + q];
            }
            sums[k - 1][q] = v;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0)   // a(1) of the FOLD rounds from the previous round (one product per such round)
        for (int j = 2; j <= d; ++j)
            if (rounds[j - 1].a1_derived) {
                const fr p0 = sums[j - 2][SLOT_A0], p1 = sums[j - 2][SLOT_A1];
                sums[j - 1][SLOT_A1] = fr_sub(fr_add(p0, fr_mul_s(sc->r[j - 2], fr_sub(p1, p0))), sums[j - 1][SLOT_A0]);
            }
    __syncthreads();
    if (k <= d) {
        fr s[5];
        for (int q = 0; q < 5; ++q) s[q] = sums[k - 1][q];
        const RoundConst q = rc[k - 1];
        fr tab[4];
        if (k <= n) {
            for (int t = 0; t < 4; ++t) tab[t] = tab_sums[(k - 1) * 4 + t];
        } else {
            const fr tb = tfin[0], tt = tfin[1], tm = tfin[2], te = tfin[3];
            const fr tau = (variant == ZKL_VARIANT_PAPER)
                ? fr_mul_s(tb, fr_sub(fr_mul_s(fr_mul_s(sc->alpha2, te), fr_add(tt, sc->beta)), tm))
                : fr_sub(fr_mul_s(fr_mul_s(sc->alpha2, te), fr_sub(fr_mul_s(tb, fr_add(tt, sc->beta)), tm)), tb);
            const fr c = fr_mul_s(tau, q.tscale);
            for (int t = 0; t < 4; ++t) tab[t] = c;
        }
        fr H0 = s[SLOT_H0];
        const fr H1d = s[SLOT_H1], Hinf = s[SLOT_HINF], a0 = s[SLOT_A0], a1 = s[SLOT_A1];
        fr H1c = H1d;
        if (k == 1 && prove_mode) { H0 = one; H1c = one; }
        const fr g0 = fr_add(fr_add(fr_mul_s(q.cl[0], H0), a0), tab[0]);
        const bool direct = (k == 1) || rounds[k - 1].direct_h1 || fr_is_zero(q.cl[1]);
        // H1 = p1 c + q1
        fr p1 = zero, q1 = H1c;
        Affine g1;
        if (direct) {
            g1 = Affine{zero, fr_add(fr_add(fr_mul_s(q.cl[1], H1c), a1), tab[1])};
        } else {
            p1 = q.inv_cl1;
            q1 = fr_neg(fr_mul_s(fr_add(fr_add(g0, a1), tab[1]), q.inv_cl1));
            g1 = Affine{one, fr_neg(g0)};
        }
        const fr three = fr_three_m(), six = fr_six_m();
        const fr da = fr_sub(a1, a0);
        // H2 = -H0 + 2 H1 + 2 Hinf ; H3 = -2 H0 + 3 H1 + 6 Hinf
        const Affine H2{fr_add(p1, p1), fr_add(fr_sub(fr_add(q1, q1), H0), fr_add(Hinf, Hinf))};
        const Affine H3{fr_mul_s(three, p1), fr_add(fr_sub(fr_mul_s(three, q1), fr_add(H0, H0)), fr_mul_s(six, Hinf))};
        const Affine g2{fr_mul_s(q.cl[2], H2.a), fr_add(fr_add(fr_mul_s(q.cl[2], H2.b), fr_add(a0, fr_add(da, da))), tab[2])};
        const Affine g3{fr_mul_s(q.cl[3], H3.a), fr_add(fr_add(fr_mul_s(q.cl[3], H3.b), fr_add(a0, fr_mul_s(three, da))), tab[3])};
        form[k - 1][0] = Affine{zero, g0};
        form[k - 1][1] = g1;
        form[k - 1][2] = g2;
        form[k - 1][3] = g3;
        // c_k = sum_t g_t L_t
        step[k - 1] = Affine{fr_add(fr_add(fr_mul_s(g1.a, q.L[1]), fr_mul_s(g2.a, q.L[2])), fr_mul_s(g3.a, q.L[3])),
                             fr_add(fr_add(fr_mul_s(g0, q.L[0]), fr_mul_s(g1.b, q.L[1])),
                                    fr_add(fr_mul_s(g2.b, q.L[2]), fr_mul_s(g3.b, q.L[3])))};
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        fr c = (variant == ZKL_VARIANT_PAPER) ? fr_add(sc->alpha1, sc->alpha2) : sc->alpha1;
        for (int j = 0; j < d; ++j) {
            claim[j] = c;
            c = fr_add(fr_mul_s(step[j].a, c), step[j].b);
        }
        claim[d] = c;
    }
    __syncthreads();
    if (k <= d) {
        const fr c = claim[k - 1];
        for (int t = 0; t < 4; ++t) out->evals[k - 1][t] = to_canon(fr_add(fr_mul_s(form[k - 1][t].a, c), form[k - 1][t].b));
    }
    if (threadIdx.x == 0) {
        out->finals[0] = to_canon(fin_loc[0]);
        out->finals[1] = to_canon(fin_loc[1]);
        out->finals[2] = to_canon(tfin[0]);
        out->finals[3] = to_canon(tfin[1]);
        out->finals[4] = to_canon(tfin[2]);
    }
}

// beta + T_j (zero check: DIV_ZERO_T) -> x (SoA), for the table-side batch inversion
__global__ void k_add_beta(const uint32_t* __restrict__ T, uint64_t N, const ProofScalars* __restrict__ sc,
                           uint32_t* x, unsigned long long* err) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < N; j += (uint64_t)gridDim.x * blockDim.x) {
        const fr v = fr_add(ld_fr(T, N, j), sc->beta);
        if (fr_is_zero(v)) atomic_min_i64(err, j);
        st_fr(x, N, j, v);
    }
}

// copy SoA vector (same n)
__global__ void k_copy_vec(const uint32_t* __restrict__ src, uint64_t n, uint32_t* __restrict__ dst) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < 8 * n; i += (uint64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

}  // namespace zkl

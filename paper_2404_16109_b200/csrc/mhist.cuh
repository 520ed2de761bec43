// a3 multiplicities m (Eq. hab22-coefs: m_j = #{i : S_i = T_j}) for tables of N <= 2^16
// entries: an atomic-free two-digit counting pass over the u32 index-map keys (key_i = j with S_i = T_j).
//
// Every counter is private to one thread (u16 in shared memory, [bin][thread] so a warp's 32 updates hit 16
// words in 16 banks), so no update ever races and no atomic instruction is issued, whatever the skew (C4's
// causal mask puts ~half of all keys in one bin).  With n = log2 N and h = key >> 8 the high digit:
//   k_mh_count    per 32768-key chunk c: tot[c][h]                                  (reads the keys)
//   k_mh_scan     per digit h: rel[c][h] = sum_{c' < c} tot[c'][h], total[h]        (n <= 8: m = total, done)
//   k_mh_scatter  per chunk: the low byte of every key to its slot in a digit-major byte array (reads the keys
//                 again; the positions come from the same per-thread counters, recounted)
//   k_mh_lo       per piece (<= 32768 bytes of one digit h): counts of the low byte -> row h of m, or a partial
//                 row when the digit spans several pieces
//   k_mh_fix      per digit spanning several pieces (or none): m row h = sum of its partial rows (or 0)
// Traffic ~ 3 x 4 B/key read + 1 B/key written and read back; no per-CTA N-sized rows.
#pragma once
#include <cub/block/block_scan.cuh>

#include "common.cuh"

namespace zkl {

constexpr int kMhThreads = 128;
constexpr uint32_t kMhChunk = 32768;   // keys per chunk (k_mh_count / k_mh_scatter) and bytes per piece (k_mh_lo)
constexpr int kMhBins = 256;
constexpr size_t kMhSmem = (size_t)kMhBins * kMhThreads * sizeof(uint16_t);   // 64 KB of private counters
constexpr uint32_t kMhNone = 0xffffffffu;

__host__ __device__ inline uint64_t mh_chunks(uint64_t n) { return (n + kMhChunk - 1) / kMhChunk; }

__device__ __forceinline__ void mh_zero(uint16_t* cnt) {
    uint4* p = reinterpret_cast<uint4*>(cnt);
    for (uint32_t i = threadIdx.x; i < kMhSmem / 16; i += kMhThreads) p[i] = make_uint4(0, 0, 0, 0);
}

// the keys of chunk `c` taken by this thread, in a fixed order (the scatter recounts in the same order):
// 64 uint4 per thread, 8 in flight per step.  FULL: the chunk lies inside [0, n) (no bounds checks, no sentinel)
template <bool FULL, typename F>
__device__ __forceinline__ void mh_for_keys(const uint32_t* __restrict__ keys, uint64_t n, uint64_t c, F&& f) {
    constexpr int kIters = kMhChunk / (4 * kMhThreads), kUnroll = 8;
    const uint64_t base = c * kMhChunk;
    auto load = [&](int it0, uint4 (&q)[kUnroll]) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint64_t i = base + 4 * ((uint64_t)threadIdx.x + (uint64_t)kMhThreads * (it0 + u));
            if (FULL || i + 4 <= n) {
                q[u] = __ldg(reinterpret_cast<const uint4*>(keys + i));
            } else {
                q[u].x = i < n ? keys[i] : kMhNone;
                q[u].y = i + 1 < n ? keys[i + 1] : kMhNone;
                q[u].z = i + 2 < n ? keys[i + 2] : kMhNone;
                q[u].w = i + 3 < n ? keys[i + 3] : kMhNone;
            }
        }
    };
    // the next 8 loads are in flight while the current 32 keys are counted
    uint4 q[kUnroll], qn[kUnroll];
    load(0, q);
#pragma unroll 1
    for (int it0 = 0; it0 < kIters; it0 += kUnroll) {
        if (it0 + kUnroll < kIters) load(it0 + kUnroll, qn);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            f(q[u].x);
            f(q[u].y);
            f(q[u].z);
            f(q[u].w);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) q[u] = qn[u];
    }
}

// sum over threads of the counters of bin b (rotated start: the 128 threads summing their bins use 32 banks)
__device__ __forceinline__ uint32_t mh_bin_sum(const uint16_t* cnt, int b) {
    const uint32_t* row = reinterpret_cast<const uint32_t*>(cnt + b * kMhThreads);
    uint32_t s = 0;
#pragma unroll 8
    for (int j = 0; j < kMhThreads / 2; ++j) {
        const uint32_t w = row[(j + threadIdx.x) & (kMhThreads / 2 - 1)];
        s += (w & 0xffffu) + (w >> 16);
    }
    return s;
}

__device__ __forceinline__ void mh_count_chunk(const uint32_t* __restrict__ keys, uint64_t n, uint64_t c, int sh,
                                               uint16_t* cnt) {
    uint16_t* mine = cnt + threadIdx.x;
    if ((c + 1) * kMhChunk <= n)
        mh_for_keys<true>(keys, n, c, [&](uint32_t k) { mine[(k >> sh) * kMhThreads] += 1; });
    else
        mh_for_keys<false>(keys, n, c, [&](uint32_t k) {
            if (k != kMhNone) mine[(k >> sh) * kMhThreads] += 1;
        });
}

// tot[c][h] (h = key >> sh; sh = 8 if n > 8, else 0 and h is the key itself)
__global__ void __launch_bounds__(kMhThreads)
k_mh_count(const uint32_t* __restrict__ keys, uint64_t n, int sh, uint32_t* __restrict__ tot) {
    extern __shared__ __align__(16) uint16_t mh_cnt[];
    mh_zero(mh_cnt);
    __syncthreads();
    mh_count_chunk(keys, n, blockIdx.x, sh, mh_cnt);
    __syncthreads();
    for (int b = threadIdx.x; b < kMhBins; b += kMhThreads) tot[(uint64_t)blockIdx.x * kMhBins + b] = mh_bin_sum(mh_cnt, b);
}

// one CTA per digit h: rel[c][h] = sum_{c' < c} tot[c'][h] and total[h]; m_direct (n <= 8): m[h] = total[h], h < N
__global__ void __launch_bounds__(256)
k_mh_scan(const uint32_t* __restrict__ tot, uint32_t C, uint32_t* __restrict__ rel, uint32_t* __restrict__ total,
          uint32_t* __restrict__ m_direct, uint32_t N) {
    typedef cub::BlockScan<uint32_t, 256> Scan;
    __shared__ typename Scan::TempStorage tmp;
    const int h = blockIdx.x;
    const uint32_t per = (C + 255) / 256, c0 = threadIdx.x * per, c1 = min(C, c0 + per);
    uint32_t s = 0;
    for (uint32_t c = c0; c < c1; ++c) s += tot[(uint64_t)c * kMhBins + h];
    uint32_t ex, all;
    Scan(tmp).ExclusiveSum(s, ex, all);
    if (rel)
        for (uint32_t c = c0; c < c1; ++c) {
            rel[(uint64_t)c * kMhBins + h] = ex;
            ex += tot[(uint64_t)c * kMhBins + h];
        }
    if (threadIdx.x == 0) {
        total[h] = all;
        if (m_direct && (uint32_t)h < N) m_direct[h] = all;
    }
}

// exclusive scan of total[0 .. 255] into base[] (128 threads, 2 digits each); with npc: pieces per digit and the
// first piece of each digit (pfirst[256] = all pieces)
__device__ __forceinline__ void mh_digit_bases(const uint32_t* __restrict__ total, uint32_t* base, uint32_t* npc,
                                               uint32_t* pfirst) {
    typedef cub::BlockScan<uint32_t, kMhThreads> Scan;
    __shared__ typename Scan::TempStorage tmp;
    const int t = threadIdx.x;
    const uint32_t a = total[2 * t], b = total[2 * t + 1];
    uint32_t ex;
    Scan(tmp).ExclusiveSum(a + b, ex);
    base[2 * t] = ex;
    base[2 * t + 1] = ex + a;
    if (npc) {
        __syncthreads();
        const uint32_t pa = (a + kMhChunk - 1) / kMhChunk, pb = (b + kMhChunk - 1) / kMhChunk;
        uint32_t ep, allp;
        Scan(tmp).ExclusiveSum(pa + pb, ep, allp);
        npc[2 * t] = pa;
        npc[2 * t + 1] = pb;
        pfirst[2 * t] = ep;
        pfirst[2 * t + 1] = ep + pa;
        if (t == 0) pfirst[kMhBins] = allp;
    }
    __syncthreads();
}

// per chunk: the low byte of each key to out[base[h] + rel[c][h] + (rank among the chunk's keys of digit h)].
// The chunk is first ordered by digit in shared memory (local positions from the private counters), then each
// digit's run is copied out by one warp with consecutive lanes on consecutive bytes (coalesced stores).
constexpr size_t kMhScatterSmem = kMhSmem + kMhChunk;
__global__ void __launch_bounds__(kMhThreads)
k_mh_scatter(const uint32_t* __restrict__ keys, uint64_t n, const uint32_t* __restrict__ tot,
             const uint32_t* __restrict__ rel, const uint32_t* __restrict__ total, uint8_t* __restrict__ out) {
    extern __shared__ __align__(16) uint16_t mh_cnt[];
    uint8_t* buf = reinterpret_cast<uint8_t*>(mh_cnt + kMhBins * kMhThreads);
    __shared__ uint32_t start[kMhBins], lstart[kMhBins + 1];
    mh_digit_bases(total, start, nullptr, nullptr);
    {   // the chunk's digit runs in shared memory: lstart = exclusive scan of tot[c][.] (k_mh_count)
        typedef cub::BlockScan<uint32_t, kMhThreads> Scan;
        __shared__ typename Scan::TempStorage tmp;
        const int t = threadIdx.x;
        const uint32_t* ct = tot + (uint64_t)blockIdx.x * kMhBins;
        const uint32_t a = ct[2 * t], b = ct[2 * t + 1];
        uint32_t ex, all;
        Scan(tmp).ExclusiveSum(a + b, ex, all);
        lstart[2 * t] = ex;
        lstart[2 * t + 1] = ex + a;
        if (t == 0) lstart[kMhBins] = all;
    }
    for (int b = threadIdx.x; b < kMhBins; b += kMhThreads) start[b] += rel[(uint64_t)blockIdx.x * kMhBins + b];
    mh_zero(mh_cnt);
    __syncthreads();
    mh_count_chunk(keys, n, blockIdx.x, 8, mh_cnt);
    __syncthreads();
    // per bin, the local position of each thread's first key: lstart[b] + exclusive prefix over the threads (one
    // warp per bin, 4 counters per lane; < kMhChunk fits u16)
    {
        const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int b = w; b < kMhBins; b += kMhThreads / 32) {
            uint2* p = reinterpret_cast<uint2*>(mh_cnt + b * kMhThreads) + lane;
            const uint2 q = *p;
            const uint32_t c0 = q.x & 0xffffu, c1 = q.x >> 16, c2 = q.y & 0xffffu, c3 = q.y >> 16;
            const uint32_t sum = c0 + c1 + c2 + c3;
            uint32_t inc = sum;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, inc, off);
                if (lane >= off) inc += v;
            }
            const uint32_t e0 = lstart[b] + inc - sum, e1 = e0 + c0, e2 = e1 + c1, e3 = e2 + c2;
            *p = make_uint2(e0 | (e1 << 16), e2 | (e3 << 16));
        }
    }
    __syncthreads();
    uint16_t* mine = mh_cnt + threadIdx.x;
    auto put = [&](uint32_t k) {
        uint16_t& pos = mine[(k >> 8) * kMhThreads];
        buf[pos] = (uint8_t)k;
        pos += 1;
    };
    if ((blockIdx.x + 1) * (uint64_t)kMhChunk <= n)
        mh_for_keys<true>(keys, n, blockIdx.x, put);
    else
        mh_for_keys<false>(keys, n, blockIdx.x, [&](uint32_t k) { if (k != kMhNone) put(k); });
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int h = w; h < kMhBins; h += kMhThreads / 32) {
        const uint32_t l0 = lstart[h], c = lstart[h + 1] - l0;
        uint8_t* dst = out + start[h];
        for (uint32_t i = lane; i < c; i += 32) dst[i] = buf[l0 + i];
    }
}

// per piece (<= kMhChunk bytes of one digit): counts of the low byte; a digit of one piece writes its m row
__global__ void __launch_bounds__(kMhThreads)
k_mh_lo(const uint8_t* __restrict__ out, const uint32_t* __restrict__ total, uint32_t* __restrict__ m,
        uint32_t* __restrict__ partial) {
    extern __shared__ __align__(16) uint16_t mh_cnt[];
    __shared__ uint32_t base[kMhBins], npc[kMhBins], pfirst[kMhBins + 1];
    __shared__ int s_h;
    mh_digit_bases(total, base, npc, pfirst);
    if (blockIdx.x >= pfirst[kMhBins]) return;
    if (threadIdx.x == 0) {
        int lo = 0, hi = kMhBins - 1;   // the digit h with pfirst[h] <= blockIdx.x < pfirst[h] + npc[h]
        while (lo < hi) {
            const int mid = (lo + hi + 1) / 2;
            if (pfirst[mid] <= blockIdx.x) lo = mid; else hi = mid - 1;
        }
        s_h = lo;   // nonempty: an empty digit h has pfirst[h + 1] = pfirst[h], so h + 1 would qualify too
    }
    mh_zero(mh_cnt);
    __syncthreads();
    const int h = s_h;
    const uint32_t piece = blockIdx.x - pfirst[h];
    const uint64_t s = (uint64_t)base[h] + (uint64_t)piece * kMhChunk;
    const uint64_t e = min((uint64_t)base[h] + total[h], s + kMhChunk);
    uint16_t* mine = mh_cnt + threadIdx.x;
    const uint64_t sa = min(e, (uint64_t)((s + 15) & ~15ull)), ea = max(sa, (uint64_t)(e & ~15ull));
    for (uint64_t i = s + threadIdx.x; i < sa; i += kMhThreads) mine[out[i] * kMhThreads] += 1;
    for (uint64_t i = ea + threadIdx.x; i < e; i += kMhThreads) mine[out[i] * kMhThreads] += 1;
#pragma unroll 4
    for (uint64_t i = sa + 16 * (uint64_t)threadIdx.x; i < ea; i += 16 * kMhThreads) {
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(out + i));
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int bsh = 0; bsh < 32; bsh += 8) mine[((w[j] >> bsh) & 0xffu) * kMhThreads] += 1;
    }
    __syncthreads();
    for (int v = threadIdx.x; v < kMhBins; v += kMhThreads) {
        const uint32_t c = mh_bin_sum(mh_cnt, v);
        if (npc[h] == 1) m[((uint64_t)h << 8) + v] = c;
        else partial[(uint64_t)blockIdx.x * kMhBins + v] = c;
    }
}

// per digit h (of nd = N / 256): rows of digits with no keys are 0; digits spanning several pieces sum them
__global__ void __launch_bounds__(kMhThreads)
k_mh_fix(const uint32_t* __restrict__ total, const uint32_t* __restrict__ partial, uint32_t* __restrict__ m) {
    __shared__ uint32_t base[kMhBins], npc[kMhBins], pfirst[kMhBins + 1];
    mh_digit_bases(total, base, npc, pfirst);
    const int h = blockIdx.x;
    const uint32_t np = npc[h];
    if (np == 1) return;
    for (int v = threadIdx.x; v < kMhBins; v += kMhThreads) {
        uint32_t s = 0;
        for (uint32_t q = 0; q < np; ++q) s += partial[(uint64_t)(pfirst[h] + q) * kMhBins + v];
        m[((uint64_t)h << 8) + v] = s;
    }
}

}  // namespace zkl

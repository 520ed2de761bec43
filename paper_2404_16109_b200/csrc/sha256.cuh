// SHA-256 (FIPS 180-4) for the device-side Fiat-Shamir transcript.  Single-thread,
// message-at-a-time: the transcript hashes a few hundred bytes per round, off the throughput path.
#pragma once
#include <stdint.h>

namespace zkl {

__device__ __constant__ uint32_t kSha256K[64] = {
    0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u, 0xab1c5ed5u,
    0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu, 0x9bdc06a7u, 0xc19bf174u,
    0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, 0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau,
    0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, 0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u,
    0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, 0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u,
    0xa2bfe8a1u, 0xa81a664bu, 0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u,
    0x19a4c116u, 0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
    0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u, 0xc67178f2u};

__device__ __forceinline__ uint32_t sha_rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

// Fully unrolled: the 16-word message schedule window stays in registers and the round constants become immediates
// (a rolled loop kept w[64] in local memory: the per-round transcript hash was ~5x slower).
__device__ inline void sha256_block(uint32_t (&h)[8], const uint8_t* blk) {
    uint32_t w[16];
#pragma unroll
    for (int i = 0; i < 16; ++i)
        w[i] = ((uint32_t)blk[4 * i] << 24) | ((uint32_t)blk[4 * i + 1] << 16) | ((uint32_t)blk[4 * i + 2] << 8) |
               (uint32_t)blk[4 * i + 3];
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], k = h[7];
#pragma unroll
    for (int i = 0; i < 64; ++i) {
        if (i >= 16) {
            const uint32_t w15 = w[(i - 15) & 15], w2 = w[(i - 2) & 15];
            const uint32_t s0 = sha_rotr(w15, 7) ^ sha_rotr(w15, 18) ^ (w15 >> 3);
            const uint32_t s1 = sha_rotr(w2, 17) ^ sha_rotr(w2, 19) ^ (w2 >> 10);
            w[i & 15] = w[i & 15] + s0 + w[(i - 7) & 15] + s1;
        }
        const uint32_t S1 = sha_rotr(e, 6) ^ sha_rotr(e, 11) ^ sha_rotr(e, 25);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t t1 = k + S1 + ch + kSha256K[i] + w[i & 15];
        const uint32_t S0 = sha_rotr(a, 2) ^ sha_rotr(a, 13) ^ sha_rotr(a, 22);
        const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        const uint32_t t2 = S0 + mj;
        k = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += k;
}

// one compression from 16 message words (big-endian words of the byte stream).  One out-of-line copy with the 64
// rounds as 4 passes of 16 unrolled rounds: the 16-word schedule window stays in registers (constant indices) and the
// code is ~300 instructions instead of ~1,000 per inlined copy -- the transcript runs on one warp between grid
// barriers, where a long straight-line stream misses the instruction cache on every round.
static __device__ __noinline__ void sha256_block_w(uint32_t (&h)[8], const uint32_t* m) {
    uint32_t w[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) w[i] = m[i];
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], k = h[7];
#pragma unroll 1
    for (int r = 0; r < 64; r += 16) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (r > 0) {
                const uint32_t w15 = w[(i + 1) & 15], w2 = w[(i + 14) & 15];
                const uint32_t s0 = sha_rotr(w15, 7) ^ sha_rotr(w15, 18) ^ (w15 >> 3);
                const uint32_t s1 = sha_rotr(w2, 17) ^ sha_rotr(w2, 19) ^ (w2 >> 10);
                w[i] = w[i] + s0 + w[(i + 9) & 15] + s1;
            }
            const uint32_t S1 = sha_rotr(e, 6) ^ sha_rotr(e, 11) ^ sha_rotr(e, 25);
            const uint32_t ch = (e & f) ^ (~e & g);
            const uint32_t t1 = k + S1 + ch + kSha256K[r + i] + w[i];
            const uint32_t S0 = sha_rotr(a, 2) ^ sha_rotr(a, 13) ^ sha_rotr(a, 22);
            const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
            const uint32_t t2 = S0 + mj;
            k = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
        }
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += k;
}

__device__ __forceinline__ void sha256_init(uint32_t (&h)[8]) {
    h[0] = 0x6a09e667u; h[1] = 0xbb67ae85u; h[2] = 0x3c6ef372u; h[3] = 0xa54ff53au;
    h[4] = 0x510e527fu; h[5] = 0x9b05688cu; h[6] = 0x1f83d9abu; h[7] = 0x5be0cd19u;
}

// The two per-round transcript hashes on words, no byte buffers (the byte layout is the one
// sha256() would hash).  hw: the digest as its 8 big-endian words.
// h_k = SHA256(h_{k-1} || "g" || le32(k) || g_k(0..3) as 4 x 8 LE words): 165 bytes, 3 blocks
static __device__ __noinline__ void sha256_round_msg(uint32_t (&hw)[8], uint32_t k, const uint32_t (&e)[32]) {
    uint32_t m[48];
#pragma unroll
    for (int i = 0; i < 8; ++i) m[i] = hw[i];
    m[8] = (0x67u << 24) | ((k & 0xffu) << 16) | (((k >> 8) & 0xffu) << 8) | ((k >> 16) & 0xffu);
    uint32_t prev = k >> 24;   // the byte before the current word's first three
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        m[9 + j] = (prev << 24) | (__byte_perm(e[j], 0, 0x0123) >> 8);
        prev = e[j] >> 24;
    }
    m[41] = (prev << 24) | (0x80u << 16);
#pragma unroll
    for (int i = 42; i < 47; ++i) m[i] = 0;
    m[47] = 165u * 8u;
    uint32_t h[8];
    sha256_init(h);
    sha256_block_w(h, m);
    sha256_block_w(h, m + 16);
    sha256_block_w(h, m + 32);
#pragma unroll
    for (int i = 0; i < 8; ++i) hw[i] = h[i];
}

// SHA256(h || label || le32(idx)) for a label of <= 7 bytes (one block); d: the digest's big-endian words
static __device__ __noinline__ void sha256_chal_msg(const uint32_t (&hw)[8], const char* label, int llen,
                                                    uint32_t idx, uint32_t (&d)[8]) {
    uint32_t m[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) m[i] = hw[i];
#pragma unroll
    for (int i = 8; i < 16; ++i) m[i] = 0;
    const int n = 32 + llen + 4;
    auto put = [&](int pos, uint32_t byte) { m[pos >> 2] |= byte << (24 - 8 * (pos & 3)); };
    for (int i = 0; i < llen; ++i) put(32 + i, (uint8_t)label[i]);
    for (int i = 0; i < 4; ++i) put(32 + llen + i, (idx >> (8 * i)) & 0xffu);
    put(n, 0x80u);
    m[15] = (uint32_t)n * 8u;
    sha256_init(d);
    sha256_block_w(d, m);
}

// digest (32 bytes, big-endian words as in FIPS 180-4) of msg[0..len); one out-of-line copy per translation unit
static __device__ __noinline__ void sha256(const uint8_t* msg, uint32_t len, uint8_t* out) {
    uint32_t h[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                     0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
    uint8_t blk[64];
    uint32_t i = 0;
    for (; i + 64 <= len; i += 64) sha256_block(h, msg + i);
    const uint32_t rem = len - i;
    for (uint32_t j = 0; j < rem; ++j) blk[j] = msg[i + j];
    blk[rem] = 0x80;
    for (uint32_t j = rem + 1; j < 64; ++j) blk[j] = 0;
    if (rem >= 56) {
        sha256_block(h, blk);
        for (int j = 0; j < 64; ++j) blk[j] = 0;
    }
    const uint64_t bits = (uint64_t)len * 8;
    for (int j = 0; j < 8; ++j) blk[63 - j] = (uint8_t)(bits >> (8 * j));
    sha256_block(h, blk);
    for (int j = 0; j < 8; ++j) {
        out[4 * j] = (uint8_t)(h[j] >> 24);
        out[4 * j + 1] = (uint8_t)(h[j] >> 16);
        out[4 * j + 2] = (uint8_t)(h[j] >> 8);
        out[4 * j + 3] = (uint8_t)h[j];
    }
}

}  // namespace zkl

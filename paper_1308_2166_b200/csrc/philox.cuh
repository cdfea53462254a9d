// philox.cuh -- device-side counter-based randomness for the estimator update.
//
// Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11) and Lemire's multiply-shift bounded integer
// with rejection.  The draw placement is DESIGN.md reading R7 (the paper is silent on the RNG;
// PAPER.md:988-989): per (global estimator id i, non-empty batch index b) ONE Philox block
//     ctr = (i.lo32, i.hi32, b, 0), key = (seed.lo32, seed.hi32)
// whose words (x,y) feed Step 1's draw randInt(|W|+|E|) and (z,w) Step 2's draw
// over chi^- + chi^+ (PAPER.md:564-569, 825-830).  A rejected Lemire sample takes retry t from the
// block with ctr.w = base + t (base 0x10000 for Step 1, 0x20000 for Step 2), low 64 bits.
#pragma once
#include <cstdint>

namespace tcb {

struct PhiloxKey {
    uint32_t k0, k1;
};

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, PhiloxKey k) {
#pragma unroll
    for (int rnd = 0; rnd < 10; ++rnd) {
        if (rnd) {
            k.k0 += 0x9E3779B9u;
            k.k1 += 0xBB67AE85u;
        }
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k.k0, lo1, hi0 ^ c.w ^ k.k1, lo0);
    }
    return c;
}

struct DrawCtx {
    uint64_t id;
    uint32_t batch;
    PhiloxKey key;
};

__device__ __forceinline__ uint64_t retry_word(const DrawCtx &d, uint32_t w) {
    const uint4 o = philox4x32_10(make_uint4((uint32_t)d.id, (uint32_t)(d.id >> 32), d.batch, w), d.key);
    return (uint64_t)o.x | ((uint64_t)o.y << 32);
}

// Lemire: hi64(x*n) unless lo64(x*n) < (2^64 - n) mod n, in which case redraw.
__device__ __forceinline__ uint64_t bounded(uint64_t n, uint64_t x, const DrawCtx &d, uint32_t base) {
    uint64_t lo = x * n;
    uint64_t hi = __umul64hi(x, n);
    if (lo < n) {  // rare: the slow path computes the exact rejection threshold
        const uint64_t t = (0ull - n) % n;
        uint32_t k = 0;
        while (lo < t) {
            x = retry_word(d, base + (++k));
            lo = x * n;
            hi = __umul64hi(x, n);
        }
    }
    return hi;
}

}  // namespace tcb

// index.cuh -- device data structures of the per-batch incidence index.
//
// Per batch W = <w_0 .. w_{s-1}> the GPU builds, in HBM:
//   E[k]      uint2  normalized edge (lo < hi)                        (the F array's edges)
//   vt        open-addressing vertex table, 16 B slots {key, epoch, deg, start}: deg_W(x) and the start
//             of x's segment in segS; epoch-tagged so no per-batch clearing
//   segS      uint32 per arc (k<<1 | side), grouped by vertex, ascending k inside a group: the rankAll
//             order of Fig. 4 read backwards (src asc, pos desc <=> rank asc), so
//             rank(x->y) of arc at sorted slot s is segEnd(x) - 1 - s (Definition Rank)
//   einfo[k]  uint4 {slot of the lo-arc, segEnd(lo), slot of the hi-arc, segEnd(hi)}
//   pt        edge-pair hash, 16 B slots {lo, hi, k, epoch}: Step 3's (src,dst)-sorted "edges" array
//             with its multisearch replaced by one O(1) probe
#pragma once
#include <cstdint>

namespace tcb {

constexpr uint32_t kEmptyV = 0xFFFFFFFFu;
constexpr uint32_t kClosedBit = 0x80000000u;
constexpr uint32_t kCMask = 0x7FFFFFFFu;

// error word bits (host decodes with priority INVAL > LOOP > DUP > OVF)
constexpr uint32_t kErrInval = 1u;
constexpr uint32_t kErrLoop = 2u;
constexpr uint32_t kErrDup = 4u;
constexpr uint32_t kErrOvf = 8u;

// in-segment ordering classes
constexpr uint32_t kSmallSeg = 32;   // deg <= kSmallSeg: per-arc counting rank
constexpr uint32_t kChunk = 2048;    // big segments: smem bitonic sort per chunk of <= kChunk arcs

struct __align__(16) VSlot {
    uint32_t key, epoch, deg, start;
};
struct __align__(16) PSlot {
    uint32_t lo, hi, pos, epoch;
};

__device__ __forceinline__ uint32_t hash_vertex(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

__device__ __forceinline__ uint32_t hash_pair(uint32_t lo, uint32_t hi) {
    uint64_t x = ((uint64_t)lo << 32) | hi;
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return (uint32_t)x;
}

// Probe the (complete, read-only) vertex table: deg_W(v) and segment end, (0, 0) when v is not in W.
__device__ __forceinline__ void vt_find(const VSlot *__restrict__ vt, uint32_t mask, uint32_t epoch, uint32_t v,
                                        uint32_t &deg, uint32_t &end) {
    uint32_t h = hash_vertex(v) & mask;
    while (true) {
        const uint4 s = __ldg(reinterpret_cast<const uint4 *>(vt) + h);
        if (s.y != epoch) {
            deg = 0;
            end = 0;
            return;
        }
        if (s.x == v) {
            deg = s.z;
            end = s.w + s.z;
            return;
        }
        h = (h + 1) & mask;
    }
}

// Probe the (complete, read-only) edge-pair hash: batch position of (lo, hi) or -1.
__device__ __forceinline__ int64_t pt_find(const PSlot *__restrict__ pt, uint32_t mask, uint32_t epoch, uint32_t lo,
                                           uint32_t hi) {
    uint32_t h = hash_pair(lo, hi) & mask;
    while (true) {
        const uint4 s = __ldg(reinterpret_cast<const uint4 *>(pt) + h);
        if (s.w != epoch) return -1;
        if (s.x == lo && s.y == hi) return (int64_t)s.z;
        h = (h + 1) & mask;
    }
}

}  // namespace tcb

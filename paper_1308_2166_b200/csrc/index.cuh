// index.cuh -- device data structures of the per-batch incidence index.
//
// Per batch W = <w_0 .. w_{s-1}> the GPU builds, in HBM:
//   E[k]      uint2  normalized edge (lo < hi)                        (the F array's edges)
//   vertex table (open addressing, 8-key buckets = one 32-byte sector):
//             vkey[slot] u32 vertex id (kEmptyV = free), vinfo[slot] = {deg_W(x), start of x's segment}
//   segS      uint32 per arc (k<<1 | side), grouped by vertex, ascending k inside a group: the rankAll
//             order of Fig. 4 read backwards (src asc, pos desc <=> rank asc), so
//             rank(x->y) of the arc at sorted slot s is segEnd(x) - 1 - s (Definition Rank)
//   einfo[k]  uint4 {slot of the lo-arc, segEnd(lo), slot of the hi-arc, segEnd(hi)}
//   edge-pair hash (4-key buckets = one 32-byte sector): pkey[slot] u64 = lo<<32 | hi, ppos[slot] = k:
//             Step 3's (src,dst)-sorted "edges" array with its multisearch replaced by
//             one O(1) probe
// Tables are emptied after every batch by clearing exactly the slots the batch used (no full memset).
#pragma once
#include <cstdint>

namespace tcb {

constexpr uint32_t kEmptyV = 0xFFFFFFFFu;
constexpr unsigned long long kEmptyP = ~0ull;
constexpr uint32_t kNoSlot = 0xFFFFFFFFu;
constexpr uint32_t kClosedBit = 0x80000000u;
constexpr uint32_t kCMask = 0x7FFFFFFFu;

// error word bits (host decodes with priority INVAL > LOOP > DUP > OVF)
constexpr uint32_t kErrInval = 1u;
constexpr uint32_t kErrLoop = 2u;
constexpr uint32_t kErrDup = 4u;
constexpr uint32_t kErrOvf = 8u;

// in-segment ordering classes (by deg_W)
constexpr uint32_t kTinySeg = 16;   // thread per segment, register sorting network
constexpr uint32_t kMidSeg = 256;   // warp per segment, shared-memory bitonic network
constexpr uint32_t kChunk = 2048;   // block per chunk of <= kChunk arcs; chunks merged by rank

constexpr uint32_t kVBucket = 8;  // vertex keys per probe (32 B)
constexpr uint32_t kPBucket = 4;  // pair keys per probe (32 B)

__device__ __forceinline__ uint32_t hash_vertex(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

__device__ __forceinline__ uint32_t hash_pair(unsigned long long key) {
    uint64_t x = key;
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return (uint32_t)x;
}

__device__ __forceinline__ unsigned long long pair_key(uint32_t lo, uint32_t hi) {
    return ((unsigned long long)lo << 32) | hi;
}

// index of the first lane of a uint4 equal to v (0..3), or -1
__device__ __forceinline__ int match4(uint4 k, uint32_t v) {
    return k.x == v ? 0 : k.y == v ? 1 : k.z == v ? 2 : k.w == v ? 3 : -1;
}

// Probe the complete (read-only) vertex table: {deg_W(v), segment start}, or {0, 0} when v is not in W.
__device__ __forceinline__ uint2 vt_find(const uint32_t *__restrict__ vkey, const uint2 *__restrict__ vinfo,
                                         uint32_t mask, uint32_t v) {
    uint32_t b = hash_vertex(v) & mask & ~(kVBucket - 1);
    while (true) {
        const uint4 *p = reinterpret_cast<const uint4 *>(vkey + b);
        const uint4 k0 = __ldg(p), k1 = __ldg(p + 1);
        int j = match4(k0, v);
        if (j < 0) {
            j = match4(k1, v);
            if (j >= 0) j += 4;
        }
        if (j >= 0) return __ldg(vinfo + b + j);
        if (match4(k0, kEmptyV) >= 0 || match4(k1, kEmptyV) >= 0) return make_uint2(0u, 0u);
        b = (b + kVBucket) & mask;
    }
}

// Probe the complete (read-only) edge-pair hash: batch position of (lo, hi) or -1.
__device__ __forceinline__ int64_t pt_find(const unsigned long long *__restrict__ pkey,
                                           const uint32_t *__restrict__ ppos, uint32_t mask,
                                           unsigned long long key) {
    uint32_t b = hash_pair(key) & mask & ~(kPBucket - 1);
    while (true) {
        const ulonglong2 *p = reinterpret_cast<const ulonglong2 *>(pkey + b);
        const ulonglong2 a = __ldg(p), c = __ldg(p + 1);
        const int j = a.x == key ? 0 : a.y == key ? 1 : c.x == key ? 2 : c.y == key ? 3 : -1;
        if (j >= 0) return (int64_t)__ldg(ppos + b + j);
        if (a.x == kEmptyP || a.y == kEmptyP || c.x == kEmptyP || c.y == kEmptyP) return -1;
        b = (b + kPBucket) & mask;
    }
}

}  // namespace tcb

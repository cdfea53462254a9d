// index.cuh -- device data structures of the per-batch incidence index.
//
// Per batch W = <w_0 .. w_{s-1}> the GPU builds, in HBM:
//   E[k]      uint2  normalized edge (lo < hi)                        (the F array's edges)
//   sorted arcs: the 2|W| arcs (vertex, k<<1|side) stably radix-sorted by vertex.  Because arcs enter in
//             arrival order, each vertex's run holds its arcs in increasing k: the rankAll order of
//             Fig. 4 read backwards inside each src group (src asc, pos desc <=> rank asc,
//             PAPER.md:730-734), so rank(x->y) of the arc at sorted slot s is segEnd(x) - 1 - s
//             (Definition Rank).  segS = the sorted value array.
//   vertex table (open addressing, 16 B slots, 2 per 32 B sector): {x, deg_W(x), segment start, tag}
//   einfo[k]  uint4 {slot of the lo-arc, segEnd(lo), slot of the hi-arc, segEnd(hi)}
//   edge-pair hash (16 B slots, 2 per sector): {lo<<32 | hi, k, tag}: Step 3's (src,dst)-sorted "edges"
//             array with its multisearch replaced by one O(1) probe
// A slot is live only when its tag equals the batch's tag, so the tables are never cleared; a slot is
// claimed with one 128-bit CAS that installs key, payload and tag together.
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
// errors found while staging (they stop the index build); a duplicate (found by k_pairs concurrently) or
// an overflow (set by the host) only stop the estimator update
constexpr uint32_t kErrStage = kErrInval | kErrLoop;

// radix sort of arcs by vertex id
constexpr uint32_t kRadixBits = 8;
constexpr uint32_t kRadix = 1u << kRadixBits;
constexpr uint32_t kPasses = 32 / kRadixBits;
constexpr uint32_t kSortThreads = 256;
constexpr uint32_t kSortItems = 16;
constexpr uint32_t kRadixTile = kSortThreads * kSortItems;  // arcs per radix tile (= 2048 edges)
constexpr uint32_t kRunItems = 8;
constexpr uint32_t kTile = kSortThreads * kRunItems;  // arcs per segment tile (k_runs / k_fix)

// device counters (ctr[])
constexpr int kCtrD = 0;    // vertices of W (claimed vertex-table slots)
constexpr int kCtrErr = 3;  // error bits
constexpr int kCtrWords = 16;

struct __align__(16) VSlot {
    uint32_t key, deg, start, tag;
};
struct __align__(16) PSlot {
    unsigned long long key;
    uint32_t pos, tag;
};

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

// Probe the complete (read-only) vertex table: {deg_W(v), segment start}, or {0, 0} when v is not in W.
// One probe = one 32-byte sector holding two slots.
__device__ __forceinline__ uint2 vt_find(const VSlot *__restrict__ vt, uint32_t mask, uint32_t tag, uint32_t v) {
    uint32_t b = hash_vertex(v) & mask & ~1u;
    while (true) {
        const uint4 *p = reinterpret_cast<const uint4 *>(vt + b);
        const uint4 s0 = __ldg(p), s1 = __ldg(p + 1);
        const bool l0 = s0.w == tag, l1 = s1.w == tag;
        if (l0 && s0.x == v) return make_uint2(s0.y, s0.z);
        if (l1 && s1.x == v) return make_uint2(s1.y, s1.z);
        if (!l0 || !l1) return make_uint2(0u, 0u);
        b = (b + 2) & mask;
    }
}

// Two independent vertex probes whose first sectors are requested together.
__device__ __forceinline__ void vt_find2(const VSlot *__restrict__ vt, uint32_t mask, uint32_t tag, uint32_t u,
                                         uint32_t v, uint2 &iu, uint2 &iv) {
    const uint32_t bu = hash_vertex(u) & mask & ~1u, bv = hash_vertex(v) & mask & ~1u;
    const uint4 *pu = reinterpret_cast<const uint4 *>(vt + bu);
    const uint4 *pv = reinterpret_cast<const uint4 *>(vt + bv);
    const uint4 u0 = __ldg(pu), u1 = __ldg(pu + 1), v0 = __ldg(pv), v1 = __ldg(pv + 1);
    const bool lu0 = u0.w == tag, lu1 = u1.w == tag, lv0 = v0.w == tag, lv1 = v1.w == tag;
    if (lu0 && u0.x == u) iu = make_uint2(u0.y, u0.z);
    else if (lu1 && u1.x == u) iu = make_uint2(u1.y, u1.z);
    else if (!lu0 || !lu1) iu = make_uint2(0u, 0u);
    else iu = vt_find(vt, mask, tag, u);  // rare: first bucket full without u
    if (lv0 && v0.x == v) iv = make_uint2(v0.y, v0.z);
    else if (lv1 && v1.x == v) iv = make_uint2(v1.y, v1.z);
    else if (!lv0 || !lv1) iv = make_uint2(0u, 0u);
    else iv = vt_find(vt, mask, tag, v);
}

// Probe the complete (read-only) edge-pair hash: batch position of (lo, hi) or -1.
__device__ __forceinline__ int64_t pt_find(const PSlot *__restrict__ pt, uint32_t mask, uint32_t tag,
                                           unsigned long long key) {
    uint32_t b = hash_pair(key) & mask & ~1u;
    while (true) {
        const ulonglong2 *p = reinterpret_cast<const ulonglong2 *>(pt + b);
        const ulonglong2 s0 = __ldg(p), s1 = __ldg(p + 1);
        const bool l0 = (uint32_t)(s0.y >> 32) == tag, l1 = (uint32_t)(s1.y >> 32) == tag;
        if (l0 && s0.x == key) return (int64_t)(uint32_t)s0.y;
        if (l1 && s1.x == key) return (int64_t)(uint32_t)s1.y;
        if (!l0 || !l1) return -1;
        b = (b + 2) & mask;
    }
}

}  // namespace tcb

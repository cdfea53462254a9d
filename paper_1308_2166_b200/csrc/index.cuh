// index.cuh -- device data structures of the per-batch incidence index (DESIGN.md §5 "HBM layout").
//
// Per batch W = <w_0 .. w_{s-1}> the GPU builds, in HBM:
//   E[k]      uint2  normalised edge (lo < hi)                       (the F array's edges)
//   segS[]    u32    the 2|W| arcs (k<<1 | side) grouped by vertex, arrival order inside a vertex: rankAll's
//             (src asc, pos desc) order read backwards inside each src group, so
//             rank(x->y) of the arc at slot s = segEnd(x) - 1 - s (Definition Rank).
//             Vertices are grouped by BUCKET (the top bv bits of hash_vertex), each bucket owns the slot
//             range of its arcs; inside a bucket vertices appear in hash order.
//   apos[k]   uint2  partition positions of edge k's two arcs; pslot[p] uint2 {slot in segS, segment end} of the
//             arc at partition position p (a fresh f1 = W[j] reads apos[j], then its two pslot entries)
//   vertex table: one open-addressing slice per vertex bucket, min(next_pow2(2 D_b), 2 n_b) slots (load <= 1/2)
//             for the bucket's D_b distinct vertices (n_b arcs), 16 B slots {x, deg_W(x), segment start, 0}, at
//             offset 2 * (the bucket's first arc slot) -- slices never overlap and need no prefix sum;
//             vslice[b] = {offset, size}.
//             Slices are written whole every batch (empty slots included), so the table needs no tags.
//   edge-pair table: ceil(3w / 4) groups of four 8-byte slots {k, tag|fp} (one 32-byte sector per group, load
//             <= 1/3); a pair probes its home group A, then (if A is full) an independent group B, then
//             A+1, A+2, ...; Step 3's (src,dst)-sorted "edges" array with its
//             multisearch becomes one sector read (a fingerprint hit is verified against E[k]).
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
constexpr uint32_t kErrInternal = 16u;  // a TC_CHECKED build's device bounds check failed (TC_EINTERNAL)
// errors found while counting (they stop the index build); a duplicate (found by the pair-bucket kernel,
// concurrently with the vertex buckets) or an overflow (set by the host) only stop the estimator update
constexpr uint32_t kErrStage = kErrInval | kErrLoop;

// partitioning
#ifndef TC_TILE_EDGES
#define TC_TILE_EDGES 4096
#endif
constexpr uint32_t kTileEdges = TC_TILE_EDGES;  // edges per count/scatter tile
constexpr uint32_t kTileThreads = 512;
#ifndef TC_PART_BITS
#define TC_PART_BITS 11  // 12 measured 5 % slower at C3: k_count's per-warp counters need 128 KB (1 CTA/SM)
#endif
constexpr uint32_t kMaxBucketBits = 15;   // at most 2^15 vertex buckets
constexpr uint32_t kMaxPartBits = TC_PART_BITS;  // the partition kernels: at most 2^11 vertex buckets
constexpr uint32_t kMaxSplitBits = kMaxBucketBits - kMaxPartBits;  // k_split: each into at most 2^4 sub-buckets
constexpr uint32_t kVBucketThreads = 256; // vertex-bucket CTA
constexpr uint32_t kVItems = 24;          // arcs per thread held in registers by the vertex-bucket sort
constexpr uint32_t kVChunk = kVBucketThreads * kVItems;  // 6144 arcs: larger buckets take the chunked path

// device counters (ctr[])
constexpr int kCtrD = 0;       // distinct vertices of W
constexpr int kCtrTicket = 1;  // k_vhub's bucket ticket
constexpr int kCtrBig = 2;     // vertex buckets larger than vcap (k_vhub's)
constexpr int kCtrErr = 3;     // error bits
constexpr int kCtrDefer = 4;   // buckets k_vhub deferred to k_vbig
constexpr int kCtrTicket2 = 5; // k_vbig's bucket ticket
constexpr int kCtrFailB = 6;   // batch index of the first batch that found the error word set (async mode)
constexpr int kCtrArcsBig = 7; // arcs grouped by the large-bucket kernels (k_vhub / k_vbig)
constexpr int kCtrDBig = 8;    // distinct vertices of those buckets
constexpr int kCtrCursor = 9;  // k_small_index: next free segment slot (each bucket CTA takes its range)
constexpr int kCtrQ = 10;      // large batches: Step 3 queries queued by k_update for k_close_q
constexpr int kCtrWords = 16;

// Per-batch values the kernels read from device memory (written by k_desc, the first node of every push), so
// that one captured CUDA graph per batch shape is relaunched unchanged from batch to batch.
// Bounds checks of computed indices (the substitute for compute-sanitizer, which this GPU pool refuses):
// compiled in with -DTC_CHECKED (tests/test_checked_build.py), a violation sets kErrInternal in the error word
// and the push fails with TC_EINTERNAL; compiled out otherwise.
#ifdef TC_CHECKED
#define TC_CHECK(cond, ctr)                                                  \
    do {                                                                     \
        if (!(cond)) atomicOr(const_cast<uint32_t *>(&(ctr)[kCtrErr]), kErrInternal); \
    } while (0)
#else
#define TC_CHECK(cond, ctr) \
    do {                    \
    } while (0)
#endif

struct __align__(32) BatchDesc {
    const uint2 *in;             // the raw batch on this device
    unsigned long long m_prev;   // |E| before the batch
    uint32_t batch;              // index b of this non-empty batch (the Philox counter word)
    uint32_t ptag;               // edge-pair slot tag of this push (1..254)
    uint32_t slot;               // S accumulator slot of this batch
    uint32_t pad;
};

struct __align__(16) VSlot {
    uint32_t key, deg, start, pad;
};

// lowbias32 (a bijection on 32 bits) and its inverse.
__host__ __device__ __forceinline__ uint32_t hash_vertex(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}
__host__ __device__ __forceinline__ uint32_t unhash_vertex(uint32_t x) {
    x ^= x >> 16;
    x *= 0x43021123u;
    x ^= (x >> 15) ^ (x >> 30);
    x *= 0x1d69e2a5u;
    x ^= x >> 16;
    return x;
}

__host__ __device__ __forceinline__ uint64_t hash_pair64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

__host__ __device__ __forceinline__ uint64_t pair_key(uint32_t lo, uint32_t hi) {
    return ((uint64_t)lo << 32) | hi;
}

__host__ __device__ __forceinline__ uint32_t vbucket_of(uint32_t h, uint32_t bv) { return bv ? h >> (32 - bv) : 0u; }
// slot position word (bits 20..51) and 24-bit fingerprint (bits 0..23) of a pair hash; a slot is
// {k, tag << 24 | fingerprint} and is live only when its tag is the batch's (1..254), so the table is
// cleared once per 254 batches, not per batch
__host__ __device__ __forceinline__ uint32_t pslot_word(uint64_t h) { return (uint32_t)(h >> 20); }
__host__ __device__ __forceinline__ uint32_t pfinger(uint64_t h) { return (uint32_t)h & 0xFFFFFFu; }
__host__ __device__ __forceinline__ uint32_t pgroup_start(uint64_t h, uint32_t groups) {
    return (uint32_t)(((uint64_t)pslot_word(h) * groups) >> 32);
}
// Probe sequence of a pair over the G groups: its home group A, a second independent group B, then
// A+1, A+2, ... (a key sits in the first group of its sequence that had room when it was inserted).
__host__ __device__ __forceinline__ uint32_t pgroup_second(uint64_t h, uint32_t groups, uint32_t A) {
    const uint32_t B = (uint32_t)(((uint64_t)hash_vertex((uint32_t)(h >> 32) ^ 0x9E3779B9u) * groups) >> 32);
    return (B != A || groups == 1) ? B : (A + 1 == groups ? 0u : A + 1);
}
__host__ __device__ __forceinline__ uint32_t pgroup_at(uint32_t A, uint32_t B, uint32_t i, uint32_t groups) {
    if (i == 0) return A;
    if (i == 1) return B;
    const uint64_t g = (uint64_t)A + i - 1;
    return (uint32_t)(g % groups);
}

// Vertex-table slices: bucket b (n_b arcs, D_b distinct vertices) owns the S_b = min(next_pow2(2 D_b), 2 n_b)
// slots at offset 2 * (its first arc slot) (load <= 1/2, slices disjoint).  A vertex with hash h probes the
// slot pairs (one 32-byte sector) from vslot_start(h, S) on, wrapping at S (S is even).
__host__ __device__ __forceinline__ uint32_t vslot_start(uint32_t h, uint32_t S) {
    // the bucket is the top bits of h: remix so that the low bits choose the slot
    return (uint32_t)(((uint64_t)(h * 0x9E3779B9u) * S) >> 32) & ~1u;
}
__host__ __device__ __forceinline__ uint32_t vslot_next(uint32_t s, uint32_t S) { return s + 2 >= S ? 0u : s + 2; }

// Small batches: a bit filter over the batch's vertices lets the estimator pass skip
// every estimator the batch cannot change -- a retained f1 with neither endpoint in W gets no chi^+ and no
// closing edge (that edge would touch f1's endpoint x).  The filter has no false negatives, so skipping is
// exact; a false positive only costs the full update.
constexpr uint32_t kFilterBits = 1u << 18;                 // 32 KB
constexpr uint32_t kFilterWords = kFilterBits / 32;
__host__ __device__ __forceinline__ uint32_t vfilter_bit(uint32_t hv) { return hv & (kFilterBits - 1u); }

// Read-only loads of one-shot random probes (the edge-pair table, segS, pslot / apos / E of a fresh f1) with
// an L2 evict-first policy, so that the tables every estimator probes (the vertex table, the pair filter, vslice) stay in L2
// while ~1 GB of probe lines per C3 batch pass through it.  Measured (tools/l2hint.cu): a 48 MB table probed
// alongside random misses into 1 GB stays resident only when the misses are marked evict-first (DRAM bytes per
// probe pair 168 -> 127, time -18 %); marking the hot table evict-last does nothing.
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// EF: the batch is large (kPairFilterMin edges or more) -- below that the whole index stays in L2 and the hint only
// costs hits (C2: k_update 68 vs 63 us with it).  A template parameter, so the other instantiations carry nothing.
template <bool EF>
__device__ __forceinline__ uint4 ldf(const uint4 *p) {
    if (!EF) return __ldg(p);
    uint4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(l2_evict_first()));
    return v;
}
template <bool EF>
__device__ __forceinline__ uint2 ldf(const uint2 *p) {
    if (!EF) return __ldg(p);
    uint2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(l2_evict_first()));
    return v;
}

// Large batches: a blocked Bloom filter over the batch's pairs (16 bits per edge, one 32-bit word per pair with
// four of its bits set), filled by k_count as it normalises the edges (two filters alternate by batch parity:
// k_count zeroes the next batch's while it fills this one's).  The filter is ~w·2 bytes
// (17 MB at w = 2^23), so it stays in L2, whereas the pair table (24 B per edge) does not: Step 3's closing
// probe reads the filter word first and goes to the table only when all four bits are set (every pair of the
// batch; ~0.8 % of the others).  No false negatives, so results are unchanged.  On this part a random read that
// misses L2 costs a whole 128-byte line of DRAM traffic (tools/randbench.cu, profiles/randbench_r02.txt), so
// the filter turns most closing probes from a DRAM line into an L2 hit.
__host__ __device__ __forceinline__ uint32_t pf_words(uint32_t w) { return w < 2 ? 1u : w / 2; }
__host__ __device__ __forceinline__ uint32_t pf_word(uint64_t h, uint32_t nw) {
    return (uint32_t)(((h >> 32) * (uint64_t)nw) >> 32);
}
__host__ __device__ __forceinline__ uint32_t pf_mask(uint64_t h) {
    return (1u << (h & 31u)) | (1u << ((h >> 5) & 31u)) | (1u << ((h >> 10) & 31u)) | (1u << ((h >> 15) & 31u));
}

struct Lookup {
    const uint2 *E;
    const VSlot *vt;
    const uint2 *vslice;   // [BV] {offset, size}
    uint32_t bv;
    const uint2 *pt;       // pair slots {k, tag << 24 | fp}, groups of 4
    uint32_t G;            // pair-table groups
    uint32_t ptag;         // this batch's slot tag
    const uint32_t *pf;    // pair filters (large batches; this batch's at pf + slot * pfs) or null
    uint32_t pfw;          // words of a filter at this batch's size (0: no filter)
    uint32_t pfs;          // stride between the two filters
};

// Large batches: the pair filter and the evict-first probes of the estimator pass, a half-full edge-pair table
constexpr uint32_t kPairFilterMin = 1u << 21;

// Edge-pair table groups (4 slots each) for a batch of w edges: load 1/3, or 1/2 for large batches, whose probes
// mostly stop at the pair filter: at C3 the smaller table (134 MB instead of 201) builds in 219 us instead of 249
// (a compact table of 4-byte slots, 8 per group, was slower: its CAS contention cost more than L2 residency gained)
__host__ __device__ __forceinline__ uint32_t pair_groups(uint32_t w) {
    return (uint32_t)(((uint64_t)w * (w >= kPairFilterMin ? 4u : 6u) + 7) / 8);
}
// groups allocated for batches of up to cap edges
__host__ __device__ __forceinline__ uint32_t pair_groups_alloc(uint32_t cap) {
    const uint32_t a = pair_groups(cap), b = pair_groups(cap < kPairFilterMin ? cap : kPairFilterMin - 1u);
    return a > b ? a : b;
}

// Continue a vertex probe at slot pair b of slice sl (after the first pair missed without an empty slot).
static __device__ __noinline__ uint2 vt_find_from(const Lookup &L, uint2 sl, uint32_t b, uint32_t v) {
    for (uint32_t it = 0; it < sl.y / 2; ++it) {  // every slot pair once (slices are at most half full)
        b = vslot_next(b, sl.y);
        const uint4 *p = reinterpret_cast<const uint4 *>(L.vt + sl.x + b);
        const uint4 s0 = __ldg(p), s1 = __ldg(p + 1);
        if (s0.x == v) return make_uint2(s0.y, s0.z);
        if (s1.x == v) return make_uint2(s1.y, s1.z);
        if (s0.x == kEmptyV || s1.x == kEmptyV) return make_uint2(0u, 0u);
    }
    return make_uint2(0u, 0u);
}

// Pair probe split in two so that its load can be issued together with other probes: pt_issue() reads
// the home group A (one 32-byte sector); pt_resolve() scans it and, only when A is full (rare at load
// 1/3), goes on to B, A+1, ...  Inside a group the filled slots form a prefix, so the first empty slot
// ends the search.  Result: batch position of {lo, hi} (lo < hi), or -1.
struct PairProbe {
    uint32_t lo, hi, fp, A, B, ng;
    const uint2 *sl;
    uint4 a0, a1;  // group A
};

template <bool EF = false>
__device__ __forceinline__ void pt_issue(const Lookup &L, uint32_t lo, uint32_t hi, bool active, PairProbe &P) {
    const uint64_t h = hash_pair64(pair_key(lo, hi));
    const uint32_t ng = active ? L.G : 0u;
    P.lo = lo;
    P.hi = hi;
    P.fp = (L.ptag << 24) | pfinger(h);
    P.ng = ng;
    P.sl = L.pt;  // 32-byte aligned
    P.A = ng ? pgroup_start(h, ng) : 0u;
    P.B = ng ? pgroup_second(h, ng, P.A) : 0u;
    P.a0 = P.a1 = make_uint4(0u, 0u, 0u, 0u);  // tag 0: free
    if (ng) {
        const uint4 *qa = reinterpret_cast<const uint4 *>(P.sl + 4 * P.A);
        P.a0 = ldf<EF>(qa);
        P.a1 = ldf<EF>(qa + 1);
    }
}

// 0: not in the group and the group has room (absent); 1: found (*k set); 2: group full, go on.
template <bool EF = false>
__device__ __forceinline__ int pt_group(const Lookup &L, const PairProbe &P, uint4 q0, uint4 q1, uint32_t *k) {
    const uint32_t ks[4] = {q0.x, q0.z, q1.x, q1.z}, fs[4] = {q0.y, q0.w, q1.y, q1.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if ((fs[i] >> 24) != L.ptag) return 0;  // free slot (stale tag)
        if (fs[i] == P.fp) {
            const uint2 e = ldf<EF>(L.E + ks[i]);
            if (e.x == P.lo && e.y == P.hi) {
                *k = ks[i];
                return 1;
            }
        }
    }
    return 2;
}

template <bool EF = false>
static __device__ __noinline__ int64_t pt_walk(const Lookup &L, PairProbe P) {
    for (uint32_t i = 2; i <= P.ng; ++i) {  // every group once
        const uint4 *q = reinterpret_cast<const uint4 *>(P.sl + 4 * pgroup_at(P.A, P.B, i, P.ng));
        uint32_t k;
        const int r = pt_group<EF>(L, P, ldf<EF>(q), ldf<EF>(q + 1), &k);
        if (r == 0) return -1;
        if (r == 1) return (int64_t)k;
    }
    return -1;
}

template <bool EF = false>
__device__ __forceinline__ int64_t pt_resolve(const Lookup &L, const PairProbe &P) {
    if (P.ng == 0) return -1;
    uint32_t k;
    int r = pt_group<EF>(L, P, P.a0, P.a1, &k);
    if (r == 2) {  // group A full (rare at load 1/3): read B now
        const uint4 *qb = reinterpret_cast<const uint4 *>(P.sl + 4 * P.B);
        r = pt_group<EF>(L, P, ldf<EF>(qb), ldf<EF>(qb + 1), &k);
        if (r == 2) return pt_walk<EF>(L, P);
    }
    if (r == 0) return -1;
    return (int64_t)k;
}

template <bool EF = false>
__device__ __forceinline__ int64_t pt_find(const Lookup &L, uint32_t lo, uint32_t hi) {
    PairProbe P;
    pt_issue<EF>(L, lo, hi, true, P);
    return pt_resolve<EF>(L, P);
}

// pt_find behind the pair filter (when the batch has one): a pair whose four filter bits are not all set is not
// in the batch.
template <bool EF>
__device__ __forceinline__ int64_t pt_find_filtered(const Lookup &L, uint32_t lo, uint32_t hi) {
    if (L.pfw) {
        const uint64_t h = hash_pair64(pair_key(lo, hi));
        const uint32_t m = pf_mask(h);
        if ((__ldg(L.pf + pf_word(h, L.pfw)) & m) != m) return -1;
    }
    return pt_find<EF>(L, lo, hi);
}

// Vertex probe split likewise: first sector (two 16-byte slots) of each of u and v.
struct VertProbe {
    uint2 sl;
    uint32_t b;
    uint4 s0, s1;
};

__device__ __forceinline__ void vt_issue(const Lookup &L, uint32_t v, VertProbe &P) {
    const uint32_t h = hash_vertex(v);
    P.sl = __ldg(L.vslice + vbucket_of(h, L.bv));
    P.b = vslot_start(h, P.sl.y);
    const uint4 *p = reinterpret_cast<const uint4 *>(L.vt + (P.sl.y ? P.sl.x + P.b : 0u));
    P.s0 = __ldg(p);
    P.s1 = __ldg(p + 1);
}

// {deg_W(v), segment start of v}, or {0, 0} when v has no batch arc
__device__ __forceinline__ uint2 vt_resolve(const Lookup &L, const VertProbe &P, uint32_t v) {
    if (P.sl.y == 0) return make_uint2(0u, 0u);
    if (P.s0.x == v) return make_uint2(P.s0.y, P.s0.z);
    if (P.s1.x == v) return make_uint2(P.s1.y, P.s1.z);
    if (P.s0.x == kEmptyV || P.s1.x == kEmptyV) return make_uint2(0u, 0u);
    return vt_find_from(L, P.sl, P.b, v);
}

}  // namespace tcb

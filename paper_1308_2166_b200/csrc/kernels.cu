// kernels.cu -- the per-batch hot path of bulkUpdateAll on sm_100a.
//
// Pipeline for one batch W.  The incidence index is PARTITIONED first (a stable scatter of
// the arcs into vertex-hash buckets) and then built bucket by bucket in shared memory, so the global
// tables are written whole and coalesced, and stay small enough to live in L2 while the estimator pass
// probes them:
//   k_count      a1      : load W (coalesced), validate, normalise into E, stable in-tile ranks of the arcs
//                          by partition bucket (top bits of hash_vertex; one ballot per bit) and per-(bucket,
//                          tile) counts
//   k_scan_cols / k_scan_tot : tile offsets inside each bucket, bucket sizes and starts; the list of
//                          oversized buckets (k_vhub's)
//   k_scatter    a1      : arcs {vertex, k<<1|side, neighbour} to their bucket STABLY (staged in shared
//                          memory, written as coalesced runs), so each bucket holds its arcs in arrival order
//                          -- the F array of rankAll's proof, partitioned
//   k_split      a1      : (w > 2^21 only) each bucket stably split again by the next hash bits
//   k_pairs      a3      : (second stream, alongside the vertex phase) every edge of the raw batch into the
//                          edge-pair table (64-bit CAS; a repeat is TC_EDUP); small batches also fill the
//                          vertex filter
//   k_vhash      a2      : one CTA per vertex bucket: bucket-local vertex ids from a shared-memory hash
//                          table, one stable ranking pass by local id (replaces rankAll's sort by (src, -pos),
//                          PAPER.md:680-684), segment starts -> segS, per-arc {slot, segEnd} (rank = segEnd -
//                          1 - slot, Def. Rank), the bucket's vertex-table slice {deg_W, start}
//   k_vhub / k_vbig a2   : (third stream) oversized buckets: hub peeling + the same hash path; radix sort
//   k_update     a4..a8  : ONE pass over the estimator SoA: Step 1 (level-1 reservoir), Step 2 (chi^+ from
//                          ranks / degrees, level-2 pick by segment arithmetic), Step 3 (closing-edge probe),
//                          block partial sums of chi over closed estimators
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "index.cuh"
#include "kernels.h"
#include "event.h"
#include "philox.cuh"

namespace tcb {

typedef unsigned __int128 u128;
constexpr uint32_t kFull = 0xffffffffu;

__device__ __forceinline__ uint2 norm_edge(uint2 e) { return make_uint2(min(e.x, e.y), max(e.x, e.y)); }

// Lanes of the warp holding the same NB-bit digit d (invalid lanes group together), NB known at compile time.
template <int NB>
__device__ __forceinline__ uint32_t digit_peers_c(uint32_t d, bool valid) {
    uint32_t m = __ballot_sync(kFull, valid);
    if (!valid) m = ~m;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const uint32_t bit = (d >> b) & 1u;
        m &= __ballot_sync(kFull, bit) ^ (bit - 1u);
    }
    return m;
}

// Lanes of the warp holding the same nbits-bit digit d (invalid lanes group together).  nbits is
// warp-uniform.  One ballot per digit bit.
__device__ __forceinline__ uint32_t digit_peers(uint32_t d, bool valid, uint32_t nbits) {
    uint32_t m = __ballot_sync(kFull, valid);
    if (!valid) m = ~m;
#pragma unroll
    for (uint32_t b = 0; b < kMaxPartBits; ++b) {
        if (b < nbits) {
            const uint32_t bit = (d >> b) & 1u;
            m &= __ballot_sync(kFull, bit) ^ (bit - 1u);  // lanes whose bit b equals mine
        }
    }
    return m;
}

// The same with one __match_any_sync (cheaper than ballots for wide digits).
__device__ __forceinline__ uint32_t match_peers(uint32_t d, bool valid) {
    return __match_any_sync(kFull, valid ? d : 0xFFFFFFFFu);
}

// Block-wide exclusive scan of one value per thread (NT threads); returns the prefix, *total the sum.
template <int NT>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t x, uint32_t *sh_warp, uint32_t *total) {
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint32_t incl = x;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, off);
        if (lane >= (uint32_t)off) incl += y;
    }
    if (lane == 31) sh_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t v = lane < NT / 32 ? sh_warp[lane] : 0u;
        uint32_t iv = v;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, iv, off);
            if (lane >= (uint32_t)off) iv += y;
        }
        if (lane < NT / 32) sh_warp[lane] = iv - v;
        if (lane == NT / 32 - 1) sh_warp[NT / 32] = iv;
    }
    __syncthreads();
    const uint32_t r = sh_warp[warp] + incl - x;
    *total = sh_warp[NT / 32];
    __syncthreads();
    return r;
}

// ------------------------------------------------------------------------------------------------
// a1: bucket histograms

struct PartArgs {
    const BatchDesc *d;  // in, ptag, slot (per batch)
    uint32_t *apos2;     // [2 w] partition position of every arc (by arc id k<<1|side)
    Geometry g;
    uint2 *E;
    uint4 *arcs;  // {vertex, k<<1|side, neighbour, 0}
    uint32_t *cntV;    // [tiles][nV] per-(tile, bucket) arc counts
    uint32_t *offV;    // [tiles][nV] the tile's offset inside the bucket
    uint16_t *arank;   // [2 w] in-tile ranks
    uint32_t *vstart;  // bucket sizes (k_scan_cols) -> exclusive prefixes (k_scan_tot)
    uint2 *pt;         // edge-pair table (G groups of 4 slots)
    uint32_t G;
    uint32_t *ctr;
    uint32_t *filt;    // small batches: the vertex filter to fill (else null)
    unsigned long long *S;  // the two S accumulators: k_count zeroes this batch's (d->slot) and the counters
    uint32_t *pf;      // large batches: the two pair filters (k_count fills this batch's, d->slot, and zeroes the other), else null
    uint32_t pfw;      // words of a filter at this batch's size
    uint32_t pfs;      // stride between the two filters
};

// a3: insert edge k = {lo, hi} into the edge-pair table: the first free slot (stale tag) of the first group
// with room along its probe sequence (A, B, A+1, ...), by 64-bit CAS, so the live slots of a group form a
// prefix.  Meeting the
// same pair (confirmed against the raw batch, which is stable while E is being written) returns true.
__device__ __forceinline__ bool pt_insert(const PartArgs &a, const uint2 *in, uint32_t ptag, uint2 n, uint32_t k) {
    const uint64_t h = hash_pair64(pair_key(n.x, n.y));
    const uint32_t tf = (ptag << 24) | pfinger(h);
    const unsigned long long mine = (unsigned long long)k | ((unsigned long long)tf << 32);
    unsigned long long *t64 = reinterpret_cast<unsigned long long *>(a.pt);
    const uint32_t A = pgroup_start(h, a.G), B = pgroup_second(h, a.G, A);
    for (uint32_t step = 0;; ++step) {
        if (step > a.G) {  // every group visited: cannot happen at load <= 1/3 -- an internal error, not a hang
            atomicOr(&a.ctr[kCtrErr], kErrInternal);
            return false;
        }
        const uint32_t g = pgroup_at(A, B, step, a.G);
        TC_CHECK(g < a.G, a.ctr);
        const ulonglong2 *q = reinterpret_cast<const ulonglong2 *>(t64 + 4ull * g);
        const ulonglong2 a0 = __ldcg(q), a1 = __ldcg(q + 1);
        const unsigned long long cur4[4] = {a0.x, a0.y, a1.x, a1.y};
#pragma unroll
        for (uint32_t i = 0; i < 4; ++i) {
            unsigned long long cur = cur4[i];
            if ((uint32_t)(cur >> 56) != ptag) {
                const unsigned long long old = atomicCAS(t64 + 4ull * g + i, cur, mine);
                if (old == cur) return false;
                cur = old;  // taken meanwhile (by this batch)
            }
            if ((uint32_t)(cur >> 32) == tf) {
                const uint2 o = norm_edge(__ldg(in + (uint32_t)cur));
                if (o.x == n.x && o.y == n.y) return true;
            }
        }
    }
}

__global__ void __launch_bounds__(256) k_pairs(PartArgs a) {
    if (a.ctr[kCtrErr] & (kErrStage | kErrDup)) return;  // sticky error of an earlier async batch
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    const uint2 *in = a.d->in;
    const uint32_t ptag = a.d->ptag;
    bool dup = false;
    if (k < a.g.w) {
        const uint2 e = __ldg(in + k);
        if (e.x != kEmptyV && e.y != kEmptyV && e.x != e.y) {  // k_count reports the rest
            const uint2 n = norm_edge(e);
            dup = pt_insert(a, in, ptag, n, k);
            if (a.filt) {
                const uint32_t b0 = vfilter_bit(hash_vertex(n.x)), b1 = vfilter_bit(hash_vertex(n.y));
                atomicOr(a.filt + (b0 >> 5), 1u << (b0 & 31u));
                atomicOr(a.filt + (b1 >> 5), 1u << (b1 & 31u));
            }
        }
    }
    if (__any_sync(kFull, dup) && (threadIdx.x & 31u) == 0) atomicOr(&a.ctr[kCtrErr], kErrDup);
}

// Tile ranking: validate and normalise W, write E, and rank every arc (by vertex bucket) and every edge (by
// pair bucket) inside its tile, stably in arrival order.  Arc a of the tile (a = 2 e + side) is owned by
// warp a / kArcsPerWarp, round (a % kArcsPerWarp) / 32, lane a % 32; edges likewise.  Ranks come from
// ballots and per-warp counters (no shared-memory atomics: they cost 2 cycles per lane on this part).
constexpr uint32_t kTileWarps = kTileThreads / 32;
constexpr uint32_t kArcRounds = 2 * kTileEdges / kTileThreads;   // 16
constexpr uint32_t kEdgeRounds = kTileEdges / kTileThreads;      // 8
constexpr uint32_t kArcsPerWarp = kArcRounds * 32, kEdgesPerWarp = kEdgeRounds * 32;

template <int NB>  // the partition bits a.g.bp1, as a compile-time constant
__global__ void __launch_bounds__(kTileThreads) k_count(PartArgs a) {
    if (blockIdx.x == 0) {  // per-batch resets (every later kernel of the batch starts after this one); this
                            // batch's S slot is k_desc's (zeroed, or carried over in the event mode)
        if (threadIdx.x < (uint32_t)kCtrWords && threadIdx.x != (uint32_t)kCtrErr && threadIdx.x != (uint32_t)kCtrFailB)
            a.ctr[threadIdx.x] = 0u;
    }
    uint32_t *pfill = nullptr;
    if (a.pf) {  // pair filters: this batch's is filled below; the other one (the next batch's) is zeroed here,
                 // its tile's share (the host zeroes a filter itself when no earlier batch did)
        const uint32_t slot = a.d->slot, lo = blockIdx.x * (kTileEdges / 2), hi = min(a.pfw, lo + kTileEdges / 2);
        uint32_t *clr = a.pf + (size_t)(slot ^ 1u) * a.pfs;
        for (uint32_t i = lo + threadIdx.x; i < hi; i += kTileThreads) clr[i] = 0u;
        pfill = a.pf + (size_t)slot * a.pfs;
    }
    if (a.ctr[kCtrErr] & kErrStage) return;  // sticky error of an earlier async batch
    const uint2 *in = a.d->in;
    extern __shared__ uint32_t dsh[];
    constexpr uint32_t nV = 1u << NB;  // == 1 << a.g.bp1 (the launch dispatches on it)
    uint16_t *wv = reinterpret_cast<uint16_t *>(dsh);  // [kTileWarps][nV]
    for (uint32_t i = threadIdx.x; i < kTileWarps * nV / 2; i += kTileThreads) dsh[i] = 0;
    __syncthreads();
    const uint32_t t = blockIdx.x, e0 = t * kTileEdges;
    const uint32_t ne = min(kTileEdges, a.g.w - e0);
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, lt = (1u << lane) - 1u;
    // edges: validate, normalise, E
    uint32_t bad = 0;
#pragma unroll
    for (uint32_t j = 0; j < kEdgeRounds; ++j) {
        const uint32_t i = warp * kEdgesPerWarp + j * 32u + lane;
        if (i < ne) {
            const uint2 e = __ldg(in + e0 + i);
            const uint2 n = norm_edge(e);
            a.E[e0 + i] = n;
            if (e.x == kEmptyV || e.y == kEmptyV) bad |= kErrInval;
            else if (e.x == e.y) bad |= kErrLoop;
            else if (pfill) {  // (filled in k_scatter instead: C3 step +9 us)
                const uint64_t h = hash_pair64(pair_key(n.x, n.y));
                atomicOr(pfill + pf_word(h, a.pfw), pf_mask(h));
            }
        }
    }
    bad = __reduce_or_sync(kFull, bad);
    if (bad && lane == 0) atomicOr(&a.ctr[kCtrErr], bad);
    // arcs: stable rank by vertex bucket (this warp's edges, re-read through L1)
    uint32_t pa[kArcRounds];
#pragma unroll
    for (uint32_t j = 0; j < kArcRounds; ++j) {
        const uint32_t ai = warp * kArcsPerWarp + j * 32u + lane;
        const bool valid = (ai >> 1) < ne;
        uint32_t d = 0;
        if (valid) {
            const uint2 n = norm_edge(__ldg(in + e0 + (ai >> 1)));
            d = vbucket_of(hash_vertex((ai & 1u) ? n.y : n.x), (uint32_t)NB);
        }
        const uint32_t peers = digit_peers_c<NB>(d, valid);
        const uint32_t before = __popc(peers & lt);
        uint32_t c = 0;
        if (valid) c = wv[warp * nV + d];
        __syncwarp();
        if (valid && before == 0) wv[warp * nV + d] = (uint16_t)(c + __popc(peers));
        __syncwarp();
        pa[j] = valid ? (d << 16) | (c + before) : 0xFFFFFFFFu;
    }
    __syncthreads();
    // per bucket: exclusive prefix over warps, tile count
    for (uint32_t d = threadIdx.x; d < nV; d += kTileThreads) {
        uint32_t run = 0;
#pragma unroll
        for (uint32_t x = 0; x < kTileWarps; ++x) {
            const uint32_t c = wv[x * nV + d];
            wv[x * nV + d] = (uint16_t)run;
            run += c;
        }
        a.cntV[(size_t)t * nV + d] = run;  // tile-major: this tile's counts are one contiguous row
    }
    __syncthreads();
    // in-tile ranks (coalesced u16 stores)
#pragma unroll
    for (uint32_t j = 0; j < kArcRounds; ++j) {
        if (pa[j] == 0xFFFFFFFFu) continue;
        const uint32_t ai = warp * kArcsPerWarp + j * 32u + lane;
        const uint32_t d = pa[j] >> 16;
        a.arank[2 * e0 + ai] = (uint16_t)(wv[warp * nV + d] + (pa[j] & 0xFFFFu));
    }
}

// One block: vertex-bucket sizes -> exclusive prefixes (entry nV = 2w); vperm = the vertex buckets with more
// than vcap arcs (processed by k_vbig, concurrently with k_vhash), then the others; ctr[kCtrBig] = how many
// are large.
__global__ void __launch_bounds__(1024) k_scan_tot(uint32_t *vstart, uint32_t nV, uint32_t vcap, uint32_t *vperm,
                                                   uint32_t *ctr) {
    if (ctr[kCtrErr] & kErrStage) return;
    __shared__ uint32_t ws[33];
    const uint32_t i0 = threadIdx.x * 4;  // nV <= 4096: 4 per thread
    uint32_t v[4], s = 0, big = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        v[q] = i0 + q < nV ? vstart[i0 + q] : 0u;
        s += v[q];
        big += (i0 + q < nV && v[q] > vcap) ? 1u : 0u;
    }
    uint32_t nbig;
    uint32_t pb = block_exclusive_scan<1024>(big, ws, &nbig);
    uint32_t ps = nbig + min(i0, nV) - pb;  // small buckets before mine go after all the large ones
    uint32_t tot;
    uint32_t run = block_exclusive_scan<1024>(s, ws, &tot);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (i0 + q < nV) {
            vstart[i0 + q] = run;
            if (v[q] > vcap) vperm[pb++] = i0 + q;
            else vperm[ps++] = i0 + q;
        }
        run += v[q];
    }
    if (threadIdx.x == 0) {
        vstart[nV] = tot;
        ctr[kCtrBig] = nbig;
    }
}


// Tile-major counts cnt[t][b]: one block per 32 buckets (a column strip); warp w sums its slice of tiles for
// each of the 32 columns (coalesced 128-byte rows), a prefix over the 32 warps, then the exclusive prefix
// down each column is written to off[t][b] (the tile's offset inside the bucket) and the column total (the
// bucket size) to vstart[b].
#ifndef TC_SCAN_WARPS
#define TC_SCAN_WARPS 32
#endif
constexpr uint32_t kScanWarps = TC_SCAN_WARPS;
__global__ void __launch_bounds__(kScanWarps * 32) k_scan_cols(const uint32_t *cntV, uint32_t *offV, uint32_t *vstart,
                                                               uint32_t tiles, uint32_t nV, const uint32_t *ctr) {
    if (ctr[kCtrErr] & kErrStage) return;
    __shared__ uint32_t part[kScanWarps][33];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t b = blockIdx.x * 32u + lane;
    const bool on = b < nV;
    const uint32_t per = (tiles + kScanWarps - 1) / kScanWarps, t0 = min(tiles, warp * per), t1 = min(tiles, t0 + per);
    uint32_t sum = 0;
    for (uint32_t t = t0; t < t1; ++t) sum += on ? cntV[(size_t)t * nV + b] : 0u;
    part[warp][lane] = sum;
    __syncthreads();
    uint32_t run = 0;
    for (uint32_t x = 0; x < warp; ++x) run += part[x][lane];
    for (uint32_t t = t0; t < t1; ++t) {
        if (on) {
            const uint32_t c = cntV[(size_t)t * nV + b];
            offV[(size_t)t * nV + b] = run;
            run += c;
        }
    }
    if (warp == kScanWarps - 1 && on) vstart[b] = run;  // the last warp's running sum is the column total
}

// Tile scatter: arc {vertex, k<<1|side, neighbour} -> arcs[start(bucket) + offset(bucket, tile) + rank in
// tile].  Pure streaming: the ranks come from k_count.
// kSmemE: the tile's edges staged in shared memory (12 B of shared memory per tile edge), else read from E through
// L1 (4 B per tile edge: more CTAs per SM).  Measured: staging wins at C2 (20.7 vs 25.0 us), E through L1 at C3
// (174 vs 180 us), so batches of 2^22 edges and more take the second.
constexpr uint32_t kScatterGlobalEMin = 1u << 22;
template <bool kSmemE>
__global__ void __launch_bounds__(kTileThreads) k_scatter(PartArgs a) {
    if (a.ctr[kCtrErr] & kErrStage) return;
    extern __shared__ uint32_t dsh[];
    __shared__ uint32_t ws[kTileThreads / 32 + 1];
    const uint32_t nV = 1u << a.g.bp1;
    uint32_t *soff = dsh, *toff = dsh + nV;                            // [nV] each
    const uint32_t t = blockIdx.x, e0 = t * kTileEdges;
    uint2 *sEs = reinterpret_cast<uint2 *>(dsh + 2 * nV);              // [kTileEdges] the tile's edges (kSmemE)
    const uint2 *sE = kSmemE ? sEs : a.E + e0;
    uint16_t *idx = reinterpret_cast<uint16_t *>(dsh + 2 * nV + (kSmemE ? 2 * kTileEdges : 0));  // arcs in bucket order
    const uint32_t ne = min(kTileEdges, a.g.w - e0);
    for (uint32_t d = threadIdx.x; d < nV; d += kTileThreads) {
        soff[d] = a.vstart[d] + a.offV[(size_t)t * nV + d];
        toff[d] = a.cntV[(size_t)t * nV + d];
    }
    if (kSmemE)
        for (uint32_t i = threadIdx.x; i < ne; i += kTileThreads) sEs[i] = a.E[e0 + i];
    __syncthreads();
    {  // where each bucket's run starts in the tile's bucket order
        const uint32_t per = (nV + kTileThreads - 1) / kTileThreads;
        const uint32_t q0 = min(nV, threadIdx.x * per), q1 = min(nV, q0 + per);
        uint32_t sum = 0;
        for (uint32_t q = q0; q < q1; ++q) sum += toff[q];
        uint32_t tot;
        uint32_t run = block_exclusive_scan<kTileThreads>(sum, ws, &tot);
        for (uint32_t q = q0; q < q1; ++q) {
            const uint32_t c = toff[q];
            toff[q] = run;
            run += c;
        }
    }
    __syncthreads();
    for (uint32_t ai = threadIdx.x; ai < 2 * ne; ai += kTileThreads) {
        const uint2 n = sE[ai >> 1];
        const uint32_t d = vbucket_of(hash_vertex((ai & 1u) ? n.y : n.x), a.g.bp1);
        const uint32_t rk = a.arank[2 * e0 + ai];
        idx[toff[d] + rk] = (uint16_t)ai;
        a.apos2[2u * e0 + ai] = soff[d] + rk;  // the arc's partition position, written in arc order (coalesced)
    }
    __syncthreads();
    // consecutive threads write consecutive positions of the tile's bucket order: a bucket's run coalesces
    for (uint32_t pos = threadIdx.x; pos < 2 * ne; pos += kTileThreads) {
        const uint32_t ai = idx[pos];
        const uint2 n = sE[ai >> 1];
        const uint32_t v = (ai & 1u) ? n.y : n.x, nb = (ai & 1u) ? n.x : n.y;
        const uint32_t d = vbucket_of(hash_vertex(v), a.g.bp1);
        const uint32_t P = soff[d] + (pos - toff[d]);  // the arc's partition position (kept through k_split in .w)
        TC_CHECK(P < 2 * a.g.w, a.ctr);
        __stcs(a.arcs + P, make_uint4(v, 2u * e0 + ai, nb, P));
    }
}

// ------------------------------------------------------------------------------------------------
// a3: pair-table slices

// ------------------------------------------------------------------------------------------------
// a2 at large batches: the partition makes at most 4096 buckets (its per-tile counters and offsets grow
// with buckets x tiles), so for 2w > 4096 x 1024 arcs each bucket is split again, stably, by the next bs
// bits of the vertex hash into 2^bs sub-buckets (one 1024-thread CTA per bucket; ballots per sub-bucket
// value).  The sub-buckets are the vertex buckets of the rest of the batch (bucket id = top bp1 + bs bits).

struct SplitArgs {
    const uint4 *arcs;
    uint4 *arcs2;
    const uint32_t *vstart;  // partition-bucket starts
    uint32_t *vstart2;       // sub-bucket starts
    uint32_t bp1, bs, vcap;
    uint32_t *vperm;         // sub-buckets larger than vcap (k_vhub's list)
    uint32_t *ctr;
};

constexpr int kSplitThreads = 1024;

template <int BS>  // the split bits (1..kMaxSplitBits) as a compile-time constant: BS ballots per arc
__global__ void __launch_bounds__(kSplitThreads) k_split(SplitArgs a) {
    if (a.ctr[kCtrErr] & kErrStage) return;
    constexpr uint32_t NW = kSplitThreads / 32;
    static_assert(NW == 32, "the per-sub-bucket scan over warps is one warp of shuffles");
    // wc: per chunk, each warp's count of every sub-bucket value, then (after the scan) its output offset inside
    // the sub-bucket; two buffers alternate by chunk parity, so a chunk needs two barriers, not four
    __shared__ uint32_t wc[2][NW][1u << BS];
    __shared__ uint32_t tot[1u << BS], soff[1u << BS], run[1u << BS];
    const uint32_t b = blockIdx.x, S = 1u << BS;
    const uint32_t base = a.vstart[b], n = a.vstart[b + 1] - base;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, lt = (1u << lane) - 1u;
    const uint32_t sh = 32 - a.bp1 - BS, smask = S - 1u;
    if (threadIdx.x < S) {
        tot[threadIdx.x] = 0;
        run[threadIdx.x] = 0;
    }
    __syncthreads();
    // pass A: sub-bucket sizes (the lanes of each sub-bucket value found with bs ballots; its first lane adds)
    // the sub-bucket values of this thread's first kCache chunks are kept (BS bits each) for pass B
    constexpr uint32_t kCache = 32 / BS;
    uint32_t sbc = 0;
    for (uint32_t q0 = 0, c = 0; q0 < n; q0 += kSplitThreads, ++c) {
        const uint32_t i = q0 + threadIdx.x;
        const bool valid = i < n;
        const uint32_t sb = valid ? (hash_vertex(a.arcs[base + i].x) >> sh) & smask : 0u;
        if (c < kCache) sbc |= sb << (c * BS);
        const uint32_t peers = digit_peers_c<BS>(sb, valid);
        if (valid && (peers & lt) == 0) atomicAdd(&tot[sb], __popc(peers));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t r = 0;
        for (uint32_t x = 0; x < S; ++x) {
            soff[x] = r;
            a.vstart2[(b << BS) + x] = base + r;
            if (tot[x] > a.vcap) a.vperm[atomicAdd(&a.ctr[kCtrBig], 1u)] = (b << BS) + x;
            r += tot[x];
        }
        if (b == gridDim.x - 1) a.vstart2[gridDim.x << BS] = base + n;
    }
    __syncthreads();
    // pass B: stable ranks chunk by chunk (chunk order, then warp order, then lane order = arrival order)
    uint32_t par = 0;
    for (uint32_t q0 = 0, c = 0; q0 < n; q0 += kSplitThreads, par ^= 1u, ++c) {
        const uint32_t i = q0 + threadIdx.x;
        const bool valid = i < n;
        uint4 x4 = make_uint4(0u, 0u, 0u, 0u);
        if (valid) x4 = a.arcs[base + i];
        const uint32_t sb = !valid ? 0u : c < kCache ? (sbc >> (c * BS)) & smask : (hash_vertex(x4.x) >> sh) & smask;
        const uint32_t peers = digit_peers_c<BS>(sb, valid);  // lanes with my sub-bucket value (bs ballots)
        const uint32_t mine = __popc(peers & lt);
        if (lane < S) wc[par][warp][lane] = 0u;
        __syncwarp();
        if (valid && mine == 0) wc[par][warp][sb] = __popc(peers);
        __syncthreads();
        if (warp < S) {  // warp x scans sub-bucket x over the 32 warps: exclusive prefix + the running offset
            const uint32_t c = wc[par][lane][warp];
            uint32_t inc = c;
#pragma unroll
            for (uint32_t o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, inc, o);
                if (lane >= o) inc += y;
            }
            const uint32_t r0 = run[warp];
            wc[par][lane][warp] = soff[warp] + r0 + inc - c;
            if (lane == 31) run[warp] = r0 + inc;  // only this warp touches run[warp]
        }
        __syncthreads();
        TC_CHECK(!valid || wc[par][warp][sb] + mine < n, a.ctr);
        if (valid) a.arcs2[base + wc[par][warp][sb] + mine] = x4;
    }
}

// ------------------------------------------------------------------------------------------------
// a2: vertex buckets

struct VertArgs {
    uint4 *arcs;        // bucketed arcs {vertex, val, neighbour, 0} (overwritten by the chunked path)
    uint2 *scratch;
    uint4 *scratch4;    // the same memory, as uint4 (k_vhub's rest arcs)
    const uint2 *E;
    const uint32_t *vstart;
    uint2 *segS;        // [2 w] {k<<1|side, neighbour} grouped by vertex
    uint2 *pslot;       // [2 w]: pslot[partition position of an arc] = {its slot in segS, its segment's end}
    const uint32_t *apos2;  // [2 w] partition position by arc id (the radix-sort paths carry arc ids only)
    VSlot *vt;
    uint2 *vslice;
    const uint32_t *vperm;
    uint32_t *vdefer;
    uint32_t bv;
    uint32_t vcap;      // buckets with more arcs go to k_vbig
    uint32_t sortcap;   // k_vbig: buckets with more arcs take the chunked global-memory path
    uint32_t *ctr;
    uint32_t narcs;     // 2 w (TC_CHECKED bounds)
};

constexpr uint32_t kVWarps = kVBucketThreads / 32;
constexpr uint32_t kVAux = kVChunk > kVWarps * 256 + 256 ? kVChunk : kVWarps * 256 + 256;
constexpr uint32_t kVSmemBytes = kVChunk * 8 + kVAux * 4 + kVChunk * 2;  // sbuf | aux | run_start
static_assert(kVChunk * 8 >= 2 * 4 * kVChunk, "the u16 slice table (<= 4 D slots) must fit in sbuf");

// smallest power of two >= x (x >= 1)
__device__ __forceinline__ uint32_t pow2_ceil(uint32_t x) { return x <= 1 ? 1u : 1u << (32 - __clz(x - 1)); }
__device__ __forceinline__ uint32_t log2_ceil(uint32_t x) { return x <= 1 ? 0u : 32 - __clz(x - 1); }

// vertex-table slice of D vertices in a bucket of n arcs (D <= n): load <= 1/2, at most 2 n slots
// (A load-0.6 sizing, min(13 D / 8 + 2, 2 n) -- 64 MB instead of ~120 MB at C3 -- measured slower: k_update
// 383 vs 329 us and k_vhash 351 vs 334 us at C3, the longer probe runs costing more than the L2 hits gained.)
__device__ __forceinline__ uint32_t slice_size(uint32_t D, uint32_t n) { return D ? min(pow2_ceil(2 * D), 2 * n) : 0u; }

// one vertex-table slot {x, deg_W(x), segment start}
__device__ __forceinline__ void vt_put(const VertArgs &a, uint64_t s, uint32_t x, uint32_t deg, uint32_t start) {
    reinterpret_cast<uint4 *>(a.vt)[s] = make_uint4(x, deg, start, 0u);
}

// One LSD pass over the items held in registers (warp-blocked layout, R rounds): stable rank by the digit
// (key >> shift) & ((1 << bits) - 1); returns the destination index of every item in `dst`.
__device__ __forceinline__ void rank_pass(const uint32_t (&key)[kVItems], uint32_t R, uint32_t nvalid_base,
                                          uint32_t n, uint32_t shift, uint32_t bits, uint32_t *whist,
                                          uint32_t *dtot, uint32_t (&dst)[kVItems]) {
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, lt = (1u << lane) - 1u;
    const uint32_t mask = (1u << bits) - 1u;
    for (uint32_t i = threadIdx.x; i < kVWarps * 256; i += kVBucketThreads) whist[i] = 0;
    __syncthreads();
#pragma unroll
    for (uint32_t j = 0; j < kVItems; ++j) {
        if (j < R) {
            const uint32_t i = nvalid_base + warp * 32u * R + j * 32u + lane;
            const bool valid = i < n;
            const uint32_t d = (key[j] >> shift) & mask;
            const uint32_t peers = digit_peers(d, valid, bits);
            const uint32_t before = __popc(peers & lt);
            uint32_t b = 0;
            if (valid) b = whist[warp * 256 + d];
            __syncwarp();
            if (valid && before == 0) whist[warp * 256 + d] = b + __popc(peers);
            __syncwarp();
            dst[j] = valid ? (d << 16) | (b + before) : 0xFFFFFFFFu;
        }
    }
    __syncthreads();
    if (threadIdx.x < 256) {  // per digit: exclusive prefix over warps; digit totals
        uint32_t run = 0;
#pragma unroll
        for (uint32_t x = 0; x < kVWarps; ++x) {
            const uint32_t c = whist[x * 256 + threadIdx.x];
            whist[x * 256 + threadIdx.x] = run;
            run += c;
        }
        dtot[threadIdx.x] = run;
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive scan of the 256 digit totals (8 per lane)
        uint32_t v[8], s = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            v[q] = dtot[threadIdx.x * 8 + q];
            s += v[q];
        }
        uint32_t incl = s;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, incl, off);
            if (lane >= (uint32_t)off) incl += y;
        }
        uint32_t run = incl - s;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            dtot[256 + threadIdx.x * 8 + q] = run;  // digit base
            run += v[q];
        }
    }
    __syncthreads();
#pragma unroll
    for (uint32_t j = 0; j < kVItems; ++j) {
        if (j < R && dst[j] != 0xFFFFFFFFu) {
            const uint32_t d = dst[j] >> 16;
            dst[j] = dtot[256 + d] + whist[warp * 256 + d] + (dst[j] & 0xFFFFu);
        }
    }
}

// Table insert of run r (vertex hash h) into a power-of-two table of u16 run indices, 2-slot aligned
// linear probing (the probe order vt_find assumes).
__device__ __forceinline__ void stable_insert16(uint16_t *table, uint32_t S, uint32_t h, uint32_t r, uint32_t *ctr) {
    uint32_t s = vslot_start(h, S);
    for (uint32_t it = 0; it < S; ++it) {
        if (table[s] == 0xFFFFu && atomicCAS(&table[s], (unsigned short)0xFFFFu, (unsigned short)r) == 0xFFFFu) return;
        if (++s == S) s = 0;
    }
    atomicOr(&ctr[kCtrErr], kErrInternal);  // a full table: an internal error, never a hang
}

// The other endpoint of the edge of arc val = k<<1 | side (side 0 = the lo endpoint).
__device__ __forceinline__ uint32_t arc_neighbour(const uint2 *E, uint32_t val) {
    const uint2 e = E[val >> 1];
    return (val & 1u) ? e.x : e.y;
}

// One large vertex bucket by LSD radix sort on the vertex hash: in shared memory when it holds at most
// sortcap arcs, else chunked through global memory.  Called by the whole CTA.
__device__ __forceinline__ void vbucket_sort(const VertArgs &a, uint32_t b, unsigned char *vsm, uint32_t *dtot,
                                          uint32_t *ws) {
    uint2 *sbuf = reinterpret_cast<uint2 *>(vsm);                    // [kVChunk] {key, val}; later the table
    uint32_t *aux = reinterpret_cast<uint32_t *>(vsm + kVChunk * 8);  // [kVAux]: sort histograms | run keys
    uint16_t *run_start = reinterpret_cast<uint16_t *>(vsm + kVChunk * 8 + kVAux * 4);  // [kVChunk]
    const uint32_t base = a.vstart[b], n = a.vstart[b + 1] - base;
    // the bucket's vertex-table slice: min(next_pow2(2 D), 2 n) slots at offset 2 * base (disjoint slices)
    const uint64_t off = 2ull * base;
    const uint32_t keybits = 32 - a.bv;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint32_t D = 0;

    if (n <= a.sortcap) {
        // ---------------- the whole bucket in registers + shared memory ----------------
        const uint32_t R = (n + kVBucketThreads - 1) / kVBucketThreads;  // rounds (<= kVItems)
        uint32_t key[kVItems], val[kVItems], dst[kVItems];
#pragma unroll
        for (uint32_t j = 0; j < kVItems; ++j) {
            if (j < R) {
                const uint32_t i = warp * 32u * R + j * 32u + lane;
                if (i < n) {
                    const uint4 x = a.arcs[base + i];
                    key[j] = hash_vertex(x.x);
                    val[j] = x.y;
                } else {
                    key[j] = 0;
                    val[j] = 0;
                }
            }
        }
        for (uint32_t shift = 0; shift < keybits; shift += 8) {
            rank_pass(key, R, 0, n, shift, min(8u, keybits - shift), aux, dtot, dst);
#pragma unroll
            for (uint32_t j = 0; j < kVItems; ++j)
                if (j < R && dst[j] != 0xFFFFFFFFu) sbuf[dst[j]] = make_uint2(key[j], val[j]);
            __syncthreads();
            if (shift + 8 < keybits) {
#pragma unroll
                for (uint32_t j = 0; j < kVItems; ++j) {
                    if (j < R) {
                        const uint32_t i = warp * 32u * R + j * 32u + lane;
                        if (i < n) {
                            const uint2 x = sbuf[i];
                            key[j] = x.x;
                            val[j] = x.y;
                        }
                    }
                }
                __syncthreads();
            }
        }
        // runs of equal key (= equal vertex: hash_vertex is a bijection); blocked items per thread
        uint32_t *run_key = aux;  // [D] key of each run (the sort's histograms are dead now)
        const uint32_t i0 = threadIdx.x * R, i1 = min(n, i0 + R);
        uint32_t heads = 0;
        for (uint32_t i = i0; i < i1; ++i) heads += (i == 0 || sbuf[i].x != sbuf[i - 1].x) ? 1u : 0u;
        const uint32_t rid0 = block_exclusive_scan<kVBucketThreads>(heads, ws, &D);  // runs started before i0
        {
            uint32_t q = rid0;
            for (uint32_t i = i0; i < i1; ++i) {
                const uint32_t k = sbuf[i].x;
                if (i == 0 || k != sbuf[i - 1].x) {
                    run_start[q] = (uint16_t)i;
                    run_key[q] = k;
                    ++q;
                }
            }
        }
        __syncthreads();
        // per arc: segS and {slot, segment end}
        uint32_t r = rid0;
        for (uint32_t i = i0; i < i1; ++i) {
            const uint2 x = sbuf[i];
            if (i == 0 || x.x != sbuf[i - 1].x) ++r;
            const uint32_t end = r < D ? run_start[r] : n;  // run r-1 ends where run r starts
            TC_CHECK(base + end <= a.narcs && x.y < a.narcs && a.apos2[x.y] < a.narcs, a.ctr);
            a.segS[base + i] = make_uint2(x.y, arc_neighbour(a.E, x.y));
            a.pslot[a.apos2[x.y]] = make_uint2(base + i, base + end);
        }
        // the slice, built in shared memory and written whole
        if (threadIdx.x == 0) {
            a.vslice[b] = make_uint2((uint32_t)off, slice_size(D, n));
            if (D) atomicAdd(&a.ctr[kCtrD], D);
            if (D) atomicAdd(&a.ctr[kCtrDBig], D);
        }
        __syncthreads();  // sbuf is dead: it holds the table now
        const uint32_t S = slice_size(D, n);
        uint16_t *table = reinterpret_cast<uint16_t *>(sbuf);
        for (uint32_t s = threadIdx.x; s < S; s += kVBucketThreads) table[s] = 0xFFFFu;
        __syncthreads();
        for (uint32_t q = threadIdx.x; q < D; q += kVBucketThreads) stable_insert16(table, S, run_key[q], q, a.ctr);
        __syncthreads();
        for (uint32_t s = threadIdx.x; s < S; s += kVBucketThreads) {
            const uint32_t q = table[s];
            if (q != 0xFFFFu) {
                const uint32_t st = run_start[q], en = q + 1 < D ? run_start[q + 1] : n;
                vt_put(a, off + s, unhash_vertex(run_key[q]), en - st, base + st);
            } else {
                vt_put(a, off + s, kEmptyV, 0u, 0u);
            }
        }
        return;
    }

    // ---------------- chunked path (a bucket larger than vcap, e.g. a hub): global-memory buffers ----------------
    // pass 0 reads the uint4 arcs; then {key, val} ping-pongs between scratch and the bucket's own arc memory
    uint2 *src = reinterpret_cast<uint2 *>(a.arcs) + 2ull * base, *dstb = a.scratch + base;
    const uint4 *arcs4 = a.arcs + base;
    const uint32_t R = kVItems, C = kVChunk;
    uint32_t key[kVItems], val[kVItems], dst[kVItems];
    for (uint32_t shift = 0; shift < keybits; shift += 8) {
        const uint32_t bits = min(8u, keybits - shift), mask = (1u << bits) - 1u;
        const bool first = shift == 0;
        // digit histogram over the whole bucket
        uint32_t *ghist = dtot;  // [256] running digit offsets
        for (uint32_t i = threadIdx.x; i < 256; i += kVBucketThreads) aux[i] = 0;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < n; i += kVBucketThreads) {
            const uint32_t k = first ? hash_vertex(arcs4[i].x) : src[i].x;
            atomicAdd(&aux[(k >> shift) & mask], 1u);
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            uint32_t v[8], s = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                v[q] = aux[threadIdx.x * 8 + q];
                s += v[q];
            }
            uint32_t incl = s;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, incl, off);
                if (lane >= (uint32_t)off) incl += y;
            }
            uint32_t run = incl - s;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                sbuf[threadIdx.x * 8 + q].x = run;  // running offsets live in sbuf[0..256).x
                run += v[q];
            }
        }
        __syncthreads();
        for (uint32_t c0 = 0; c0 < n; c0 += C) {
            const uint32_t cn = min(C, n - c0);
#pragma unroll
            for (uint32_t j = 0; j < kVItems; ++j) {
                const uint32_t i = warp * 32u * R + j * 32u + lane;
                if (i < cn) {
                    if (first) {
                        const uint4 x = arcs4[c0 + i];
                        key[j] = hash_vertex(x.x);
                        val[j] = x.y;
                    } else {
                        const uint2 x = src[c0 + i];
                        key[j] = x.x;
                        val[j] = x.y;
                    }
                } else {
                    key[j] = 0;
                    val[j] = 0;
                }
            }
            rank_pass(key, R, 0, cn, shift, bits, aux + 256, ghist, dst);  // dst = in-chunk digit position
            // in-chunk position = digit base (in chunk) + ...; global = running offset[d] + (pos - chunk base[d])
#pragma unroll
            for (uint32_t j = 0; j < kVItems; ++j) {
                if (dst[j] != 0xFFFFFFFFu) {
                    const uint32_t d = (key[j] >> shift) & mask;
                    const uint32_t p = sbuf[d].x + (dst[j] - ghist[256 + d]);
                    dstb[p] = make_uint2(key[j], val[j]);
                }
            }
            __syncthreads();
            if (threadIdx.x < 256) sbuf[threadIdx.x].x += ghist[threadIdx.x];  // chunk's digit totals
            __syncthreads();
        }
        uint2 *t = src;
        src = dstb;
        dstb = t;
        __syncthreads();
    }
    // sorted {key, val} in src; runs -> run starts in dstb (as u32)
    uint32_t *gruns = reinterpret_cast<uint32_t *>(dstb);
    uint32_t carry = 0;
    for (uint32_t c0 = 0; c0 < n; c0 += C) {
        const uint32_t cn = min(C, n - c0);
        const uint32_t i0 = c0 + threadIdx.x * R, i1 = min(c0 + cn, i0 + R);
        uint32_t heads = 0;
        for (uint32_t i = i0; i < i1; ++i) heads += (i == 0 || src[i].x != src[i - 1].x) ? 1u : 0u;
        uint32_t tot;
        uint32_t rid = carry + block_exclusive_scan<kVBucketThreads>(heads, ws, &tot);
        for (uint32_t i = i0; i < i1; ++i)
            if (i == 0 || src[i].x != src[i - 1].x) gruns[rid++] = i;
        carry += tot;
    }
    D = carry;
    __syncthreads();
    carry = 0;
    for (uint32_t c0 = 0; c0 < n; c0 += C) {
        const uint32_t cn = min(C, n - c0);
        const uint32_t i0 = c0 + threadIdx.x * R, i1 = min(c0 + cn, i0 + R);
        uint32_t heads = 0;
        for (uint32_t i = i0; i < i1; ++i) heads += (i == 0 || src[i].x != src[i - 1].x) ? 1u : 0u;
        uint32_t tot;
        uint32_t r = carry + block_exclusive_scan<kVBucketThreads>(heads, ws, &tot);  // runs started before i0
        for (uint32_t i = i0; i < i1; ++i) {
            const uint2 x = src[i];
            if (i == 0 || x.x != src[i - 1].x) ++r;
            const uint32_t run = r - 1;
            const uint32_t end = run + 1 < D ? gruns[run + 1] : n;
            TC_CHECK(base + end <= a.narcs && x.y < a.narcs && a.apos2[x.y] < a.narcs, a.ctr);
            a.segS[base + i] = make_uint2(x.y, arc_neighbour(a.E, x.y));
            a.pslot[a.apos2[x.y]] = make_uint2(base + i, base + end);
        }
        carry += tot;
    }
    if (threadIdx.x == 0) {
        a.vslice[b] = make_uint2((uint32_t)off, slice_size(D, n));
        if (D) atomicAdd(&a.ctr[kCtrD], D);
        if (D) atomicAdd(&a.ctr[kCtrDBig], D);
    }
    const uint32_t S = slice_size(D, n);
    VSlot *sl = a.vt + off;
    for (uint32_t s = threadIdx.x; s < S; s += kVBucketThreads)
        reinterpret_cast<uint4 *>(sl)[s] = make_uint4(kEmptyV, 0u, 0u, 0u);
    __threadfence();
    __syncthreads();
    const u128 empty = (u128)kEmptyV;
    for (uint32_t q = threadIdx.x; q < D; q += kVBucketThreads) {
        const uint32_t st = gruns[q], en = q + 1 < D ? gruns[q + 1] : n;
        const uint32_t h = src[st].x;
        const u128 v = (u128)unhash_vertex(h) | ((u128)(en - st) << 32) | ((u128)(base + st) << 64);
        uint32_t s = vslot_start(h, S), it = 0;
        while (atomicCAS(reinterpret_cast<u128 *>(sl + s), empty, v) != empty) {
            if (++s == S) s = 0;
            if (++it == S) {
                atomicOr(&a.ctr[kCtrErr], kErrInternal);
                break;
            }
        }
    }
}

// Persistent CTAs over the buckets k_vhub deferred (vdefer[0 .. ctr[kCtrDefer])), after it on its stream.
__global__ void __launch_bounds__(kVBucketThreads, 1) k_vbig(VertArgs a) {
    if (a.ctr[kCtrErr] & kErrStage) return;
    extern __shared__ __align__(16) unsigned char vsm[];
    __shared__ uint32_t dtot[512];
    __shared__ uint32_t ws[33];
    __shared__ uint32_t s_b;
    const uint32_t ndef = a.ctr[kCtrDefer];
    while (true) {
        if (threadIdx.x == 0) {
            const uint32_t t = atomicAdd(&a.ctr[kCtrTicket2], 1u);
            s_b = t < ndef ? a.vdefer[t] : 0xFFFFFFFFu;
        }
        __syncthreads();
        const uint32_t b = s_b;
        __syncthreads();
        if (b == 0xFFFFFFFFu) return;
        vbucket_sort(a, b, vsm, dtot, ws);
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------------------
// a2, common case: a vertex bucket of at most vcap (<= kHCapSmall) arcs.  Vertices get bucket-local ids from a
// shared-memory hash table (claim order), then ONE stable ranking pass by local id (__match_any_sync peers,
// per-warp counters) -- instead of three radix passes on the vertex hash -- gives every arc its rank inside
// its vertex.

constexpr uint32_t kHThreads = 256;

constexpr int kHubThreadsC = 1024;  // k_vhub's CTA size (the hash path counts its vertices apart)

// Shared-memory layout of the hash path for buckets of at most CAP arcs: R1 = {hkey u32[2 CAP], lid
// u16[2 CAP]} while hashing; then {whist u16[8][SW], segst u32[CAP + 1]}; the slice table (u32,
// <= 2 CAP slots) reuses whist; vkey u32[CAP] apart.
template <uint32_t CAP, int NT = kHThreads>
struct HL {
    static constexpr uint32_t T = 2 * CAP;
    static constexpr uint32_t SW = CAP < 2048 ? CAP : 2048;
    static constexpr uint32_t WH = (NT / 32) * SW * 2;
    static constexpr uint32_t TBL = 4 * 2 * CAP;
    static constexpr uint32_t SEGOFF = WH > TBL ? WH : TBL;
    static constexpr uint32_t R1A = T * 6, R1B = SEGOFF + (CAP + 1) * 4;
    static constexpr uint32_t R1 = (R1A > R1B ? R1A : R1B) + 64;
    static constexpr uint32_t BYTES = R1 + CAP * 4;
};

// Arcs of a bucket as the hash path reads them: straight from the bucketed arcs, or (after a hub vertex
// was peeled off) from a shared-memory list of the remaining arcs.
struct ArcSrc {
    const uint4 *g;                    // global {vertex, val, neighbour, partition position} (g != nullptr), else:
    const uint32_t *sv, *sval, *snb;   // shared-memory lists
    __device__ __forceinline__ uint32_t v(uint32_t i) const { return g ? g[i].x : sv[i]; }
    __device__ __forceinline__ uint2 vv(uint32_t i) const {
        if (g) {
            const uint4 x = g[i];
            return make_uint2(x.x, x.y);
        }
        return make_uint2(sv[i], sval[i]);
    }
    // {vertex, val, neighbour, partition position (pslot index)}: the position is carried in .w by the
    // partitioned build; the shared-memory lists belong to k_small_index, where it is the arc id itself
    __device__ __forceinline__ uint4 all(uint32_t i) const {
        if (g) return g[i];
        return make_uint4(sv[i], sval[i], snb[i], sval[i]);
    }
};

// Hash-path grouping of n arcs (src) of bucket b whose segments start at slot base + off0; `hub` (if
// hubn > 0) is an extra vertex whose segment [base, base + hubn) was already written.
template <int R, uint32_t CAP, int NT = kHThreads>
__device__ __forceinline__ void vbucket_hash(const VertArgs &a, uint32_t b, uint32_t base, const ArcSrc &src, uint32_t n,
                                             uint32_t off0, uint32_t hub, uint32_t hubn, unsigned char *sm,
                                             uint32_t *ws, uint32_t *sD) {
    using L = HL<CAP, NT>;
    constexpr uint32_t NW = NT / 32;
    static_assert((uint32_t)R * NT <= CAP, "items per thread exceed the layout");
    uint32_t *hkey = reinterpret_cast<uint32_t *>(sm);
    uint16_t *lid = reinterpret_cast<uint16_t *>(sm + L::T * 4);
    uint16_t *whist = reinterpret_cast<uint16_t *>(sm);
    uint32_t *segst = reinterpret_cast<uint32_t *>(sm + L::SEGOFF);
    uint32_t *table = reinterpret_cast<uint32_t *>(sm);
    uint32_t *vkey = reinterpret_cast<uint32_t *>(sm + L::R1);
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, lt = (1u << lane) - 1u;
    const uint32_t Tb = pow2_ceil(2 * max(n, 1u));
    for (uint32_t s = threadIdx.x; s < Tb; s += NT) hkey[s] = kEmptyV;
    if (threadIdx.x == 0) *sD = 0;
    __syncthreads();
    // phase 1: local ids (claim order) through the shared hash table; warp w owns items [w 32 R, (w+1) 32 R)
    uint32_t val[R], pk[R], nbv[R];
    uint32_t prw[R];  // the arc's partition position, kept from the one read of the arc
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const uint32_t i = warp * 32u * R + j * 32u + lane;
        pk[j] = 0xFFFFFFFFu;
        if (i < n) {
            const uint4 x = src.all(i);
            prw[j] = x.w;
            val[j] = x.y;
            nbv[j] = x.z;
            uint32_t s = hash_vertex(x.x) & (Tb - 1);
            for (uint32_t it = 0;; ++it) {
                if (it == Tb) {  // a full table: an internal error, never a hang
                    atomicOr(&a.ctr[kCtrErr], kErrInternal);
                    break;
                }
                uint32_t k = hkey[s];
                if (k == kEmptyV) {
                    k = atomicCAS(&hkey[s], kEmptyV, x.x);
                    if (k == kEmptyV) {
                        const uint32_t l = atomicAdd(sD, 1u);
                        lid[s] = (uint16_t)l;
                        vkey[l] = x.x;
                        break;
                    }
                }
                if (k == x.x) break;
                s = (s + 1) & (Tb - 1);
            }
            pk[j] = s;
        }
    }
    __syncthreads();
    const uint32_t D = *sD;
#pragma unroll
    for (int j = 0; j < R; ++j)
        if (pk[j] != 0xFFFFFFFFu) pk[j] = (uint32_t)lid[pk[j]] << 16;  // local id << 16 | rank (below)
    __syncthreads();  // R1 becomes whist + segst
    // phase 2: stable rank of each arc inside its vertex, local ids in sweeps of kHSweep
    for (uint32_t l0 = 0; l0 < D; l0 += L::SW) {
        const uint32_t nd = min(L::SW, D - l0);
        const uint32_t bits = log2_ceil(nd);
        for (uint32_t i = threadIdx.x; i < NW * nd; i += NT) whist[i] = 0;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const uint32_t d = (pk[j] >> 16) - l0;
            const bool in = pk[j] != 0xFFFFFFFFu && d < nd;
            const uint32_t peers = match_peers(d, in);
            const uint32_t before = __popc(peers & lt);
            uint32_t c = 0;
            if (in) c = whist[warp * nd + d];
            __syncwarp();
            if (in && before == 0) whist[warp * nd + d] = (uint16_t)(c + __popc(peers));
            __syncwarp();
            if (in) pk[j] += c + before;
        }
        __syncthreads();
        for (uint32_t d = threadIdx.x; d < nd; d += NT) {  // exclusive prefix over warps; degree
            uint32_t run = 0;
#pragma unroll
            for (uint32_t x = 0; x < NW; ++x) {
                const uint32_t c = whist[x * nd + d];
                whist[x * nd + d] = (uint16_t)run;
                run += c;
            }
            segst[l0 + d] = run;
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const uint32_t d = (pk[j] >> 16) - l0;
            if (pk[j] != 0xFFFFFFFFu && d < nd) pk[j] += whist[warp * nd + d];
        }
        __syncthreads();
    }
    // phase 3: segment starts = exclusive scan of the degrees over local ids
    {
        const uint32_t per = (D + NT - 1) / NT;
        const uint32_t q0 = min(D, threadIdx.x * per), q1 = min(D, q0 + per);
        uint32_t sum = 0;
        for (uint32_t q = q0; q < q1; ++q) sum += segst[q];
        uint32_t tot;
        uint32_t run = block_exclusive_scan<NT>(sum, ws, &tot);
        for (uint32_t q = q0; q < q1; ++q) {
            const uint32_t c = segst[q];
            segst[q] = run;
            run += c;
        }
        if (threadIdx.x == 0) segst[D] = n;
        __syncthreads();
    }
    // phase 4: per arc, segS and {slot, segment end}
    const uint32_t b0 = base + off0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
        if (pk[j] == 0xFFFFFFFFu) continue;
        const uint32_t l = pk[j] >> 16;
        const uint32_t pos = segst[l] + (pk[j] & 0xFFFFu);
        TC_CHECK(pos < n && b0 + segst[l + 1] <= a.narcs && val[j] < a.narcs, a.ctr);
        a.segS[b0 + pos] = make_uint2(val[j], nbv[j]);
        // by the arc's partition position: this bucket's own range, so the writes fill whole sectors in L2
        const uint32_t pre = prw[j];
        TC_CHECK(pre < a.narcs, a.ctr);
        a.pslot[pre] = make_uint2(b0 + pos, b0 + segst[l + 1]);
    }
    // phase 5: the vertex-table slice, built in shared memory (over whist) and written whole; the hub (if
    // any) is entry D
    const uint32_t Dt = D + (hubn ? 1u : 0u);
    const uint32_t S = slice_size(Dt, off0 + n);
    const uint64_t off = 2ull * base;
    if (threadIdx.x == 0) {
        a.vslice[b] = make_uint2((uint32_t)off, S);
        if (Dt) atomicAdd(&a.ctr[kCtrD], Dt);
        if (Dt && NT == kHubThreadsC) atomicAdd(&a.ctr[kCtrDBig], Dt);
    }
    for (uint32_t s = threadIdx.x; s < S; s += NT) table[s] = kEmptyV;
    __syncthreads();
    for (uint32_t l = threadIdx.x; l < Dt; l += NT) {
        uint32_t s = vslot_start(hash_vertex(l < D ? vkey[l] : hub), S), it = 0;
        while (atomicCAS(&table[s], kEmptyV, l) != kEmptyV) {
            if (++s == S) s = 0;
            if (++it == S) {
                atomicOr(&a.ctr[kCtrErr], kErrInternal);
                break;
            }
        }
    }
    __syncthreads();
    for (uint32_t s = threadIdx.x; s < S; s += NT) {
        const uint32_t l = table[s];
        if (l < D) vt_put(a, off + s, vkey[l], segst[l + 1] - segst[l], b0 + segst[l]);
        else if (l == D) vt_put(a, off + s, hub, hubn, base);
        else vt_put(a, off + s, kEmptyV, 0u, 0u);
    }
}

template <uint32_t CAP, int NT, typename F>
__device__ __forceinline__ void hash_dispatch(uint32_t n, F f) {
    constexpr int RMAX = (int)(CAP / NT);  // 8 or 16
    if (n <= 1u * NT) f(std::integral_constant<int, 1>());
    else if (n <= 2u * NT) f(std::integral_constant<int, 2>());
    else if (n <= 4u * NT) f(std::integral_constant<int, 4>());
    else if (RMAX <= 8 || n <= 8u * NT) f(std::integral_constant<int, (RMAX >= 8 ? 8 : 4)>());
    else f(std::integral_constant<int, (RMAX >= 16 ? 16 : 8)>());
}

// Common buckets (<= vcap <= kHCapSmall arcs): 4 CTAs per SM.
constexpr uint32_t kHCapSmall = 2048;
constexpr uint32_t kVHashSmemBytes = HL<kHCapSmall>::BYTES;

__global__ void __launch_bounds__(kHThreads, 4) k_vhash(VertArgs a) {
    if (a.ctr[kCtrErr] & kErrStage) return;
    extern __shared__ __align__(16) unsigned char hsm[];
    __shared__ uint32_t ws[9];
    __shared__ uint32_t sD;
    const uint32_t b = blockIdx.x;
    const uint32_t base = a.vstart[b], n = a.vstart[b + 1] - base;
    if (n > a.vcap) return;  // k_vhub's
    const ArcSrc src{a.arcs + base, nullptr, nullptr, nullptr};
    hash_dispatch<kHCapSmall, kHThreads>(n, [&](auto r) {
        vbucket_hash<decltype(r)::value, kHCapSmall, kHThreads>(a, b, base, src, n, 0u, 0u, 0u, hsm, ws, &sD);
    });
}

// Large buckets (more than vcap arcs; at batch sizes of 2^22 and beyond, most buckets): 512-thread CTAs with
// the hash path for up to kHubCap arcs.  A bucket larger than that is almost always one hub vertex plus
// about a normal bucket's worth of others: the most frequent vertex of a sample is peeled off (its arcs are
// one segment, already in arrival order: a 1-bit stable partition) and the rest, copied to the scratch
// buffer, goes through the hash path.  Buckets whose rest is still too large are deferred to k_vbig.
// Persistent CTAs (one per SM) over vperm[0 .. ctr[kCtrBig]).
constexpr int kHubThreads = kHubThreadsC;
constexpr uint32_t kHubWarps = kHubThreads / 32;
constexpr uint32_t kHubCap = 8192;
constexpr uint32_t kHubSample = kHubThreads;
constexpr uint32_t kVHubSmemBytes = HL<kHubCap, kHubThreads>::BYTES;

__global__ void __launch_bounds__(kHubThreads, 1) k_vhub(VertArgs a) {
    if (a.ctr[kCtrErr] & kErrStage) return;
    extern __shared__ __align__(16) unsigned char hsm[];
    __shared__ uint32_t ws[kHubWarps + 1];
    __shared__ uint32_t sD, s_b, s_h, s_cnt;
    __shared__ uint32_t skey[2 * kHubSample], scnt[2 * kHubSample];
    __shared__ uint32_t wtot[2][kHubWarps];
    __shared__ unsigned long long wbest[kHubWarps];
    const uint32_t nbig = a.ctr[kCtrBig];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, lt = (1u << lane) - 1u;
    while (true) {
        if (threadIdx.x == 0) {
            const uint32_t t = atomicAdd(&a.ctr[kCtrTicket], 1u);
            s_b = t < nbig ? a.vperm[t] : 0xFFFFFFFFu;
        }
        __syncthreads();
        const uint32_t b = s_b;
        if (b == 0xFFFFFFFFu) return;
        const uint32_t base = a.vstart[b], n = a.vstart[b + 1] - base;
        const uint4 *arcs = a.arcs + base;
        if (threadIdx.x == 0) atomicAdd(&a.ctr[kCtrArcsBig], n);
        if (n <= kHubCap) {  // no peeling needed
            const ArcSrc src{arcs, nullptr, nullptr, nullptr};
            hash_dispatch<kHubCap, kHubThreads>(n, [&](auto r) {
                vbucket_hash<decltype(r)::value, kHubCap, kHubThreads>(a, b, base, src, n, 0u, 0u, 0u, hsm, ws, &sD);
            });
            __syncthreads();
            continue;
        }
        // 1. candidate hub = the most frequent vertex of kHubSample evenly spaced arcs
        for (uint32_t s = threadIdx.x; s < 2 * kHubSample; s += kHubThreads) {
            skey[s] = kEmptyV;
            scnt[s] = 0;
        }
        if (threadIdx.x == 0) s_cnt = 0;
        __syncthreads();
        {
            const uint32_t v = arcs[(uint32_t)(((uint64_t)threadIdx.x * n) / kHubSample)].x;
            uint32_t s = hash_vertex(v) & (2 * kHubSample - 1);
            for (uint32_t it = 0; it < 2 * kHubSample; ++it) {  // 1024 samples in 2048 slots: always room
                const uint32_t k = atomicCAS(&skey[s], kEmptyV, v);
                if (k == kEmptyV || k == v) break;
                s = (s + 1) & (2 * kHubSample - 1);
            }
            atomicAdd(&scnt[s], 1u);
        }
        __syncthreads();
        {
            uint32_t best = 0, bs = 0;
            for (uint32_t t2 = threadIdx.x; t2 < 2 * kHubSample; t2 += kHubThreads)
                if (scnt[t2] > best) {
                    best = scnt[t2];
                    bs = t2;
                }
            unsigned long long pkd = ((unsigned long long)best << 32) | bs;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long y = __shfl_xor_sync(kFull, pkd, o);
                pkd = y > pkd ? y : pkd;
            }
            if (lane == 0) wbest[warp] = pkd;
            __syncthreads();
            if (threadIdx.x == 0) {
                unsigned long long m = wbest[0];
                for (uint32_t x = 1; x < kHubWarps; ++x) m = wbest[x] > m ? wbest[x] : m;
                s_h = skey[(uint32_t)m];
            }
            __syncthreads();
        }
        const uint32_t h = s_h;
        // 2. hub arcs H; the rest must fit the hash path (with the hub, D + 1 <= kHubCap vertices)
        uint32_t mine = 0;
        for (uint32_t i = threadIdx.x; i < n; i += kHubThreads) mine += arcs[i].x == h ? 1u : 0u;
        mine = __reduce_add_sync(kFull, mine);
        if (lane == 0) atomicAdd(&s_cnt, mine);
        __syncthreads();
        const uint32_t H = s_cnt;
        if (n - H > kHubCap - 1) {  // not one hub: the radix-sort kernel takes it
            if (threadIdx.x == 0) a.vdefer[atomicAdd(&a.ctr[kCtrDefer], 1u)] = b;
            __syncthreads();
            continue;
        }
        // 3. stable 1-bit partition: hub arcs -> segment [base, base + H); the rest -> scratch[base ..)
        uint4 *rest = a.scratch4 + base;
        uint32_t hubrun = 0, restrun = 0;
        for (uint32_t q0 = 0; q0 < n; q0 += kHubThreads) {
            const uint32_t i = q0 + threadIdx.x;
            uint4 x = make_uint4(0u, 0u, 0u, 0u);
            if (i < n) x = arcs[i];
            const bool valid = i < n, isH = valid && x.x == h;
            const uint32_t bh = __ballot_sync(kFull, isH), br = __ballot_sync(kFull, valid && !isH);
            if (lane == 0) {
                wtot[0][warp] = __popc(bh);
                wtot[1][warp] = __popc(br);
            }
            __syncthreads();
            uint32_t ph = hubrun, pr = restrun, th = 0, tr = 0;
#pragma unroll
            for (uint32_t w2 = 0; w2 < kHubWarps; ++w2) {
                if (w2 < warp) {
                    ph += wtot[0][w2];
                    pr += wtot[1][w2];
                }
                th += wtot[0][w2];
                tr += wtot[1][w2];
            }
            if (isH) {
                const uint32_t pos = ph + __popc(bh & lt);
                TC_CHECK(pos < H && base + H <= a.narcs && x.w < a.narcs, a.ctr);
                a.segS[base + pos] = make_uint2(x.y, x.z);
                a.pslot[x.w] = make_uint2(base + pos, base + H);
            } else if (valid) {
                rest[pr + __popc(br & lt)] = x;
            }
            hubrun += th;
            restrun += tr;
            __syncthreads();
        }
        __threadfence_block();
        __syncthreads();
        // 4. the rest through the hash path (segments after the hub's), the hub as an extra vertex
        const ArcSrc src{rest, nullptr, nullptr, nullptr};
        hash_dispatch<kHubCap, kHubThreads>(n - H, [&](auto r) {
            vbucket_hash<decltype(r)::value, kHubCap, kHubThreads>(a, b, base, src, n - H, H, h, H, hsm, ws, &sD);
        });
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------------------
// a1..a3 for small batches (w <= kSmallIndexMax): ONE kernel instead of the partitioned build's eight launches,
// whose fixed latency dominates small batches.  CTA b of 2^bv: validates the whole batch (it is small), writes
// E / apos / the edge-pair table for its slice of the edges, compacts the arcs of vertex bucket b in arrival
// order into shared memory (a block-wide stable prefix), takes its segment range with one atomic, and groups
// them through the hash path.  Same tables and lookups as the partitioned build (a bucket's partition position
// of an arc is its arc id here).  The per-batch counter resets are done by k_desc, ahead of every CTA.
// Two instances: <256 threads, 4096-arc buckets> up to w = 2048, <512, 8192> up to w = 4096 (a bucket may hold
// every arc of the batch).  2w / 64 CTAs (Tuning::small_index_arcs; measured 16..512 arcs per CTA): at w = 4096
// 128 CTAs take 20.0 us vs 25.2 for the 16 CTAs of ~512 arcs (256 CTAs: 29.2), at w = 2048 16.8 vs 22.9 us --
// the kernel is a chain of dependent phases, and a CTA with fewer arcs finishes its hash path sooner.
template <int kSmallThreads, uint32_t kSmallCap>
struct SmallIndexCfg {
    static constexpr uint32_t kHashBytes = HL<kSmallCap, kSmallThreads>::BYTES;
    static constexpr uint32_t kSmemBytes = kHashBytes + 3 * kSmallCap * 4;
};

template <int kSmallThreads, uint32_t kSmallCap>
__global__ void __launch_bounds__(kSmallThreads) k_small_index(PartArgs a, VertArgs v) {
    constexpr uint32_t kSmallHashBytes = SmallIndexCfg<kSmallThreads, kSmallCap>::kHashBytes;
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t *sv = reinterpret_cast<uint32_t *>(smem + kSmallHashBytes), *sval = sv + kSmallCap, *snb = sval + kSmallCap;
    __shared__ uint32_t ws[kSmallThreads / 32 + 1];
    __shared__ uint32_t sD, s_base, s_cnt;
    if (a.ctr[kCtrErr] & kErrStage) return;  // sticky error of an earlier asynchronous batch
    const uint2 *in = a.d->in;
    const uint32_t ptag = a.d->ptag, w = a.g.w, b = blockIdx.x, bv = a.g.bv, NB = gridDim.x;
    const uint32_t lane = threadIdx.x & 31u;
    // one coalesced pass over the batch (every CTA, the batch is small): validation -- a rejected batch must not
    // insert anything -- and the vertex bucket of every arc into shared memory (the hash path's region, free
    // until the grouping), so that the compaction below scans shared memory instead of the batch twice
    uint16_t *sbk = reinterpret_cast<uint16_t *>(smem);
    static_assert(2 * kSmallCap * 2 <= kSmallHashBytes, "arc bucket ids must fit the hash region");
    uint32_t bad = 0;
    for (uint32_t k = threadIdx.x; k < w; k += kSmallThreads) {
        const uint2 e = __ldg(in + k);
        if (e.x == kEmptyV || e.y == kEmptyV) bad |= kErrInval;
        else if (e.x == e.y) bad |= kErrLoop;
        const uint2 n = norm_edge(e);
        sbk[2 * k] = (uint16_t)vbucket_of(hash_vertex(n.x), bv);
        sbk[2 * k + 1] = (uint16_t)vbucket_of(hash_vertex(n.y), bv);
    }
    bad = __reduce_or_sync(kFull, bad);
    if (bad && lane == 0) atomicOr(&a.ctr[kCtrErr], bad);
    if (__syncthreads_or(bad != 0)) return;
    // this CTA's slice of the edges: E, partition positions (= arc ids), pair table, small-batch filter
    bool dup = false;
    for (uint32_t k = (uint32_t)((uint64_t)b * w / NB) + threadIdx.x, k1 = (uint32_t)((uint64_t)(b + 1) * w / NB);
         k < k1; k += kSmallThreads) {
        const uint2 n = norm_edge(__ldg(in + k));
        a.E[k] = n;
        a.apos2[2 * k] = 2 * k;
        a.apos2[2 * k + 1] = 2 * k + 1;
        dup |= pt_insert(a, in, ptag, n, k);
        if (a.filt) {
            const uint32_t b0 = vfilter_bit(hash_vertex(n.x)), b1 = vfilter_bit(hash_vertex(n.y));
            atomicOr(a.filt + (b0 >> 5), 1u << (b0 & 31u));
            atomicOr(a.filt + (b1 >> 5), 1u << (b1 & 31u));
        }
    }
    if (__any_sync(kFull, dup) && lane == 0) atomicOr(&a.ctr[kCtrErr], kErrDup);
    // bucket b's arcs in arrival order (arc a = 2k + side), compacted stably: warp w owns the contiguous arcs
    // [w C, (w+1) C); it counts its matches with ballots, one block scan turns the counts into offsets, and a
    // second sweep (the batch is in L1/L2 by now) writes them
    constexpr uint32_t NWS = kSmallThreads / 32;
    const uint32_t warp = threadIdx.x >> 5, C = (2 * w + NWS - 1) / NWS;
    const uint32_t c0 = min(2 * w, warp * C), c1 = min(2 * w, c0 + C);
    uint32_t cnt = 0;
    for (uint32_t ai0 = c0; ai0 < c1; ai0 += 32) {
        const uint32_t ai = ai0 + lane;
        cnt += __popc(__ballot_sync(kFull, ai < c1 && sbk[ai] == b));
    }
    uint32_t tot;
    const uint32_t wpre = block_exclusive_scan<kSmallThreads>(lane == 0 ? cnt : 0u, ws, &tot);
    const uint32_t woff = __shfl_sync(kFull, wpre, 0);
    uint32_t run = 0;
    for (uint32_t ai0 = c0; ai0 < c1; ai0 += 32) {
        const uint32_t ai = ai0 + lane;
        const bool mine = ai < c1 && sbk[ai] == b;
        const uint32_t m = __ballot_sync(kFull, mine);
        if (mine) {
            const uint2 ne = norm_edge(__ldg(in + (ai >> 1)));
            const uint32_t vx = (ai & 1u) ? ne.y : ne.x, nb = (ai & 1u) ? ne.x : ne.y;
            const uint32_t q = woff + run + __popc(m & ((1u << lane) - 1u));
            sv[q] = vx;
            sval[q] = ai;
            snb[q] = nb;
        }
        run += __popc(m);
    }
    if (threadIdx.x == 0) s_cnt = tot;
    __syncthreads();
    const uint32_t n = s_cnt;
    if (threadIdx.x == 0) s_base = atomicAdd(&a.ctr[kCtrCursor], n);  // segments: any bucket order will do
    __syncthreads();
    const uint32_t base = s_base;
    TC_CHECK(n <= kSmallCap && base + n <= 2 * w, a.ctr);
    const ArcSrc src{nullptr, sv, sval, snb};
    hash_dispatch<kSmallCap, kSmallThreads>(n, [&](auto r) {
        vbucket_hash<decltype(r)::value, kSmallCap, kSmallThreads>(v, b, base, src, n, 0u, 0u, 0u, smem, ws, &sD);
    });
}

// ------------------------------------------------------------------------------------------------
// a4..a8: the fused estimator update, one thread per estimator.

struct UpdateIdx {
    Lookup L;
    const uint2 *apos;   // [w] partition positions of edge k's two arcs
    const uint2 *pslot;  // [2 w] by partition position: {slot in segS, segment end}
    const uint2 *segS;
    uint32_t *ctr;
};

struct EstState {
    uint2 r1, r2;
    uint32_t cf, p1, p2;
};

struct UpdateArgs {
    uint2 *r1s, *r2s;
    uint32_t *cfs, *p1s, *p2s;
    uint64_t count, first, seed;
    uint32_t batch, w;          // batch: filled from the descriptor at kernel entry (with_desc)
    uint64_t m_prev;            // likewise
    const BatchDesc *d;
};

// The per-batch values of the descriptor into the kernel's own copies of its arguments.
__device__ __forceinline__ void with_desc(UpdateArgs &u, Lookup &L) {
    u.batch = u.d->batch;
    u.m_prev = u.d->m_prev;
    L.ptag = u.d->ptag;
    if (L.pf) L.pf += (size_t)u.d->slot * L.pfs;  // this batch's pair filter
}

template <bool kSmall>
__device__ __forceinline__ EstState load_state(const UpdateArgs &u, uint64_t t) {
    EstState e;
    e.r1 = __ldcs(u.r1s + t);
    e.cf = __ldcs(u.cfs + t);
    e.r2 = __ldcs(u.r2s + t);
    if (!kSmall) {  // the small-batch pass writes p1 / p2 only when it replaces them: it never reads them
        e.p1 = __ldcs(u.p1s + t);
        e.p2 = __ldcs(u.p2s + t);
    } else {
        e.p1 = e.p2 = 0u;
    }
    return e;
}

__device__ __forceinline__ bool filter_has(const uint32_t *f, uint32_t bit) { return (f[bit >> 5] >> (bit & 31u)) & 1u; }

// Steps 1-3 for estimator t (local index) whose state was read into `old`.  Returns chi if it ends closed.
// Written straight-line: the loads of the fresh-f1 and retained-f1 paths are predicated, not branched, so
// a warp with both kinds of lanes waits for one round trip, not two.
// Step 1's draw for estimator t: the Philox block of (global id, batch) (reading R7) and the level-1 decision.
struct Step1 {
    uint64_t d1, xhi;  // randInt(|E| + |W|) and the word of Step 2's draw
    bool fresh;
};

__device__ __forceinline__ Step1 step1_draw(const UpdateArgs &u, uint64_t t) {
    const uint64_t gid = u.first + t;
    const DrawCtx dc{gid, u.batch, PhiloxKey{(uint32_t)u.seed, (uint32_t)(u.seed >> 32)}};
    const uint4 o = philox4x32_10(make_uint4((uint32_t)gid, (uint32_t)(gid >> 32), u.batch, 0u), dc.key);
    const uint64_t xlo = (uint64_t)o.x | ((uint64_t)o.y << 32);
    Step1 s;
    s.xhi = (uint64_t)o.z | ((uint64_t)o.w << 32);
    // ---- Step 1: level-1 reservoir ----
    s.d1 = bounded(u.m_prev + u.w, xlo, dc, 0x10000u);
    s.fresh = s.d1 >= u.m_prev;
    return s;
}

// A retained f1 changes only if the batch has an arc at one of its endpoints: chi^+ > 0, or the closing edge of an
// open wedge (it touches f1's endpoint x).  The filter has no false negatives.
__device__ __forceinline__ bool touched_by(const uint32_t *sf, uint2 r1) {
    return filter_has(sf, vfilter_bit(hash_vertex(r1.x))) || filter_has(sf, vfilter_bit(hash_vertex(r1.y)));
}

template <bool kSmall, bool kEF>
__device__ __forceinline__ uint32_t update_rest(const UpdateArgs &u, const UpdateIdx &ix, uint64_t t, const EstState &old,
                                                const Step1 &s1, uint32_t &n_fresh, uint32_t &n_r2old);

template <bool kSmall, bool kEF>
__device__ __forceinline__ uint32_t update_one(const UpdateArgs &u, const UpdateIdx &ix, uint64_t t, const EstState &old,
                                               uint32_t &n_fresh, uint32_t &n_r2old, uint32_t &n_skip, const uint32_t *sf) {
    const Step1 s1 = step1_draw(u, t);
    if (kSmall && !s1.fresh && !touched_by(sf, old.r1)) {  // nothing changes or is written
        ++n_skip;
        return (old.cf & kClosedBit) ? (old.cf & kCMask) : 0u;
    }
    return update_rest<kSmall, kEF>(u, ix, t, old, s1, n_fresh, n_r2old);
}

// Steps 2-3 and the state writes, after Step 1's draw (s1).  Returns chi if the estimator ends closed.
template <bool kSmall, bool kEF>
__device__ __forceinline__ uint32_t update_rest(const UpdateArgs &u, const UpdateIdx &ix, uint64_t t, const EstState &old,
                                                const Step1 &s1, uint32_t &n_fresh, uint32_t &n_r2old) {
    const uint64_t gid = u.first + t;
    const DrawCtx dc{gid, u.batch, PhiloxKey{(uint32_t)u.seed, (uint32_t)(u.seed >> 32)}};
    const uint64_t m_prev = u.m_prev, d1 = s1.d1, xhi = s1.xhi;
    const bool fresh = s1.fresh;
    const uint32_t j = fresh ? (uint32_t)(d1 - m_prev) : 0u;
    // ---- Step 2a: chi^+ = rank(u->v) + rank(v->u) ----
    // fresh f1 = w_j: its ranks from its arcs' pslot entries (apos[j]); retained f1: rank(u->v) = deg_W(u) (footnote
    // PAPER.md:818-821)
    uint2 r1 = old.r1;
    uint4 inf = make_uint4(0u, 0u, 0u, 0u);
    uint2 su = make_uint2(0u, 0u), sv = make_uint2(0u, 0u);
    const uint32_t hu = hash_vertex(r1.x), hv = hash_vertex(r1.y);
    if (fresh) {
        r1 = ldf<kEF>(ix.L.E + j);
        const uint2 ap = ldf<kEF>(ix.apos + j);
        TC_CHECK(j < u.w && ap.x < 2 * u.w && ap.y < 2 * u.w, ix.ctr);
        const uint2 pu = ldf<kEF>(ix.pslot + ap.x), pv = ldf<kEF>(ix.pslot + ap.y);
        TC_CHECK(pu.x < pu.y && pu.y <= 2 * u.w && pv.x < pv.y && pv.y <= 2 * u.w, ix.ctr);
        inf = make_uint4(pu.x, pu.y, pv.x, pv.y);
    } else {
        su = __ldg(ix.L.vslice + vbucket_of(hu, ix.L.bv));
        sv = __ldg(ix.L.vslice + vbucket_of(hv, ix.L.bv));
    }
    const uint32_t bu = vslot_start(hu, su.y), bw = vslot_start(hv, sv.y);
    uint4 u0 = make_uint4(kEmptyV, 0u, 0u, 0u), u1 = u0, v0 = u0, v1 = u0;
    if (su.y) {
        const uint4 *p = reinterpret_cast<const uint4 *>(ix.L.vt + su.x + bu);
        u0 = __ldg(p);
        u1 = __ldg(p + 1);
    }
    if (sv.y) {
        const uint4 *p = reinterpret_cast<const uint4 *>(ix.L.vt + sv.x + bw);
        v0 = __ldg(p);
        v1 = __ldg(p + 1);
    }
    uint32_t ld, rd, endU, endV;
    if (fresh) {
        ld = inf.y - 1u - inf.x;
        rd = inf.w - 1u - inf.z;
        endU = inf.y;
        endV = inf.w;
    } else {
        uint2 iu = u0.x == r1.x ? make_uint2(u0.y, u0.z) : u1.x == r1.x ? make_uint2(u1.y, u1.z) : make_uint2(0u, 0u);
        uint2 iv = v0.x == r1.y ? make_uint2(v0.y, v0.z) : v1.x == r1.y ? make_uint2(v1.y, v1.z) : make_uint2(0u, 0u);
        if (su.y && u0.x != r1.x && u1.x != r1.x && u0.x != kEmptyV && u1.x != kEmptyV)
            iu = vt_find_from(ix.L, su, bu, r1.x);  // rare: the first sector is full without u
        if (sv.y && v0.x != r1.y && v1.x != r1.y && v0.x != kEmptyV && v1.x != kEmptyV)
            iv = vt_find_from(ix.L, sv, bw, r1.y);
        ld = iu.x;
        rd = iv.x;
        endU = iu.y + iu.x;
        endV = iv.y + iv.x;
    }
    uint2 r2 = fresh ? make_uint2(kEmptyV, kEmptyV) : old.r2;
    uint32_t c = fresh ? 0u : (old.cf & kCMask);
    bool closed = !fresh && (old.cf & kClosedBit) != 0;
    const bool had_r2 = c > 0;  // NBSI: chi == 0 <=> f2 empty (always false for a fresh f1)
    const uint32_t chi_p = ld + rd;  // |Gamma_W(f1)|
    // ---- Step 2b: keep f2 w.p. chi^-/(chi^-+chi^+), else phi names an edge ----
    bool r2new = false;
    uint32_t k2 = 0, x = 0, z = 0;
    if (chi_p) {
        const uint64_t d2 = bounded((uint64_t)c + chi_p, xhi, dc, 0x20000u);
        r2new = d2 >= c;
        c += chi_p;
        const uint32_t phi = (uint32_t)(d2 - (c - chi_p));
        const bool atU = phi < ld;  // (src = u, rank = phi) or (src = v, rank = phi - ld)
        if (r2new) {
            TC_CHECK((atU ? endU : endV) - 1u - (atU ? phi : phi - ld) < 2 * u.w, ix.ctr);
            const uint2 arc = ldf<kEF>(ix.segS + ((atU ? endU : endV) - 1u - (atU ? phi : phi - ld)));
            const uint32_t src = atU ? r1.x : r1.y;
            k2 = arc.x >> 1;
            r2 = make_uint2(min(src, arc.y), max(src, arc.y));
            x = atU ? r1.y : r1.x;  // f1's endpoint not on f2
            z = arc.y;              // f2's endpoint not on f1
            closed = false;
        }
    }
    // ---- Step 3: closing edge after f2; an old f2 precedes every batch edge ----
    if (!r2new) {
        x = (r1.x == r2.x || r1.x == r2.y) ? r1.y : r1.x;
        z = (r2.x == r1.x || r2.x == r1.y) ? r2.y : r2.x;
    }
    // the closing edge touches x, so it can only be in W (after f2) if x has a batch arc (after f1 when f1 is
    // fresh): ld / rd count exactly those arcs, so x without any needs no probe
    const uint32_t degx = x == r1.x ? ld : rd;
    if ((r2new || had_r2) && !closed && degx) {
        const int64_t kk = pt_find_filtered<kEF>(ix.L, min(x, z), max(x, z));
        if (kk >= 0 && (!r2new || (uint32_t)kk > k2)) closed = true;
    }
    const uint32_t cf_new = c | (closed ? kClosedBit : 0u);
    if (kSmall) {  // only what changed (few estimators per batch)
        __stcs(u.cfs + t, cf_new);
        if (fresh) {
            __stcs(u.r1s + t, r1);
            __stcs(u.p1s + t, (uint32_t)d1);
        }
        if (fresh || r2new) {
            __stcs(u.r2s + t, r2);
            __stcs(u.p2s + t, r2new ? (uint32_t)(m_prev + k2) : kEmptyV);
        }
    } else {
        // every field rewritten: coalesced full sectors, no partial-sector read-modify-write
        __stcs(u.cfs + t, cf_new);
        __stcs(u.r1s + t, r1);
        __stcs(u.r2s + t, r2);
        __stcs(u.p1s + t, fresh ? (uint32_t)d1 : old.p1);
        __stcs(u.p2s + t, r2new ? (uint32_t)(m_prev + k2) : fresh ? kEmptyV : old.p2);
    }
    n_fresh += fresh ? 1u : 0u;
    n_r2old += (r2new && !fresh) ? 1u : 0u;
    return closed ? c : 0u;
}

// One pass over the estimator SoA: a grid of a few CTAs per SM loops over the estimators, reading the next
// estimator's state while it works on the current one.
#ifndef TC_UPD_MINB
#define TC_UPD_MINB 4
#endif
// kEF: a large batch (kPairFilterMin edges or more): one-shot probes evict-first in L2, as a compile-time
// constant so that the small instantiations carry no trace of it (C2: +3.5 us when it was a runtime flag)
template <bool kSmall, bool kEF>
__global__ void __launch_bounds__(256, TC_UPD_MINB) k_update(UpdateArgs u, UpdateIdx ix, unsigned long long *S,
                                                   unsigned long long *stats, const uint32_t *filt) {
    with_desc(u, ix.L);
    S += u.d->slot;
    if (ix.ctr[kCtrErr]) {  // this batch (or, in asynchronous mode, an earlier one) was rejected: no update
        // the first batch to see the sticky error word is the one that set it: record its index so that the
        // host can restore m and the batch count of the last accepted batch
        if (blockIdx.x == 0 && threadIdx.x == 0 && ix.ctr[kCtrFailB] == 0xFFFFFFFFu)
            ix.ctr[kCtrFailB] = u.batch;
        return;
    }
    __shared__ uint32_t sf[kSmall ? kFilterWords : 1];
    if (kSmall) {
        const uint4 *src = reinterpret_cast<const uint4 *>(filt);
        for (uint32_t i = threadIdx.x; i < kFilterWords / 4; i += blockDim.x) reinterpret_cast<uint4 *>(sf)[i] = __ldg(src + i);
        __syncthreads();
    }
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long contrib = 0;
    uint32_t n_fresh = 0, n_r2old = 0, n_skip = 0;
    EstState cur;
    if (t < u.count) cur = load_state<kSmall>(u, t);
    while (t < u.count) {
        const uint64_t tn = t + stride;
        EstState nxt;
        if (tn < u.count) nxt = load_state<kSmall>(u, tn);
        contrib += update_one<kSmall, kEF>(u, ix, t, cur, n_fresh, n_r2old, n_skip, sf);
        cur = nxt;
        t = tn;
    }
    // ---- a8: partial sum of chi over closed estimators (+ event counts for the byte model) ----
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        contrib += __shfl_xor_sync(kFull, contrib, off);
        n_fresh += __shfl_xor_sync(kFull, n_fresh, off);
        n_r2old += __shfl_xor_sync(kFull, n_r2old, off);
        if (kSmall) n_skip += __shfl_xor_sync(kFull, n_skip, off);
    }
    __shared__ unsigned long long ws[8];
    __shared__ uint32_t wf[8], wr[8], wk[8];
    if ((threadIdx.x & 31u) == 0) {
        ws[threadIdx.x >> 5] = contrib;
        wf[threadIdx.x >> 5] = n_fresh;
        wr[threadIdx.x >> 5] = n_r2old;
        wk[threadIdx.x >> 5] = n_skip;
    }
    __syncthreads();
    if (threadIdx.x < 8) {
        unsigned long long v = ws[threadIdx.x];
        uint32_t f = wf[threadIdx.x], q = wr[threadIdx.x], sk = wk[threadIdx.x];
#pragma unroll
        for (int off = 4; off > 0; off >>= 1) {
            v += __shfl_xor_sync(0xffu, v, off);
            f += __shfl_xor_sync(0xffu, f, off);
            q += __shfl_xor_sync(0xffu, q, off);
            if (kSmall) sk += __shfl_xor_sync(0xffu, sk, off);
        }
        if (threadIdx.x == 0) {
            if (v) atomicAdd(S, v);
            if (f) atomicAdd(stats + 0, (unsigned long long)f);
            if (q) atomicAdd(stats + 1, (unsigned long long)q);
            if (kSmall && sk) atomicAdd(stats + 4, (unsigned long long)sk);
            if (blockIdx.x == 0) {
                atomicAdd(stats + 2, (unsigned long long)ix.ctr[kCtrD]);
                atomicAdd(stats + 3, 1ull);
                atomicAdd(stats + 5, (unsigned long long)ix.ctr[kCtrArcsBig]);
                atomicAdd(stats + 6, (unsigned long long)ix.ctr[kCtrDBig]);
            }
        }
    }
}

// ------------------------------------------------------------------------------------------------
// a4..a8 split into one kernel per step (TC_TUNE_SPLIT_KERNELS): the same arithmetic as update_one, with the
// intermediate values of every estimator kept in StepBufs (per-step parity against the oracle's trace, and
// per-step timing -- the analogue of the paper's time-breakdown figure).

#define TC_GRID_STRIDE(t, n) for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (n); \
                                  t += (uint64_t)gridDim.x * blockDim.x)

// Ku1 -- Step 1, level-1 reservoir: one Philox block per estimator; a replaced f1 resets
// chi, f2 and the closed flag (readings R2, R3).
__global__ void __launch_bounds__(256) k_u1_resample(UpdateArgs u, const uint2 *E, StepBufs sb, uint32_t *ctr) {
    u.batch = u.d->batch;
    u.m_prev = u.d->m_prev;
    if (ctr[kCtrErr]) {  // as k_update: the first batch to see the sticky error word records its index
        if (blockIdx.x == 0 && threadIdx.x == 0 && ctr[kCtrFailB] == 0xFFFFFFFFu) ctr[kCtrFailB] = u.batch;
        return;
    }
    TC_GRID_STRIDE(t, u.count) {
        const uint64_t gid = u.first + t;
        const DrawCtx dc{gid, u.batch, PhiloxKey{(uint32_t)u.seed, (uint32_t)(u.seed >> 32)}};
        const uint4 o = philox4x32_10(make_uint4((uint32_t)gid, (uint32_t)(gid >> 32), u.batch, 0u), dc.key);
        const uint64_t xlo = (uint64_t)o.x | ((uint64_t)o.y << 32);
        const uint64_t d1 = bounded(u.m_prev + u.w, xlo, dc, 0x10000u);
        const bool fresh = d1 >= u.m_prev;
        const uint32_t j = fresh ? (uint32_t)(d1 - u.m_prev) : kEmptyV;
        if (fresh) {
            u.r1s[t] = E[j];
            u.p1s[t] = (uint32_t)d1;
            u.cfs[t] = 0u;
            u.r2s[t] = make_uint2(kEmptyV, kEmptyV);
            u.p2s[t] = kEmptyV;
        }
        sb.j[t] = j;
        sb.xhi[t] = (uint64_t)o.z | ((uint64_t)o.w << 32);
    }
}

// Ku2 -- Step 2a, chi^+ = rank(u->v) + rank(v->u): a fresh f1's ranks from pslot (via apos), a retained
// f1's from the vertex table (deg_W, footnote PAPER.md:818-821).
__global__ void __launch_bounds__(256) k_u2_count(UpdateArgs u, UpdateIdx ix, StepBufs sb) {
    with_desc(u, ix.L);
    if (ix.ctr[kCtrErr]) return;
    TC_GRID_STRIDE(t, u.count) {
        const uint2 r1 = u.r1s[t];
        const uint32_t j = sb.j[t];
        uint32_t ld, rd, endU, endV;
        if (j != kEmptyV) {
            const uint2 ap = ix.apos[j];
            const uint2 pu = ix.pslot[ap.x], pv = ix.pslot[ap.y];
            const uint4 inf = make_uint4(pu.x, pu.y, pv.x, pv.y);
            ld = inf.y - 1u - inf.x;
            rd = inf.w - 1u - inf.z;
            endU = inf.y;
            endV = inf.w;
        } else {
            VertProbe pu, pv;
            vt_issue(ix.L, r1.x, pu);
            vt_issue(ix.L, r1.y, pv);
            const uint2 iu = vt_resolve(ix.L, pu, r1.x), iv = vt_resolve(ix.L, pv, r1.y);
            ld = iu.x;
            rd = iv.x;
            endU = iu.y + iu.x;
            endV = iv.y + iv.x;
        }
        sb.chim[t] = u.cfs[t] & kCMask;
        sb.ld[t] = ld;
        sb.rd[t] = rd;
        sb.endU[t] = endU;
        sb.endV[t] = endV;
    }
}

// Ku3 -- Step 2b, level-2 select (naming 761-767): one draw d2 over chi^- + chi^+ (reading
// R4); phi = d2 - chi^- names the (phi)-th arc at u, else the (phi - ld)-th at v, by segment arithmetic.
__global__ void __launch_bounds__(256) k_u3_select(UpdateArgs u, UpdateIdx ix, StepBufs sb) {
    with_desc(u, ix.L);
    if (ix.ctr[kCtrErr]) return;
    TC_GRID_STRIDE(t, u.count) {
        const uint32_t ld = sb.ld[t], rd = sb.rd[t], chim = sb.chim[t], chi_p = ld + rd;
        uint64_t d2 = ~0ull;
        uint32_t k2 = kEmptyV;
        if (chi_p) {
            const uint64_t gid = u.first + t;
            const DrawCtx dc{gid, u.batch, PhiloxKey{(uint32_t)u.seed, (uint32_t)(u.seed >> 32)}};
            d2 = bounded((uint64_t)chim + chi_p, sb.xhi[t], dc, 0x20000u);
            uint32_t cf = u.cfs[t];
            if (d2 >= chim) {
                const uint2 r1 = u.r1s[t];
                const uint32_t phi = (uint32_t)(d2 - chim);
                const bool atU = phi < ld;
                const uint2 arc = ix.segS[(atU ? sb.endU[t] : sb.endV[t]) - 1u - (atU ? phi : phi - ld)];
                const uint32_t src = atU ? r1.x : r1.y;
                k2 = arc.x >> 1;
                u.r2s[t] = make_uint2(min(src, arc.y), max(src, arc.y));
                u.p2s[t] = (uint32_t)(u.m_prev + k2);
                cf = 0u;  // a new f2 has no closing edge yet (reading R5)
            }
            u.cfs[t] = (cf & kClosedBit) | (chim + chi_p);
        }
        sb.d2[t] = d2;
        sb.k2[t] = k2;
    }
}

// Ku4 -- Step 3, closing edge: the wedge's closing pair in the edge-pair hash, after f2
// (reading R6); skipped exactly when f1's endpoint x has no batch arc (the closing edge would touch x).
__global__ void __launch_bounds__(256) k_u4_close(UpdateArgs u, UpdateIdx ix, StepBufs sb) {
    with_desc(u, ix.L);
    if (ix.ctr[kCtrErr]) return;
    TC_GRID_STRIDE(t, u.count) {
        const uint32_t cf = u.cfs[t];
        const uint2 r2 = u.r2s[t];
        if (r2.x == kEmptyV || (cf & kClosedBit)) continue;
        const uint2 r1 = u.r1s[t];
        const uint32_t x = (r1.x == r2.x || r1.x == r2.y) ? r1.y : r1.x;
        const uint32_t z = (r2.x == r1.x || r2.x == r1.y) ? r2.y : r2.x;
        const uint32_t degx = x == r1.x ? sb.ld[t] : sb.rd[t];
        if (!degx) continue;
        const uint32_t k2 = sb.k2[t];
        const int64_t kk = pt_find(ix.L, min(x, z), max(x, z));
        if (kk >= 0 && (k2 == kEmptyV || (uint32_t)kk > k2)) u.cfs[t] = cf | kClosedBit;
    }
}

// Kr -- aggregation: S = sum of chi over closed estimators (exact u64) + the event counts.
__global__ void __launch_bounds__(256) k_r_reduce(UpdateArgs u, StepBufs sb, unsigned long long *S,
                                                  unsigned long long *stats, const uint32_t *ctr) {
    S += u.d->slot;
    if (ctr[kCtrErr]) return;
    unsigned long long contrib = 0;
    uint32_t n_fresh = 0, n_r2old = 0;
    TC_GRID_STRIDE(t, u.count) {
        const uint32_t cf = u.cfs[t];
        if (cf & kClosedBit) contrib += cf & kCMask;
        const bool fresh = sb.j[t] != kEmptyV;
        n_fresh += fresh ? 1u : 0u;
        n_r2old += (!fresh && sb.k2[t] != kEmptyV) ? 1u : 0u;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        contrib += __shfl_xor_sync(kFull, contrib, off);
        n_fresh += __shfl_xor_sync(kFull, n_fresh, off);
        n_r2old += __shfl_xor_sync(kFull, n_r2old, off);
    }
    if ((threadIdx.x & 31u) == 0) {
        if (contrib) atomicAdd(S, contrib);
        if (n_fresh) atomicAdd(stats + 0, (unsigned long long)n_fresh);
        if (n_r2old) atomicAdd(stats + 1, (unsigned long long)n_r2old);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        atomicAdd(stats + 2, (unsigned long long)ctr[kCtrD]);
        atomicAdd(stats + 3, 1ull);
        atomicAdd(stats + 5, (unsigned long long)ctr[kCtrArcsBig]);
        atomicAdd(stats + 6, (unsigned long long)ctr[kCtrDBig]);
    }
}

__global__ void k_init_state(uint2 *r1, uint2 *r2, uint32_t *cf, uint32_t *p1, uint32_t *p2, uint64_t count) {
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += (uint64_t)gridDim.x * blockDim.x) {
        r1[t] = make_uint2(kEmptyV, kEmptyV);
        r2[t] = make_uint2(kEmptyV, kEmptyV);
        cf[t] = 0;
        p1[t] = kEmptyV;
        p2[t] = kEmptyV;
    }
}

// S_g over contiguous groups of global ids g = [floor(g N / G), floor((g+1) N / G)); local estimator t has
// global id first + t (N = 1 puts every estimator into group 0).
__global__ void k_group_sums(const uint32_t *__restrict__ cf, uint64_t count, uint64_t first, uint64_t N, uint32_t G,
                             unsigned long long *out) {
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = cf[t];
        if (!(v & kClosedBit)) continue;
        const uint64_t i = N == 1 ? 0 : first + t;
        const uint64_t g = ((i + 1) * G + N - 1) / N - 1;
        atomicAdd(out + g, (unsigned long long)(v & kCMask));
    }
}

// The first node of every push: the batch's descriptor into device memory, and the per-batch resets (the
// counters except the sticky error word and the failed-batch index, this batch's S, the small-batch filter)
// ahead of every kernel of the batch.  Event mode (edctr != null): S is carried over from the
// previous batch (d.pad bit 0), the queue is emptied, and the batch becomes a full sweep when the host asks for one
// (d.pad bit 1) or the watch-node pool has passed its rebuild threshold.
__global__ void __launch_bounds__(256) k_desc(BatchDesc d, BatchDesc *dst, uint32_t *ctr, unsigned long long *S,
                                              uint32_t *filt, uint32_t *edctr) {
    if (threadIdx.x == 0) {
        *dst = d;
        S[d.slot] = (d.pad & 1u) ? S[d.slot ^ 1u] : 0ull;
        if (edctr) {
            edctr[kEdQueue] = 0u;
            uint32_t used = 0;  // the fullest stripe of the watch-chunk pool
            for (uint32_t i = 0; i < kEdStripes; ++i) used = max(used, edctr[kEdStripe0 + i]);
            edctr[kEdFull] = ((d.pad & 2u) || used > edctr[kEdThr]) ? 1u : 0u;
        }
    }
    if (threadIdx.x < (uint32_t)kCtrWords && threadIdx.x != (uint32_t)kCtrErr && threadIdx.x != (uint32_t)kCtrFailB)
        ctr[threadIdx.x] = 0u;
    if (filt)
        for (uint32_t i = threadIdx.x; i < kFilterWords; i += blockDim.x) filt[i] = 0u;
}

int launch_desc(const IndexBufs &ix, const BatchArgs &a, const BatchDesc &d, uint32_t *edctr, cudaStream_t s) {
    k_desc<<<1, 256, 0, s>>>(d, ix.desc, ix.ctr, a.S, a.small ? ix.filt : nullptr, edctr);
    return 1;
}

const void *desc_kernel() { return (const void *)k_desc; }

// Test hooks (tc_test_draws / tc_test_philox): the estimator pass's own device functions on chosen inputs.
__global__ void k_test_draws(const uint64_t *n, const uint64_t *x, const uint64_t *id, const uint32_t *b,
                             const uint32_t *base, uint64_t seed, uint64_t count, uint64_t *out) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= count) return;
    const DrawCtx dc{id[t], b[t], PhiloxKey{(uint32_t)seed, (uint32_t)(seed >> 32)}};
    out[t] = bounded(n[t], x[t], dc, base[t]);
}

__global__ void k_test_philox(const uint4 *ctr, const uint2 *key, uint64_t count, uint4 *out) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= count) return;
    out[t] = philox4x32_10(ctr[t], PhiloxKey{key[t].x, key[t].y});
}

int launch_test_draws(const uint64_t *n, const uint64_t *x, const uint64_t *id, const uint32_t *b, const uint32_t *base,
                      uint64_t seed, uint64_t count, uint64_t *out, cudaStream_t s) {
    k_test_draws<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(n, x, id, b, base, seed, count, out);
    return 1;
}

int launch_test_philox(const uint32_t *ctr, const uint32_t *key, uint64_t count, uint32_t *out, cudaStream_t s) {
    k_test_philox<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(reinterpret_cast<const uint4 *>(ctr),
                                                                  reinterpret_cast<const uint2 *>(key), count,
                                                                  reinterpret_cast<uint4 *>(out));
    return 1;
}

// ------------------------------------------------------------------------------------------------
static int g_sms = 0;
int sm_count() {
    if (!g_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_sms <= 0) g_sms = 148;
    }
    return g_sms;
}

#ifndef TC_UPD_WAVES
#define TC_UPD_WAVES 1
#endif
constexpr uint32_t kUpdateCTAsPerSM = TC_UPD_MINB, kUpdateWaves = TC_UPD_WAVES;  // k_update grid

static inline uint32_t grid_for(uint64_t items, uint32_t threads, uint32_t per_sm) {
    const uint64_t want = (items + threads - 1) / threads;
    const uint64_t cap = (uint64_t)sm_count() * per_sm;
    return (uint32_t)std::max<uint64_t>(1, std::min(want, cap));
}

static inline uint32_t ceil_log2(uint64_t x) {
    uint32_t b = 0;
    while ((1ull << b) < x) ++b;
    return b;
}

Geometry make_geometry(uint32_t w, const Tuning &t) {
    Geometry g;
    g.w = w;
    g.small_index = t.small_index == 2 ? (w <= kSmallIndexMax) : t.small_index == 1 ? false : (w <= kSmallIndexMax);
    g.tiles = (w + kTileEdges - 1) / kTileEdges;
    g.bv = std::min(kMaxBucketBits, ceil_log2((2ull * w + t.vbucket_arcs - 1) / t.vbucket_arcs));
    g.bp1 = std::min(g.bv, kMaxPartBits);
    g.bs = g.bv - g.bp1;
    g.vcap = std::min(t.vcap, kHCapSmall);
    g.sortcap = std::min(t.sortcap, kVChunk);
    if (g.small_index) {  // one CTA per vertex bucket of ~small_index_arcs arcs (no partition kernels)
        g.bv = std::min<uint32_t>(kSmallIndexMaxBits, ceil_log2((2ull * w + t.small_index_arcs - 1) / t.small_index_arcs));
        g.bp1 = g.bs = 0;
    }
    return g;
}

static PartArgs part_args(const IndexBufs &ix, const BatchArgs &a) {
    return PartArgs{ix.desc, reinterpret_cast<uint32_t *>(ix.apos), a.g, ix.E, ix.arcs, ix.cntV, ix.offV, ix.arank, ix.vstart, ix.pt, pair_groups(a.g.w), ix.ctr,
                    a.small ? ix.filt : nullptr, a.S, a.pfilt ? ix.pf : nullptr, pf_words(a.g.w),
                    pf_words((uint32_t)ix.wcap)};
}

int launch_partition(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s, const KRec &kr) {
    const Geometry &g = a.g;
    const uint32_t nV = 1u << g.bp1;
    const PartArgs p = part_args(ix, a);
    kr.beg(K_COUNT, s);
    switch (g.bp1) {
#define TC_COUNT_CASE(B) \
    case B: k_count<B><<<g.tiles, kTileThreads, 2 * kTileWarps * nV, s>>>(p); break;
        TC_COUNT_CASE(0) TC_COUNT_CASE(1) TC_COUNT_CASE(2) TC_COUNT_CASE(3) TC_COUNT_CASE(4) TC_COUNT_CASE(5)
        TC_COUNT_CASE(6) TC_COUNT_CASE(7) TC_COUNT_CASE(8) TC_COUNT_CASE(9) TC_COUNT_CASE(10) TC_COUNT_CASE(11)
        TC_COUNT_CASE(12)
#undef TC_COUNT_CASE
        default: return 0;
    }
    kr.end(K_COUNT, s);
    kr.beg(K_SCAN_COLS, s);
    k_scan_cols<<<(nV + 31) / 32, kScanWarps * 32, 0, s>>>(ix.cntV, ix.offV, ix.vstart, g.tiles, nV, ix.ctr);
    kr.end(K_SCAN_COLS, s);
    // with a split, the large-bucket list is built by k_split over the sub-buckets
    kr.beg(K_SCAN_TOT, s);
    k_scan_tot<<<1, 1024, 0, s>>>(ix.vstart, nV, g.bs ? 0xFFFFFFFFu : g.vcap, ix.vperm, ix.ctr);
    kr.end(K_SCAN_TOT, s);
    kr.beg(K_SCATTER, s);
    if (g.w >= kScatterGlobalEMin)
        k_scatter<false><<<g.tiles, kTileThreads, 8 * nV + 4 * kTileEdges, s>>>(p);
    else
        k_scatter<true><<<g.tiles, kTileThreads, 8 * nV + 12 * kTileEdges, s>>>(p);
    kr.end(K_SCATTER, s);
    if (!g.bs) return 4;
    SplitArgs sa{ix.arcs, ix.arcs2, ix.vstart, ix.vstart2, g.bp1, g.bs, g.vcap, ix.vperm, ix.ctr};
    kr.beg(K_SPLIT, s);
    static_assert(kMaxSplitBits <= 5, "k_split scans each sub-bucket with one of its 32 warps");
    switch (g.bs) {
        case 1: k_split<1><<<nV, kSplitThreads, 0, s>>>(sa); break;
        case 2: k_split<2><<<nV, kSplitThreads, 0, s>>>(sa); break;
        case 3: k_split<3><<<nV, kSplitThreads, 0, s>>>(sa); break;
        case 4: k_split<4><<<nV, kSplitThreads, 0, s>>>(sa); break;
        default: k_split<5><<<nV, kSplitThreads, 0, s>>>(sa); break;
    }
    kr.end(K_SPLIT, s);
    return 5;
}

int launch_pairs(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s, const KRec &kr) {
    kr.beg(K_PAIRS, s);
    k_pairs<<<(a.g.w + 255) / 256, 256, 0, s>>>(part_args(ix, a));
    kr.end(K_PAIRS, s);
    return 1;
}

static VertArgs vert_args(const IndexBufs &ix, const BatchArgs &a) {
    return VertArgs{a.g.bs ? ix.arcs2 : ix.arcs, ix.scratch, reinterpret_cast<uint4 *>(ix.scratch), ix.E,
                    a.g.bs ? ix.vstart2 : ix.vstart, ix.segS, ix.pslot, reinterpret_cast<const uint32_t *>(ix.apos), ix.vt, ix.vslice,
                    ix.vperm, ix.vdefer, a.g.bv, a.g.vcap, a.g.sortcap, ix.ctr, 2 * a.g.w};
}

int launch_small_index(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s, const KRec &kr) {
    kr.beg(K_SMALL, s);
    if (a.g.w <= 2048)
        k_small_index<256, 4096><<<1u << a.g.bv, 256, SmallIndexCfg<256, 4096>::kSmemBytes, s>>>(part_args(ix, a),
                                                                                             vert_args(ix, a));
    else
        k_small_index<512, 8192><<<1u << a.g.bv, 512, SmallIndexCfg<512, 8192>::kSmemBytes, s>>>(part_args(ix, a),
                                                                                             vert_args(ix, a));
    kr.end(K_SMALL, s);
    return 1;
}

int launch_vertices(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s, const KRec &kr) {
    kr.beg(K_VHASH, s);
    k_vhash<<<1u << a.g.bv, kHThreads, kVHashSmemBytes, s>>>(vert_args(ix, a));
    kr.end(K_VHASH, s);
    return 1;
}

int launch_vertices_big(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s, const KRec &kr) {
    kr.beg(K_VHUB, s);
    k_vhub<<<sm_count(), kHubThreads, kVHubSmemBytes, s>>>(vert_args(ix, a));
    kr.end(K_VHUB, s);
    kr.beg(K_VBIG, s);
    k_vbig<<<kBigCTAs, kVBucketThreads, kVSmemBytes, s>>>(vert_args(ix, a));
    kr.end(K_VBIG, s);
    return 2;
}

int launch_update(const IndexBufs &ix, const StateBufs &st, const BatchArgs &a, cudaStream_t s, const KRec &kr) {
    if (st.count == 0) return 0;
    UpdateIdx ui{Lookup{ix.E, ix.vt, ix.vslice, a.g.bv, ix.pt, pair_groups(a.g.w), 0u, a.pfilt ? ix.pf : nullptr,
                        a.pfilt ? pf_words(a.g.w) : 0u, pf_words((uint32_t)ix.wcap)},
                 ix.apos, ix.pslot, ix.segS, ix.ctr};
    UpdateArgs u{st.r1, st.r2, st.cf, st.p1, st.p2, st.count, a.first, a.seed, 0u, a.g.w, 0ull, ix.desc};
    const uint32_t grid = grid_for(st.count, 256, kUpdateCTAsPerSM * kUpdateWaves);
    kr.beg(K_UPDATE, s);
    if (a.small)
        k_update<true, false><<<grid, 256, 0, s>>>(u, ui, st.S, st.stats, ix.filt);
    else if (a.g.w >= kPairFilterMin)
        k_update<false, true><<<grid, 256, 0, s>>>(u, ui, st.S, st.stats, nullptr);
    else
        k_update<false, false><<<grid, 256, 0, s>>>(u, ui, st.S, st.stats, nullptr);
    kr.end(K_UPDATE, s);
    return 1;
}

int launch_update_split(const IndexBufs &ix, const StateBufs &st, const StepBufs &sb, const BatchArgs &a, cudaStream_t s,
                        const KRec &kr) {
    if (st.count == 0) return 0;
    UpdateIdx ui{Lookup{ix.E, ix.vt, ix.vslice, a.g.bv, ix.pt, pair_groups(a.g.w), 0u}, ix.apos, ix.pslot, ix.segS, ix.ctr};
    UpdateArgs u{st.r1, st.r2, st.cf, st.p1, st.p2, st.count, a.first, a.seed, 0u, a.g.w, 0ull, ix.desc};
    const uint32_t grid = grid_for(st.count, 256, 8);
    kr.beg(K_U1, s);
    k_u1_resample<<<grid, 256, 0, s>>>(u, ix.E, sb, ix.ctr);
    kr.end(K_U1, s);
    kr.beg(K_U2, s);
    k_u2_count<<<grid, 256, 0, s>>>(u, ui, sb);
    kr.end(K_U2, s);
    kr.beg(K_U3, s);
    k_u3_select<<<grid, 256, 0, s>>>(u, ui, sb);
    kr.end(K_U3, s);
    kr.beg(K_U4, s);
    k_u4_close<<<grid, 256, 0, s>>>(u, ui, sb);
    kr.end(K_U4, s);
    kr.beg(K_R, s);
    k_r_reduce<<<grid, 256, 0, s>>>(u, sb, st.S, st.stats, ix.ctr);
    kr.end(K_R, s);
    return 5;
}

int launch_init_state(const StateBufs &st, cudaStream_t s) {
    if (!st.count) return 0;
    k_init_state<<<grid_for(st.count, 256, 16), 256, 0, s>>>(st.r1, st.r2, st.cf, st.p1, st.p2, st.count);
    return 1;
}

int launch_group_sums(const StateBufs &st, uint64_t first, uint64_t N, uint32_t groups, unsigned long long *out,
                      cudaStream_t s) {
    if (!st.count) return 0;
    k_group_sums<<<grid_for(st.count, 256, 16), 256, 0, s>>>(st.cf, st.count, first, N, groups, out);
    return 1;
}

int set_kernel_attributes() {
    cudaError_t e1 = cudaFuncSetAttribute(k_vbig, cudaFuncAttributeMaxDynamicSharedMemorySize, kVSmemBytes);
    if (e1 == cudaSuccess) e1 = cudaFuncSetAttribute(k_vhash, cudaFuncAttributeMaxDynamicSharedMemorySize, kVHashSmemBytes);
    if (e1 == cudaSuccess) e1 = cudaFuncSetAttribute(k_vhub, cudaFuncAttributeMaxDynamicSharedMemorySize, kVHubSmemBytes);

    if (e1 == cudaSuccess)
        e1 = cudaFuncSetAttribute(k_small_index<256, 4096>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  SmallIndexCfg<256, 4096>::kSmemBytes);
    if (e1 == cudaSuccess)
        e1 = cudaFuncSetAttribute(k_small_index<512, 8192>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  SmallIndexCfg<512, 8192>::kSmemBytes);
    cudaError_t e2 = cudaSuccess;
    const void *counts[] = {(const void *)k_count<0>, (const void *)k_count<1>, (const void *)k_count<2>,
                            (const void *)k_count<3>, (const void *)k_count<4>, (const void *)k_count<5>,
                            (const void *)k_count<6>, (const void *)k_count<7>, (const void *)k_count<8>,
                            (const void *)k_count<9>, (const void *)k_count<10>, (const void *)k_count<11>,
                            (const void *)k_count<12>};
    for (int b = 0; b <= 12 && e2 == cudaSuccess; ++b)
        e2 = cudaFuncSetAttribute(counts[b], cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kTileWarps * (1 << b));
    if (e2 == cudaSuccess)
        e2 = cudaFuncSetAttribute(k_scatter<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4096 + 12 * kTileEdges);
    if (e2 == cudaSuccess)
        e2 = cudaFuncSetAttribute(k_scatter<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4096 + 4 * kTileEdges);
    return (e1 == cudaSuccess && e2 == cudaSuccess) ? 0 : -1;
}

}  // namespace tcb

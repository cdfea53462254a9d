// kernels.cu -- the per-batch hot path of bulkUpdateAll on sm_100a.
//
// Pipeline for one batch W; tiles are 2048 edges = 4096 arcs:
//   k_hist       a1      : per-tile counts of digit 0 of the arc keys, global histograms of all digits
//   k_scan               : per digit, exclusive scan over tiles + digit base = each tile's output offsets
//   k_stage      a1 + a3 : load W (coalesced), validate, normalize to (lo, hi); insert every edge into the
//                          edge-pair hash (one 128-bit CAS per claim, 8 inserts in flight per thread);
//                          rank the tile's arcs (vertex, k<<1|side) stably by digit 0 and scatter them --
//                          the F array of rankAll's proof, already radix pass 0
//   k_upsweep / k_scan / k_downsweep  a2 : the remaining stable LSD radix passes over the arcs by vertex id
//                          (passes whose digit is 0 for every arc are skipped on the device).  Stability
//                          keeps arrival order inside a vertex: this replaces rankAll's sort by (src, -pos)
//                          (PAPER.md:680-684).
//   k_runs       a2      : runs of equal vertex inside each tile -> vertex table {deg_W, segment start};
//                          rank / segment end of the arcs of tile-internal segments
//   k_fix        a2      : rank / segment end of the arcs of segments that cross tile boundaries
//   k_update     a4..a8  : ONE pass over the estimator SoA: Step 1 (level-1 reservoir), Step 2 (chi^+
//                          from ranks / degrees, level-2 pick by segment arithmetic), Step 3 (closing-edge
//                          probe), block partial sums of chi over closed estimators
// rank(x->y) of the arc at sorted slot s = segEnd(x) - 1 - s (Definition Rank).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "index.cuh"
#include "kernels.h"
#include "philox.cuh"

namespace tcb {

typedef unsigned __int128 u128;

__device__ __forceinline__ u128 pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    return (u128)a | ((u128)b << 32) | ((u128)c << 64) | ((u128)d << 96);
}
__device__ __forceinline__ u128 pack2(unsigned long long a, unsigned long long b) {
    return (u128)a | ((u128)b << 64);
}

constexpr uint32_t kTileEdges = kRadixTile / 2;
constexpr uint32_t kWarps = kSortThreads / 32;

// Arc keys are vertex ids; pass p sorts by digit (key >> 8p) & 255.
__device__ __forceinline__ uint32_t digit_of(uint32_t key, uint32_t pass) {
    return (key >> (pass * kRadixBits)) & (kRadix - 1);
}

// A pass is trivial (identity) when every arc has digit 0 there.
__device__ __forceinline__ bool pass_trivial(const uint32_t *hist, uint32_t p, uint32_t n) {
    return hist[p * kRadix] == n;
}
// k_stage always writes pass 0's output to buffer B; each executed later pass flips A/B.
__device__ __forceinline__ bool in_buffer_B(const uint32_t *hist, uint32_t upto, uint32_t n) {
    uint32_t e = 0;
    for (uint32_t p = 1; p < upto; ++p) e += pass_trivial(hist, p, n) ? 0u : 1u;
    return (e & 1u) == 0;
}

// Edge-tile loads: thread i takes edges i, i+256, ... of the tile (coalesced 8-byte loads).
__device__ __forceinline__ uint2 norm_edge(uint2 e) { return make_uint2(min(e.x, e.y), max(e.x, e.y)); }

// ------------------------------------------------------------------------------------------------
// a1: digit histograms

__global__ void __launch_bounds__(kSortThreads) k_hist(const uint2 *__restrict__ in, uint32_t w, uint32_t *hist,
                                                        uint32_t *cnt, uint32_t ntiles, const uint32_t *ctr) {
    // (a duplicate found by k_pairs of this very batch must not stop staging: only stage errors here)
    if (ctr[kCtrErr] & kErrStage) return;  // sticky error of an earlier async batch
    __shared__ uint32_t sh[kPasses][kRadix];
    for (uint32_t i = threadIdx.x; i < kPasses * kRadix; i += kSortThreads) (&sh[0][0])[i] = 0;
    __syncthreads();
    const uint32_t e0 = blockIdx.x * kTileEdges;
#pragma unroll 4
    for (uint32_t i = threadIdx.x; i < kTileEdges; i += kSortThreads) {
        if (e0 + i >= w) break;
        const uint2 e = norm_edge(__ldg(in + e0 + i));
#pragma unroll
        for (uint32_t p = 0; p < kPasses; ++p) {
            atomicAdd(&sh[p][digit_of(e.x, p)], 1u);
            atomicAdd(&sh[p][digit_of(e.y, p)], 1u);
        }
    }
    __syncthreads();
    const uint32_t d = threadIdx.x;  // kSortThreads == kRadix
    cnt[d * ntiles + blockIdx.x] = sh[0][d];
#pragma unroll
    for (uint32_t p = 0; p < kPasses; ++p)
        if (sh[p][d]) atomicAdd(hist + p * kRadix + d, sh[p][d]);
}

// Per-tile digit counts of pass p >= 1 (the keys as left by the previous executed pass).
__global__ void __launch_bounds__(kSortThreads) k_upsweep(const uint32_t *keyA, const uint32_t *keyB, uint32_t n,
                                                          const uint32_t *hist, uint32_t pass, uint32_t *cnt,
                                                          uint32_t ntiles, const uint32_t *ctr) {
    if (ctr[kCtrErr] || pass_trivial(hist, pass, n)) return;
    const uint32_t *__restrict__ kin = in_buffer_B(hist, pass, n) ? keyB : keyA;
    __shared__ uint32_t sh[kRadix];
    sh[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t t0 = blockIdx.x * kRadixTile;
    const uint4 *k4 = reinterpret_cast<const uint4 *>(kin + t0);
#pragma unroll
    for (uint32_t j = 0; j < kSortItems / 4; ++j) {
        const uint32_t q = threadIdx.x + j * kSortThreads;
        if (t0 + 4 * q + 3 < n) {
            const uint4 v = __ldcs(k4 + q);
            atomicAdd(&sh[digit_of(v.x, pass)], 1u);
            atomicAdd(&sh[digit_of(v.y, pass)], 1u);
            atomicAdd(&sh[digit_of(v.z, pass)], 1u);
            atomicAdd(&sh[digit_of(v.w, pass)], 1u);
        } else {
            for (uint32_t u = 0; u < 4; ++u)
                if (t0 + 4 * q + u < n) atomicAdd(&sh[digit_of(kin[t0 + 4 * q + u], pass)], 1u);
        }
    }
    __syncthreads();
    cnt[threadIdx.x * ntiles + blockIdx.x] = sh[threadIdx.x];
}

// One block per digit: offsets[d][t] = sum_{d' < d} hist[d'] + sum_{t' < t} cnt[d][t'].
__global__ void __launch_bounds__(kSortThreads) k_scan(uint32_t *cnt, uint32_t ntiles, const uint32_t *hist,
                                                       uint32_t pass, uint32_t n, const uint32_t *ctr) {
    if (ctr[kCtrErr]) return;
    if (pass > 0 && pass_trivial(hist, pass, n)) return;
    __shared__ uint32_t ws[kWarps];
    const uint32_t d = blockIdx.x, lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    // digit base
    uint32_t hv = threadIdx.x < d ? hist[pass * kRadix + threadIdx.x] : 0u;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) hv += __shfl_xor_sync(0xffffffffu, hv, off);
    if (lane == 0) ws[warp] = hv;
    __syncthreads();
    uint32_t base = 0;
    for (uint32_t x = 0; x < kWarps; ++x) base += ws[x];
    __syncthreads();
    // exclusive scan of the digit's row, chunk per thread
    uint32_t *row = cnt + (size_t)d * ntiles;
    const uint32_t per = (ntiles + kSortThreads - 1) / kSortThreads;
    const uint32_t c0 = threadIdx.x * per, c1 = min(ntiles, c0 + per);
    uint32_t local = 0;
    for (uint32_t i = c0; i < c1; ++i) local += row[i];
    uint32_t incl = local;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= (uint32_t)off) incl += y;
    }
    if (lane == 31) ws[warp] = incl;
    __syncthreads();
    uint32_t run = base + incl - local;
    for (uint32_t x = 0; x < warp; ++x) run += ws[x];
    for (uint32_t i = c0; i < c1; ++i) {
        const uint32_t c = row[i];
        row[i] = run;
        run += c;
    }
}

// Lanes of the warp whose 8-bit digit equals d (d == kRadix: no arc), from 9 ballots instead of
// __match_any_sync (a slow MIO op on this part).
__device__ __forceinline__ uint32_t digit_peers(uint32_t d) {
    uint32_t m = __ballot_sync(0xffffffffu, d < kRadix);
    if (d >= kRadix) m = ~m;
#pragma unroll
    for (uint32_t b = 0; b < kRadixBits; ++b) {
        const uint32_t v = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        m &= ((d >> b) & 1u) ? v : ~v;
    }
    return m;
}

// Stable in-tile ranks by digit: warp w owns arcs [512w, 512w+512) of the tile in 16 rounds of 32.
// On return whist[w][d] = arcs of digit d in warps < w, and rnk[j] = rank among digit-d arcs of warp w.
__device__ __forceinline__ void rank_tile(const uint32_t (&dg)[kSortItems], uint32_t (&rnk)[kSortItems],
                                          uint32_t (*whist)[kRadix]) {
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    for (uint32_t i = threadIdx.x; i < kWarps * kRadix; i += kSortThreads) (&whist[0][0])[i] = 0;
    __syncthreads();
#pragma unroll
    for (uint32_t j = 0; j < kSortItems; ++j) {
        const uint32_t d = dg[j];  // kRadix marks "no arc"
        const uint32_t peers = digit_peers(d);
        const uint32_t before = __popc(peers & lt);
        uint32_t b = 0;
        if (d < kRadix) b = whist[warp][d];
        __syncwarp();
        if (d < kRadix && before == 0) whist[warp][d] = b + __popc(peers);
        __syncwarp();
        rnk[j] = b + before;
    }
    __syncthreads();
    const uint32_t dd = threadIdx.x;  // per digit: exclusive prefix over warps (warp order == arc order)
    uint32_t tot = 0;
#pragma unroll
    for (uint32_t x = 0; x < kWarps; ++x) {
        const uint32_t c = whist[x][dd];
        whist[x][dd] = tot;
        tot += c;
    }
    __syncthreads();
}

// ------------------------------------------------------------------------------------------------
// a1 + a3 (+ radix pass 0): staging, validation, edge-pair hash, arcs

struct StageCtx {
    uint2 *E;
    uint32_t *keyB, *valB;  // pass-0 output
    const uint32_t *off;    // scanned per-tile digit-0 offsets
    const uint32_t *hist;
    uint32_t ntiles;
    PSlot *pt;
    uint32_t pmask;
    uint32_t tag;
    uint32_t *ctr;
};

__global__ void __launch_bounds__(kSortThreads, 3) k_stage(const uint2 *__restrict__ in, uint32_t w, StageCtx c) {
    if (c.ctr[kCtrErr] & kErrStage) return;  // sticky error of an earlier async batch
    __shared__ uint2 sedge[kTileEdges];
    __shared__ uint32_t whist[kWarps][kRadix];
    __shared__ uint32_t soff[kRadix];
    const uint32_t e0 = blockIdx.x * kTileEdges;
    const uint32_t ne = min(kTileEdges, w - e0);
    const bool trivial0 = pass_trivial(c.hist, 0, 2 * w);
    soff[threadIdx.x] = c.off[threadIdx.x * c.ntiles + blockIdx.x];
    // per edge: validate, normalize, E (the edge-pair hash is filled concurrently by k_pairs)
    constexpr uint32_t kPer = kTileEdges / kSortThreads;
    uint32_t bad = 0;
#pragma unroll
    for (uint32_t j = 0; j < kPer; ++j) {
        const uint32_t i = threadIdx.x + j * kSortThreads;
        uint2 e = make_uint2(0u, 0u);
        if (i < ne) e = __ldcs(in + e0 + i);
        const uint2 n = norm_edge(e);
        sedge[i] = n;
        if (i < ne) {
            if (e.x == kEmptyV || e.y == kEmptyV) bad |= kErrInval;
            else if (e.x == e.y) bad |= kErrLoop;
            else c.E[e0 + i] = n;
        }
    }
    // radix pass 0 over the tile's arcs (arc a = 2k + side, in arrival order)
    uint32_t dg[kSortItems], rnk[kSortItems], kv[kSortItems];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    __syncthreads();
#pragma unroll
    for (uint32_t j = 0; j < kSortItems; ++j) {
        const uint32_t a = warp * 512u + j * 32u + lane;  // arc index inside the tile
        const uint2 n = sedge[a >> 1];
        kv[j] = (a & 1u) ? n.y : n.x;
        dg[j] = (a >> 1) < ne ? digit_of(kv[j], 0) : kRadix;
    }
    if (!trivial0) rank_tile(dg, rnk, whist);
#pragma unroll
    for (uint32_t j = 0; j < kSortItems; ++j) {
        const uint32_t a = warp * 512u + j * 32u + lane;
        if ((a >> 1) >= ne) continue;
        const uint32_t ga = 2 * e0 + a;
        const uint32_t pos = trivial0 ? ga : soff[dg[j]] + whist[warp][dg[j]] + rnk[j];
        c.keyB[pos] = kv[j];
        c.valB[pos] = ga;
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (bad && lane == 0) atomicOr(&c.ctr[kCtrErr], bad);
}

// a3: the edge-pair hash {lo<<32|hi -> k} (Step 3's closing-edge index), built on a second stream
// concurrently with the radix sort.  One edge per thread (many threads in flight hide the probe round
// trips); a claim is one 128-bit CAS of {key, k, tag}; a repeat of a pair is TC_EDUP.
__global__ void __launch_bounds__(256) k_pairs(const uint2 *__restrict__ in, uint32_t w, StageCtx c) {
    if (c.ctr[kCtrErr] & (kErrInval | kErrLoop | kErrDup)) return;  // sticky error of an earlier async batch
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t bad = 0;
    if (k < w) {
        const uint2 e = __ldcs(in + k);
        if (e.x != kEmptyV && e.y != kEmptyV && e.x != e.y) {  // invalid edges: k_stage reports them
            const uint2 n = norm_edge(e);
            const unsigned long long key = pair_key(n.x, n.y);
            uint32_t b = hash_pair(key) & c.pmask & ~1u;
            while (true) {
                const ulonglong2 *p = reinterpret_cast<const ulonglong2 *>(c.pt + b);
                const ulonglong2 s0 = __ldcg(p), s1 = __ldcg(p + 1);
                const bool l0 = (uint32_t)(s0.y >> 32) == c.tag, l1 = (uint32_t)(s1.y >> 32) == c.tag;
                if ((l0 && s0.x == key) || (l1 && s1.x == key)) {
                    bad = kErrDup;
                    break;
                }
                if (l0 && l1) {
                    b = (b + 2) & c.pmask;
                    continue;
                }
                const uint32_t s = l0 ? 1u : 0u;
                const ulonglong2 o = s ? s1 : s0;
                const u128 exp = pack2(o.x, o.y);
                if (atomicCAS(reinterpret_cast<u128 *>(c.pt + b + s), exp,
                              pack2(key, ((unsigned long long)c.tag << 32) | k)) == exp)
                    break;
            }
        }
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (bad && (threadIdx.x & 31u) == 0) atomicOr(&c.ctr[kCtrErr], bad);
}

// Radix pass p >= 1: stable rank inside the tile, scatter to the scanned offsets.
__global__ void __launch_bounds__(kSortThreads, 3) k_downsweep(uint32_t *keyA, uint32_t *valA, uint32_t *keyB,
                                                            uint32_t *valB, uint32_t n, const uint32_t *hist,
                                                            uint32_t pass, const uint32_t *off, uint32_t ntiles,
                                                            const uint32_t *ctr) {
    if (ctr[kCtrErr] || pass_trivial(hist, pass, n)) return;
    const bool fromB = in_buffer_B(hist, pass, n);
    const uint32_t *__restrict__ kin = fromB ? keyB : keyA;
    const uint32_t *__restrict__ vin = fromB ? valB : valA;
    uint32_t *__restrict__ kout = fromB ? keyA : keyB;
    uint32_t *__restrict__ vout = fromB ? valA : valB;
    __shared__ uint32_t whist[kWarps][kRadix];
    __shared__ uint32_t soff[kRadix];
    soff[threadIdx.x] = off[threadIdx.x * ntiles + blockIdx.x];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t wbase = blockIdx.x * kRadixTile + warp * 512u;
    uint32_t keys[kSortItems], vals[kSortItems], dg[kSortItems], rnk[kSortItems];
#pragma unroll
    for (uint32_t j = 0; j < kSortItems; ++j) {
        const uint32_t idx = wbase + j * 32u + lane;
        const bool valid = idx < n;
        keys[j] = valid ? __ldcs(kin + idx) : 0u;
        vals[j] = valid ? __ldcs(vin + idx) : 0u;
        dg[j] = valid ? digit_of(keys[j], pass) : kRadix;
    }
    rank_tile(dg, rnk, whist);
#pragma unroll
    for (uint32_t j = 0; j < kSortItems; ++j) {
        if (dg[j] == kRadix) continue;
        const uint32_t pos = soff[dg[j]] + whist[warp][dg[j]] + rnk[j];
        kout[pos] = keys[j];
        vout[pos] = vals[j];
    }
}

// ------------------------------------------------------------------------------------------------
// a2: segments of the sorted arcs -> vertex table, ranks / segment ends

struct SegBufs {
    uint32_t *keyA, *valA, *keyB, *valB;
    const uint32_t *hist;
    VSlot *vt;
    uint32_t vmask;
    uint32_t tag;
    uint2 *einfo2;  // [2 wcap]: einfo2[k<<1|side] = {sorted slot, segment end}
    uint32_t *ctr;
};

__device__ __forceinline__ void sorted_bufs(const SegBufs &sb, uint32_t n, const uint32_t *&keys,
                                            const uint32_t *&vals) {
    const bool B = in_buffer_B(sb.hist, kPasses, n);
    keys = B ? sb.keyB : sb.keyA;
    vals = B ? sb.valB : sb.valA;
}

// Insert-or-find v with payload {deg, start}; returns the slot; claimed = this call created the entry.
__device__ __forceinline__ uint32_t vt_insert(VSlot *vt, uint32_t mask, uint32_t tag, uint32_t v, uint32_t deg,
                                              uint32_t start, bool &claimed) {
    uint32_t b = hash_vertex(v) & mask & ~1u;
    claimed = false;
    while (true) {
        const uint4 *p = reinterpret_cast<const uint4 *>(vt + b);
        const uint4 s0 = __ldcg(p), s1 = __ldcg(p + 1);
        const bool l0 = s0.w == tag, l1 = s1.w == tag;
        if (l0 && s0.x == v) return b;
        if (l1 && s1.x == v) return b + 1;
        if (l0 && l1) {
            b = (b + 2) & mask;
            continue;
        }
        const uint32_t e = l0 ? 1u : 0u;
        const uint4 s = e ? s1 : s0;
        const u128 exp = pack4(s.x, s.y, s.z, s.w);
        if (atomicCAS(reinterpret_cast<u128 *>(vt + b + e), exp, pack4(v, deg, start, tag)) == exp) {
            claimed = true;
            return b + e;
        }
    }
}

// One block per tile of kTile sorted arcs (8 consecutive per thread).
__global__ void __launch_bounds__(kSortThreads) k_runs(SegBufs sb, uint32_t n) {
    if (sb.ctr[kCtrErr]) return;
    const uint32_t *keys, *vals;
    sorted_bufs(sb, n, keys, vals);
    __shared__ uint32_t skey_[kTile + 2 + (kTile + 2) / 32 + 1];
    // skewed index (one pad word per 32) so the per-thread contiguous reads below are conflict-free
#define SKEY(i) skey_[(i) + ((i) >> 5)]
    __shared__ uint32_t run_start[kTile], run_end[kTile];
    __shared__ uint32_t wsum[kWarps];
    __shared__ uint32_t nclaim_sh;
    const uint32_t t0 = blockIdx.x * kTile;
    const uint32_t tn = min(kTile, n - t0);
    const uint32_t i0 = threadIdx.x * kRunItems;
    uint32_t myval[kRunItems];
#pragma unroll
    for (uint32_t e = 0; e < kRunItems; ++e) {
        const uint32_t i = i0 + e;
        if (i < tn) {
            SKEY(i + 1) = keys[t0 + i];
            myval[e] = vals[t0 + i];
        }
    }
    if (threadIdx.x == 0) {
        SKEY(0) = t0 > 0 ? keys[t0 - 1] : ~keys[t0];                       // halo: previous arc's key
        SKEY(tn + 1) = t0 + tn < n ? keys[t0 + tn] : ~keys[t0 + tn - 1];  // halo: next arc's key
        nclaim_sh = 0;
    }
    __syncthreads();
    // local run heads (inside the tile) -> run ids by a block scan
    uint32_t heads = 0;
#pragma unroll
    for (uint32_t e = 0; e < kRunItems; ++e) {
        const uint32_t i = i0 + e;
        if (i < tn && (i == 0 || SKEY(i + 1) != SKEY(i))) ++heads;
    }
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint32_t incl = heads;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= (uint32_t)off) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0, nruns = 0;
    for (uint32_t x = 0; x < kWarps; ++x) {
        if (x < warp) wpre += wsum[x];
        nruns += wsum[x];
    }
    uint32_t rid[kRunItems];
    {
        uint32_t r = wpre + incl - heads;  // runs started before this thread's first arc
#pragma unroll
        for (uint32_t e = 0; e < kRunItems; ++e) {
            const uint32_t i = i0 + e;
            if (i < tn && (i == 0 || SKEY(i + 1) != SKEY(i))) {
                run_start[r] = i;
                ++r;
            }
            rid[e] = r - 1;
            if (i < tn && (i + 1 == tn || SKEY(i + 2) != SKEY(i + 1))) run_end[r - 1] = i + 1;
        }
    }
    __syncthreads();
    // one thread per run: vertex table entry (whole segment in one CAS; split segments by atomics)
    uint32_t claims = 0;
    for (uint32_t r = threadIdx.x; r < nruns; r += kSortThreads) {
        const uint32_t s = run_start[r], e = run_end[r];
        const uint32_t v = SKEY(s + 1);
        const bool whole = SKEY(s) != v && SKEY(e + 1) != v;  // the segment starts and ends in this tile
        bool claimed;
        const uint32_t slot =
            vt_insert(sb.vt, sb.vmask, sb.tag, v, whole ? e - s : 0u, whole ? t0 + s : 0xFFFFFFFFu, claimed);
        if (!whole) {
            atomicAdd(&sb.vt[slot].deg, e - s);
            atomicMin(&sb.vt[slot].start, t0 + s);
            run_end[r] = 0;  // the segment crosses the tile: k_fix writes its arcs' einfo
        }
        claims += claimed ? 1u : 0u;
    }
    if (claims) atomicAdd(&nclaim_sh, claims);
    __syncthreads();
    if (threadIdx.x == 0 && nclaim_sh) atomicAdd(&sb.ctr[kCtrD], nclaim_sh);
    // arcs of tile-internal segments: einfo = {sorted slot, segment end}
#pragma unroll
    for (uint32_t e = 0; e < kRunItems; ++e) {
        const uint32_t i = i0 + e;
        if (i < tn) {
            const uint32_t end = run_end[rid[e]];
            if (end) sb.einfo2[myval[e]] = make_uint2(t0 + i, t0 + end);
        }
    }
}
#undef SKEY

// Arcs of segments that cross tile boundaries (at most the first and the last segment of a tile).
__global__ void __launch_bounds__(kSortThreads) k_fix(SegBufs sb, uint32_t n) {
    if (sb.ctr[kCtrErr]) return;
    const uint32_t *keys, *vals;
    sorted_bufs(sb, n, keys, vals);
    __shared__ uint2 seg[2];
    const uint32_t t0 = blockIdx.x * kTile;
    const uint32_t t1 = min(t0 + kTile, n);
    if (threadIdx.x < 2) {
        const uint32_t v = keys[threadIdx.x == 0 ? t0 : t1 - 1];
        const uint2 inf = vt_find(sb.vt, sb.vmask, sb.tag, v);  // {deg, start}
        seg[threadIdx.x] = make_uint2(inf.y, inf.y + inf.x);
    }
    __syncthreads();
    for (uint32_t q = 0; q < 2; ++q) {
        const uint2 sgm = seg[q];
        if (sgm.x >= t0 && sgm.y <= t1) continue;   // tile-internal: done by k_runs
        if (q == 1 && seg[0].x == sgm.x) continue;  // same segment as q == 0
        const uint32_t lo = max(sgm.x, t0), hi = min(sgm.y, t1);
        for (uint32_t i = lo + threadIdx.x; i < hi; i += kSortThreads) sb.einfo2[vals[i]] = make_uint2(i, sgm.y);
    }
}

// ------------------------------------------------------------------------------------------------
// a4..a8: the fused estimator update, one thread per estimator.

struct UpdateIdx {
    const uint2 *E;
    const uint4 *einfo;
    const VSlot *vt;
    uint32_t vmask;
    const uint32_t *valA, *valB;  // the sorted arc values (segS) live in one of them
    const uint32_t *hist;
    const PSlot *pt;
    uint32_t pmask;
    uint32_t tag;
    const uint32_t *ctr;
};

__global__ void __launch_bounds__(256, 4) k_update(uint2 *__restrict__ r1s, uint2 *__restrict__ r2s,
                                                   uint32_t *__restrict__ cfs, uint64_t *__restrict__ p1s,
                                                   uint64_t *__restrict__ p2s, uint64_t count, uint64_t first,
                                                   uint64_t seed, uint32_t batch, uint64_t m_prev, uint32_t w,
                                                   UpdateIdx ix, unsigned long long *S, unsigned long long *stats) {
    if (ix.ctr[kCtrErr]) return;
    const uint32_t *__restrict__ segS = in_buffer_B(ix.hist, kPasses, 2 * w) ? ix.valB : ix.valA;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long contrib = 0;
    uint32_t n_fresh = 0, n_r2old = 0;
    if (t < count) {
        const uint64_t gid = first + t;
        const DrawCtx dc{gid, batch, PhiloxKey{(uint32_t)seed, (uint32_t)(seed >> 32)}};
        const uint4 o = philox4x32_10(make_uint4((uint32_t)gid, (uint32_t)(gid >> 32), batch, 0u), dc.key);
        const uint64_t xlo = (uint64_t)o.x | ((uint64_t)o.y << 32);
        const uint64_t xhi = (uint64_t)o.z | ((uint64_t)o.w << 32);

        // ---- Step 1: level-1 reservoir ----
        const uint64_t d1 = bounded(m_prev + w, xlo, dc, 0x10000u);
        const bool fresh = d1 >= m_prev;
        uint2 r1, r2 = make_uint2(kEmptyV, kEmptyV);
        uint32_t c, cf_old = 0;
        bool closed;
        uint32_t ld, rd, endU, endV;
        if (fresh) {
            const uint32_t j = (uint32_t)(d1 - m_prev);
            r1 = __ldg(ix.E + j);
            c = 0;
            closed = false;
            // ---- Step 2a for a fresh f1 = w_j: ld = rank(u->v), rd = rank(v->u) ----
            const uint4 inf = __ldg(ix.einfo + j);
            ld = inf.y - 1u - inf.x;
            rd = inf.w - 1u - inf.z;
            endU = inf.y;
            endV = inf.w;
        } else {
            r1 = __ldcs(r1s + t);
            cf_old = __ldcs(cfs + t);
            r2 = __ldcs(r2s + t);  // issued early: needed by Step 3 when f2 is kept
            c = cf_old & kCMask;
            closed = (cf_old & kClosedBit) != 0;
            // ---- Step 2a for a retained f1: rank(u->v) = deg_W(u) (footnote PAPER.md:818-821) ----
            uint2 iu, iv;
            vt_find2(ix.vt, ix.vmask, ix.tag, r1.x, r1.y, iu, iv);
            ld = iu.x;
            rd = iv.x;
            endU = iu.y + iu.x;
            endV = iv.y + iv.x;
        }
        const uint32_t chi_p = ld + rd;  // |Gamma_W(f1)| = rank(u->v) + rank(v->u)
        bool r2new = false;
        uint32_t k2 = 0;
        const bool had_r2 = !fresh && c > 0;  // NBSI: chi == 0 <=> f2 empty
        if (chi_p) {
            // ---- Step 2b: keep f2 w.p. chi^-/(chi^-+chi^+), else phi names an edge ----
            const uint64_t d2 = bounded((uint64_t)c + chi_p, xhi, dc, 0x20000u);
            if (d2 >= c) {
                const uint32_t phi = (uint32_t)(d2 - c);
                const uint32_t end = phi < ld ? endU : endV;
                const uint32_t a = phi < ld ? phi : phi - ld;
                const uint32_t val = __ldg(segS + (end - 1u - a));
                k2 = val >> 1;
                r2 = __ldg(ix.E + k2);
                r2new = true;
                closed = false;
            }
            c += chi_p;
        }
        // ---- Step 3: closing edge after f2 ----
        if ((r2new || had_r2) && !closed) {
            const uint32_t x = (r1.x == r2.x || r1.x == r2.y) ? r1.y : r1.x;  // f1's endpoint not on f2
            const uint32_t z = (r2.x == r1.x || r2.x == r1.y) ? r2.y : r2.x;  // f2's endpoint not on f1
            const int64_t kk = pt_find(ix.pt, ix.pmask, ix.tag, pair_key(min(x, z), max(x, z)));
            if (kk >= 0 && (!r2new || (uint32_t)kk > k2)) closed = true;
        }
        const uint32_t cf_new = c | (closed ? kClosedBit : 0u);
        if (fresh || cf_new != cf_old) __stcs(cfs + t, cf_new);
        if (fresh) {
            __stcs(r1s + t, r1);
            __stcs(p1s + t, d1);
        }
        if (r2new) {
            __stcs(r2s + t, r2);
            __stcs(p2s + t, m_prev + k2);
        } else if (fresh) {
            __stcs(r2s + t, make_uint2(kEmptyV, kEmptyV));
            __stcs(p2s + t, ~0ull);
        }
        if (closed) contrib = c;
        n_fresh = fresh ? 1u : 0u;
        n_r2old = (r2new && !fresh) ? 1u : 0u;
    }
    // ---- a8: partial sum of chi over closed estimators (+ event counts for the byte model) ----
    n_fresh = __popc(__ballot_sync(0xffffffffu, n_fresh != 0));
    n_r2old = __popc(__ballot_sync(0xffffffffu, n_r2old != 0));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, off);
    __shared__ unsigned long long ws[8];
    __shared__ uint32_t wf[8], wr[8];
    if ((threadIdx.x & 31u) == 0) {
        ws[threadIdx.x >> 5] = contrib;
        wf[threadIdx.x >> 5] = n_fresh;
        wr[threadIdx.x >> 5] = n_r2old;
    }
    __syncthreads();
    if (threadIdx.x < 8) {
        unsigned long long v = ws[threadIdx.x];
        uint32_t f = wf[threadIdx.x], q = wr[threadIdx.x];
#pragma unroll
        for (int off = 4; off > 0; off >>= 1) {
            v += __shfl_xor_sync(0xffu, v, off);
            f += __shfl_xor_sync(0xffu, f, off);
            q += __shfl_xor_sync(0xffu, q, off);
        }
        if (threadIdx.x == 0) {
            if (v) atomicAdd(S, v);
            if (f) atomicAdd(stats + 0, (unsigned long long)f);
            if (q) atomicAdd(stats + 1, (unsigned long long)q);
            if (blockIdx.x == 0) {
                atomicAdd(stats + 2, (unsigned long long)ix.ctr[kCtrD]);
                atomicAdd(stats + 3, 1ull);
            }
        }
    }
}

__global__ void k_init_state(uint2 *r1, uint2 *r2, uint32_t *cf, uint64_t *p1, uint64_t *p2, uint64_t count) {
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += (uint64_t)gridDim.x * blockDim.x) {
        r1[t] = make_uint2(kEmptyV, kEmptyV);
        r2[t] = make_uint2(kEmptyV, kEmptyV);
        cf[t] = 0;
        p1[t] = ~0ull;
        p2[t] = ~0ull;
    }
}

// S_g over contiguous groups g = [floor(g n / G), floor((g+1) n / G)).
__global__ void k_group_sums(const uint32_t *__restrict__ cf, uint64_t n, uint32_t G, unsigned long long *out) {
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = cf[t];
        if (!(v & kClosedBit)) continue;
        const uint64_t g = ((t + 1) * G + n - 1) / n - 1;
        atomicAdd(out + g, (unsigned long long)(v & kCMask));
    }
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

static inline uint32_t grid_for(uint64_t items, uint32_t threads, uint32_t per_sm) {
    const uint64_t want = (items + threads - 1) / threads;
    const uint64_t cap = (uint64_t)sm_count() * per_sm;
    return (uint32_t)std::max<uint64_t>(1, std::min(want, cap));
}

static inline uint32_t radix_tiles(uint32_t w) { return (2 * w + kRadixTile - 1) / kRadixTile; }

int launch_stage(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s) {
    const uint32_t nt = radix_tiles(a.w);
    k_hist<<<nt, kSortThreads, 0, s>>>(a.in, a.w, ix.hist, ix.cnt, nt, ix.ctr);
    k_scan<<<kRadix, kSortThreads, 0, s>>>(ix.cnt, nt, ix.hist, 0, 2 * a.w, ix.ctr);
    StageCtx c{ix.E, ix.keyB, ix.valB, ix.cnt, ix.hist, nt, ix.pt, ix.pmask, a.tag, ix.ctr};
    k_stage<<<nt, kSortThreads, 0, s>>>(a.in, a.w, c);
    return 3;
}

int launch_pairs(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s) {
    const uint32_t nt = radix_tiles(a.w);
    StageCtx c{ix.E, ix.keyB, ix.valB, ix.cnt, ix.hist, nt, ix.pt, ix.pmask, a.tag, ix.ctr};
    k_pairs<<<(a.w + 255) / 256, 256, 0, s>>>(a.in, a.w, c);
    return 1;
}

int launch_sort(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s) {
    const uint32_t n = 2 * a.w, nt = radix_tiles(a.w);
    for (uint32_t p = 1; p < kPasses; ++p) {
        k_upsweep<<<nt, kSortThreads, 0, s>>>(ix.keyA, ix.keyB, n, ix.hist, p, ix.cnt, nt, ix.ctr);
        k_scan<<<kRadix, kSortThreads, 0, s>>>(ix.cnt, nt, ix.hist, p, n, ix.ctr);
        k_downsweep<<<nt, kSortThreads, 0, s>>>(ix.keyA, ix.valA, ix.keyB, ix.valB, n, ix.hist, p, ix.cnt, nt, ix.ctr);
    }
    return 3 * (int)(kPasses - 1);
}

int launch_segment(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s) {
    const uint32_t n = 2 * a.w;
    const uint32_t tiles = (n + kTile - 1) / kTile;
    SegBufs sb{ix.keyA, ix.valA, ix.keyB, ix.valB, ix.hist, ix.vt, ix.vmask, a.tag,
               reinterpret_cast<uint2 *>(ix.einfo), ix.ctr};
    k_runs<<<tiles, kSortThreads, 0, s>>>(sb, n);
    k_fix<<<tiles, kSortThreads, 0, s>>>(sb, n);
    return 2;
}

int launch_update(const IndexBufs &ix, const StateBufs &st, const BatchArgs &a, cudaStream_t s) {
    if (st.count == 0) return 0;
    const uint64_t blocks = (st.count + 255) / 256;
    UpdateIdx u{ix.E, ix.einfo, ix.vt, ix.vmask, ix.valA, ix.valB, ix.hist, ix.pt, ix.pmask, a.tag, ix.ctr};
    k_update<<<(uint32_t)blocks, 256, 0, s>>>(st.r1, st.r2, st.cf, st.p1, st.p2, st.count, a.first, a.seed, a.batch,
                                              a.m_prev, a.w, u, st.S + a.S_slot, st.stats);
    return 1;
}

int launch_init_tables(const IndexBufs &ix, cudaStream_t s) {
    // tag 0 marks every slot free (live tags start at 1)
    cudaMemsetAsync(ix.vt, 0, 16ull * ((uint64_t)ix.vmask + 1), s);
    cudaMemsetAsync(ix.pt, 0, 16ull * ((uint64_t)ix.pmask + 1), s);
    return 0;
}

int launch_init_state(const StateBufs &st, cudaStream_t s) {
    if (!st.count) return 0;
    k_init_state<<<grid_for(st.count, 256, 16), 256, 0, s>>>(st.r1, st.r2, st.cf, st.p1, st.p2, st.count);
    return 1;
}

int launch_group_sums(const StateBufs &st, uint32_t groups, unsigned long long *out, cudaStream_t s) {
    if (!st.count) return 0;
    k_group_sums<<<grid_for(st.count, 256, 16), 256, 0, s>>>(st.cf, st.count, groups, out);
    return 1;
}

}  // namespace tcb

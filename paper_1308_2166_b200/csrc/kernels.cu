// kernels.cu -- the per-batch hot path of bulkUpdateAll on sm_100a.
//
// Pipeline for one batch W:
//   k_stage      a1 + a3 : load W (16-byte loads = 2 edges), validate, normalize to (lo, hi); emit the 2|W|
//                          arcs (vertex, k<<1|side) in arrival order -- the F array of rankAll's proof
//                           -- and their 8-bit digit histograms; insert the edge into
//                          the edge-pair hash (one CAS round trip per probe; a repeat is TC_EDUP)
//   k_radix_pass a2      : stable LSD radix pass over the arcs by vertex id (one kernel per 8-bit digit,
//                          single sweep with decoupled look-back; passes whose digit is zero for every
//                          arc are skipped on the device).  Stability keeps arrival order inside a vertex:
//                          this replaces rankAll's sort by (src, -pos).
//   k_runs       a2      : runs of equal vertex inside each tile -> vertex table {deg_W, segment start};
//                          ranks/segment ends of the arcs of tile-internal segments
//   k_fix        a2      : ranks/segment ends of the arcs of segments that cross tile boundaries
//   k_update     a4..a8  : ONE pass over the estimator SoA: Step 1 (level-1 reservoir), Step 2 (chi^+
//                          from ranks / degrees, level-2 pick by segment arithmetic), Step 3 (closing-edge
//                          probe), block partial sums of chi over closed estimators
//   k_clear              : empties exactly the table slots this batch used
// rank(x->y) of the arc at sorted slot s = segEnd(x) - 1 - s (Definition Rank).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "index.cuh"
#include "kernels.h"
#include "philox.cuh"

namespace tcb {

// ------------------------------------------------------------------------------------------------
// a1 + a3: staging, arcs, digit histograms, edge-pair hash

struct StageCtx {
    uint2 *E;
    uint32_t *key, *val;  // arcs out (radix buffer A)
    uint32_t *hist;       // [kPasses][kRadix]
    PSlot *pt;
    uint32_t pmask;
    uint32_t *pslot;
    uint32_t *ctr;
};

// An in-flight edge-pair insert (lo, hi) -> k.
struct PIns {
    unsigned long long key;
    uint32_t b, k;
    bool armed, done, dup;
};

// One probe step: read the 2-slot bucket (one sector), CAS the first free key if the pair is absent.
__device__ __forceinline__ void pins_step(const StageCtx &c, PIns &s) {
    const ulonglong2 *p = reinterpret_cast<const ulonglong2 *>(c.pt + s.b);
    const ulonglong2 s0 = __ldcg(p), s1 = __ldcg(p + 1);
    if (s0.x == s.key || s1.x == s.key) {
        s.done = s.dup = true;
        return;
    }
    const uint32_t e = s0.x == kEmptyP ? 0u : s1.x == kEmptyP ? 1u : 2u;
    if (e == 2u) {
        s.b = (s.b + 2) & c.pmask;
        return;
    }
    const unsigned long long old = atomicCAS(&c.pt[s.b + e].key, kEmptyP, s.key);
    if (old == kEmptyP) {
        s.b += e;
        s.done = true;
    } else if (old == s.key) {
        s.done = s.dup = true;
    }
    // else: another pair took the slot; re-read the bucket
}

// Validate + normalize one edge, emit its arcs and digit counts, arm its pair insert; returns error bits.
__device__ __forceinline__ uint32_t stage_edge(const StageCtx &c, uint2 e, uint32_t k, uint32_t (*sh)[kRadix],
                                               PIns &q) {
    q.k = k;
    q.armed = false;
    q.done = true;
    q.dup = false;
    if (e.x == kEmptyV || e.y == kEmptyV || e.x == e.y) {
        c.pslot[k] = kNoSlot;
        return (e.x == kEmptyV || e.y == kEmptyV) ? kErrInval : kErrLoop;
    }
    const uint32_t lo = min(e.x, e.y), hi = max(e.x, e.y);
    c.E[k] = make_uint2(lo, hi);
    reinterpret_cast<uint2 *>(c.key)[k] = make_uint2(lo, hi);
    reinterpret_cast<uint2 *>(c.val)[k] = make_uint2(k << 1, (k << 1) | 1u);
#pragma unroll
    for (uint32_t p = 0; p < kPasses; ++p) {
        atomicAdd(&sh[p][(lo >> (p * kRadixBits)) & (kRadix - 1)], 1u);
        atomicAdd(&sh[p][(hi >> (p * kRadixBits)) & (kRadix - 1)], 1u);
    }
    q.key = pair_key(lo, hi);
    q.b = hash_pair(q.key) & c.pmask & ~1u;
    q.armed = true;
    q.done = false;
    return 0u;
}

__device__ __forceinline__ uint32_t pins_finish(const StageCtx &c, const PIns &q) {
    if (!q.armed) return 0u;
    if (q.dup) {
        c.pslot[q.k] = kNoSlot;
        return kErrDup;
    }
    c.pt[q.b].pos = q.k;
    c.pslot[q.k] = q.b;
    return 0u;
}

__global__ void __launch_bounds__(256) k_stage(const uint2 *__restrict__ in, uint32_t w, StageCtx c) {
    if (c.ctr[kCtrErr] & (kErrInval | kErrLoop | kErrDup)) return;  // sticky error of an earlier async batch
    __shared__ uint32_t sh[kPasses][kRadix];
    for (uint32_t i = threadIdx.x; i < kPasses * kRadix; i += blockDim.x) (&sh[0][0])[i] = 0;
    __syncthreads();
    uint32_t bad = 0;
    const uint32_t stride = gridDim.x * blockDim.x;
    const bool vec = (reinterpret_cast<uintptr_t>(in) & 15u) == 0;
    const uint4 *in4 = reinterpret_cast<const uint4 *>(in);
    // two edges per thread per iteration; their hash inserts are stepped together (2 round trips in flight)
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; 2 * q < w; q += stride) {
        const bool has1 = 2 * q + 1 < w;
        uint2 e0, e1 = make_uint2(0u, 0u);
        if (vec && has1) {
            const uint4 two = __ldcs(in4 + q);
            e0 = make_uint2(two.x, two.y);
            e1 = make_uint2(two.z, two.w);
        } else {
            e0 = in[2 * q];
            if (has1) e1 = in[2 * q + 1];
        }
        PIns a, b;
        bad |= stage_edge(c, e0, 2 * q, sh, a);
        b.armed = false;
        b.done = true;
        b.dup = false;
        if (has1) bad |= stage_edge(c, e1, 2 * q + 1, sh, b);
        while (!(a.done && b.done)) {
            if (!a.done) pins_step(c, a);
            if (!b.done) pins_step(c, b);
        }
        bad |= pins_finish(c, a);
        bad |= pins_finish(c, b);
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (bad && (threadIdx.x & 31u) == 0) atomicOr(&c.ctr[kCtrErr], bad);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < kPasses * kRadix; i += blockDim.x) {
        const uint32_t v = (&sh[0][0])[i];
        if (v) atomicAdd(c.hist + i, v);
    }
}

// ------------------------------------------------------------------------------------------------
// a2: stable LSD radix sort of the arcs by vertex id

// A pass is trivial (identity) when every arc has digit 0; the ping-pong parity counts executed passes.
__device__ __forceinline__ bool pass_trivial(const uint32_t *hist, uint32_t p, uint32_t n) {
    return hist[p * kRadix] == n;
}
__device__ __forceinline__ uint32_t passes_executed(const uint32_t *hist, uint32_t upto, uint32_t n) {
    uint32_t e = 0;
    for (uint32_t p = 0; p < upto; ++p) e += pass_trivial(hist, p, n) ? 0u : 1u;
    return e;
}

struct RadixBufs {
    uint32_t *keyA, *valA, *keyB, *valB;
    const uint32_t *hist;
    unsigned long long *look;
    uint32_t *ctr;
};

constexpr unsigned long long kFlagAgg = 1ull, kFlagPrefix = 2ull;

__global__ void __launch_bounds__(kSortThreads) k_radix_pass(RadixBufs rb, uint32_t n, uint32_t pass, uint32_t seq) {
    if (rb.ctr[kCtrErr]) return;
    if (pass_trivial(rb.hist, pass, n)) return;
    const bool odd = passes_executed(rb.hist, pass, n) & 1u;
    const uint32_t *__restrict__ kin = odd ? rb.keyB : rb.keyA;
    const uint32_t *__restrict__ vin = odd ? rb.valB : rb.valA;
    uint32_t *__restrict__ kout = odd ? rb.keyA : rb.keyB;
    uint32_t *__restrict__ vout = odd ? rb.valA : rb.valB;
    const uint32_t shift = pass * kRadixBits;

    __shared__ uint32_t whist[kSortThreads / 32][kRadix];  // per-warp digit counts -> warp offsets
    __shared__ uint32_t gofs[kRadix];                      // global start of each digit for this tile
    __shared__ uint32_t ws[kSortThreads / 32];
    __shared__ uint32_t tile_sh;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    for (uint32_t i = threadIdx.x; i < (kSortThreads / 32) * kRadix; i += kSortThreads) (&whist[0][0])[i] = 0;
    if (threadIdx.x == 0) tile_sh = atomicAdd(&rb.ctr[kCtrTile + pass], 1u);  // dynamic tile order
    __syncthreads();
    const uint32_t tile = tile_sh;
    const uint32_t wbase = tile * kRadixTile + warp * (32 * kSortItems);

    // stable in-tile ranks: warp w owns a contiguous 256-arc range, processed in 8 rounds of 32
    uint32_t keys[kSortItems], vals[kSortItems], rnk[kSortItems];
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (uint32_t j = 0; j < kSortItems; ++j) {
        const uint32_t idx = wbase + j * 32 + lane;
        const bool valid = idx < n;
        keys[j] = valid ? __ldcs(kin + idx) : 0u;
        vals[j] = valid ? __ldcs(vin + idx) : 0u;
    }
#pragma unroll
    for (uint32_t j = 0; j < kSortItems; ++j) {
        const bool valid = wbase + j * 32 + lane < n;
        const uint32_t d = valid ? (keys[j] >> shift) & (kRadix - 1) : kRadix;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t before = __popc(peers & lt);
        uint32_t b = 0;
        if (valid) b = whist[warp][d];
        __syncwarp();
        if (valid && before == 0) whist[warp][d] = b + __popc(peers);
        __syncwarp();
        rnk[j] = b + before;
    }
    __syncthreads();
    // per digit: exclusive prefix over warps (warp order == arc order), tile total
    const uint32_t dgt = threadIdx.x;  // kSortThreads == kRadix
    uint32_t total = 0;
#pragma unroll
    for (uint32_t x = 0; x < kSortThreads / 32; ++x) {
        const uint32_t cnt = whist[x][dgt];
        whist[x][dgt] = total;
        total += cnt;
    }
    // decoupled look-back over earlier tiles for this digit
    unsigned long long *lk = rb.look + (size_t)tile * kRadix + dgt;
    const unsigned long long tag = (unsigned long long)seq << 2;
    uint32_t excl = 0;
    if (tile == 0) {
        atomicExch(lk, ((tag | kFlagPrefix) << 32) | total);
    } else {
        atomicExch(lk, ((tag | kFlagAgg) << 32) | total);
        // walk back in windows of 8 predecessors (8 independent loads in flight)
        bool found = false;
        for (int32_t t = (int32_t)tile - 1; t >= 0 && !found; t -= 8) {
            unsigned long long v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                v[u] = t - u >= 0 ? *(const volatile unsigned long long *)(rb.look + (size_t)(t - u) * kRadix + dgt) : 0ull;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (found || t - u < 0) break;
                while ((v[u] >> 34) != seq || ((v[u] >> 32) & 3ull) == 0ull)
                    v[u] = *(const volatile unsigned long long *)(rb.look + (size_t)(t - u) * kRadix + dgt);
                excl += (uint32_t)v[u];
                found = ((v[u] >> 32) & 3ull) == kFlagPrefix;
            }
        }
        atomicExch(lk, ((tag | kFlagPrefix) << 32) | (excl + total));
    }
    // global digit offset: exclusive scan of this pass's histogram (digit order)
    const uint32_t h = rb.hist[pass * kRadix + dgt];
    uint32_t incl = h;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= (uint32_t)off) incl += y;
    }
    if (lane == 31) ws[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0;
    for (uint32_t x = 0; x < warp; ++x) wpre += ws[x];
    gofs[dgt] = wpre + incl - h + excl;
    __syncthreads();
#pragma unroll
    for (uint32_t j = 0; j < kSortItems; ++j) {
        const uint32_t idx = wbase + j * 32 + lane;
        if (idx < n) {
            const uint32_t d = (keys[j] >> shift) & (kRadix - 1);
            const uint32_t pos = gofs[d] + whist[warp][d] + rnk[j];
            kout[pos] = keys[j];
            vout[pos] = vals[j];
        }
    }
}

// ------------------------------------------------------------------------------------------------
// a2: segments of the sorted arcs -> vertex table, ranks / segment ends

struct SegBufs {
    uint32_t *keyA, *valA, *keyB, *valB;
    const uint32_t *hist;
    VSlot *vt;
    uint32_t vmask;
    uint2 *einfo2;  // [2 wcap]: einfo2[k<<1|side] = {sorted slot, segment end}
    uint32_t *vlist;
    uint32_t *ctr;
};

__device__ __forceinline__ void sorted_bufs(const SegBufs &sb, uint32_t n, const uint32_t *&keys,
                                            const uint32_t *&vals) {
    const bool odd = passes_executed(sb.hist, kPasses, n) & 1u;
    keys = odd ? sb.keyB : sb.keyA;
    vals = odd ? sb.valB : sb.valA;
}

// Insert-or-find v; returns the slot, sets claimed when this call created it.
__device__ __forceinline__ uint32_t vt_insert(VSlot *vt, uint32_t mask, uint32_t v, bool &claimed) {
    uint32_t b = hash_vertex(v) & mask & ~1u;
    claimed = false;
    while (true) {
        const uint4 *p = reinterpret_cast<const uint4 *>(vt + b);
        const uint4 s0 = __ldcg(p), s1 = __ldcg(p + 1);
        if (s0.x == v) return b;
        if (s1.x == v) return b + 1;
        const uint32_t e = s0.x == kEmptyV ? 0u : s1.x == kEmptyV ? 1u : 2u;
        if (e == 2u) {
            b = (b + 2) & mask;
            continue;
        }
        const uint32_t old = atomicCAS(&vt[b + e].key, kEmptyV, v);
        if (old == kEmptyV) {
            claimed = true;
            return b + e;
        }
        if (old == v) return b + e;
    }
}

// One block per tile of kTile sorted arcs (8 consecutive per thread).
__global__ void __launch_bounds__(kSortThreads) k_runs(SegBufs sb, uint32_t n) {
    if (sb.ctr[kCtrErr]) return;
    const uint32_t *keys, *vals;
    sorted_bufs(sb, n, keys, vals);
    __shared__ uint32_t skey[kTile + 2];
    __shared__ uint32_t run_start[kTile], run_end[kTile];
    __shared__ uint32_t wsum[kSortThreads / 32];
    __shared__ uint32_t nclaim_sh, claim_base;
    const uint32_t t0 = blockIdx.x * kTile;
    const uint32_t tn = min(kTile, n - t0);
    for (uint32_t i = threadIdx.x; i < tn; i += kSortThreads) skey[i + 1] = keys[t0 + i];
    if (threadIdx.x == 0) {
        skey[0] = t0 > 0 ? keys[t0 - 1] : ~keys[t0];                       // halo: previous arc's key
        skey[tn + 1] = t0 + tn < n ? keys[t0 + tn] : ~keys[t0 + tn - 1];  // halo: next arc's key
        nclaim_sh = 0;
    }
    __syncthreads();
    // local run heads (inside the tile) -> run ids by a block scan
    const uint32_t i0 = threadIdx.x * kRunItems;
    uint32_t heads = 0;
#pragma unroll
    for (uint32_t e = 0; e < kRunItems; ++e) {
        const uint32_t i = i0 + e;
        if (i < tn && (i == 0 || skey[i + 1] != skey[i])) ++heads;
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
    for (uint32_t x = 0; x < kSortThreads / 32; ++x) {
        if (x < warp) wpre += wsum[x];
        nruns += wsum[x];
    }
    uint32_t rid[kRunItems];
    {
        uint32_t r = wpre + incl - heads;  // runs started before this thread's first arc
#pragma unroll
        for (uint32_t e = 0; e < kRunItems; ++e) {
            const uint32_t i = i0 + e;
            if (i < tn && (i == 0 || skey[i + 1] != skey[i])) {
                run_start[r] = i;
                ++r;
            }
            rid[e] = r - 1;
            if (i < tn && (i + 1 == tn || skey[i + 2] != skey[i + 1])) run_end[r - 1] = i + 1;
        }
    }
    __syncthreads();
    // one thread per run: vertex table (complete segments by plain stores, split ones by atomics)
    for (uint32_t r = threadIdx.x; r < nruns; r += kSortThreads) {
        const uint32_t s = run_start[r], e = run_end[r];
        const uint32_t v = skey[s + 1];
        const bool ghead = skey[s] != v;      // the segment starts in this tile
        const bool gtail = skey[e + 1] != v;  // ... and ends in it
        bool claimed;
        const uint32_t slot = vt_insert(sb.vt, sb.vmask, v, claimed);
        if (ghead && gtail) {
            sb.vt[slot].deg = e - s;
            sb.vt[slot].start = t0 + s;
        } else {
            atomicAdd(&sb.vt[slot].deg, e - s);
            atomicMin(&sb.vt[slot].start, t0 + s);
            run_end[r] = 0;  // the segment crosses the tile: k_fix writes its arcs' einfo
        }
        run_start[r] = claimed ? (slot | 0x80000000u) : 0u;
        if (claimed) atomicAdd(&nclaim_sh, 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        claim_base = nclaim_sh ? atomicAdd(&sb.ctr[kCtrD], nclaim_sh) : 0u;
        nclaim_sh = 0;
    }
    __syncthreads();
    // compact the claimed slots into vlist (order inside a tile is irrelevant)
    for (uint32_t r = threadIdx.x; r < nruns; r += kSortThreads) {
        if (run_start[r] & 0x80000000u) sb.vlist[claim_base + atomicAdd(&nclaim_sh, 1u)] = run_start[r] & 0x7FFFFFFFu;
    }
    // arcs of tile-internal segments: einfo = {sorted slot, segment end}
#pragma unroll
    for (uint32_t e = 0; e < kRunItems; ++e) {
        const uint32_t i = i0 + e;
        if (i < tn) {
            const uint32_t end = run_end[rid[e]];
            if (end) sb.einfo2[vals[t0 + i]] = make_uint2(t0 + i, t0 + end);
        }
    }
}

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
        const uint2 inf = vt_find(sb.vt, sb.vmask, v);  // {deg, start}
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
    const uint32_t *ctr;
};

__global__ void __launch_bounds__(256, 4) k_update(uint2 *__restrict__ r1s, uint2 *__restrict__ r2s,
                                                uint32_t *__restrict__ cfs, uint64_t *__restrict__ p1s,
                                                uint64_t *__restrict__ p2s, uint64_t count, uint64_t first,
                                                uint64_t seed, uint32_t batch, uint64_t m_prev, uint32_t w,
                                                UpdateIdx ix, unsigned long long *S, unsigned long long *stats) {
    if (ix.ctr[kCtrErr]) return;
    const uint32_t *__restrict__ segS = (passes_executed(ix.hist, kPasses, 2 * w) & 1u) ? ix.valB : ix.valA;
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
            const uint2 iu = vt_find(ix.vt, ix.vmask, r1.x);
            const uint2 iv = vt_find(ix.vt, ix.vmask, r1.y);
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
            const int64_t kk = pt_find(ix.pt, ix.pmask, pair_key(min(x, z), max(x, z)));
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

// Empty exactly the table slots this batch used (runs even when the batch was rejected).  Four
// independent index loads per thread before the scattered stores.
__global__ void __launch_bounds__(256) k_clear(VSlot *__restrict__ vt, const uint32_t *__restrict__ vlist,
                                               PSlot *__restrict__ pt, const uint32_t *__restrict__ pslot, uint32_t w,
                                               const uint32_t *ctr) {
    const uint32_t D = ctr[kCtrD];
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < D; i += 4 * stride) {
        uint32_t s[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) s[u] = i + u * stride < D ? __ldcs(vlist + i + u * stride) : kNoSlot;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (s[u] != kNoSlot) reinterpret_cast<uint4 *>(vt)[s[u]] = make_uint4(kEmptyV, 0u, 0xFFFFFFFFu, 0u);
    }
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < w; i += 4 * stride) {
        uint32_t s[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) s[u] = i + u * stride < w ? __ldcs(pslot + i + u * stride) : kNoSlot;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (s[u] != kNoSlot) pt[s[u]].key = kEmptyP;
    }
}

__global__ void k_init_tables(VSlot *vt, uint64_t vn, PSlot *pt, uint64_t pn) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < max(vn, pn);
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (i < vn) reinterpret_cast<uint4 *>(vt)[i] = make_uint4(kEmptyV, 0u, 0xFFFFFFFFu, 0u);
        if (i < pn) {
            pt[i].key = kEmptyP;
            pt[i].pos = 0;
            pt[i].pad = 0;
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

int launch_stage(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s) {
    StageCtx c{ix.E, ix.keyA, ix.valA, ix.hist, ix.pt, ix.pmask, ix.pslot, ix.ctr};
    k_stage<<<grid_for((a.w + 1) / 2, 256, 8), 256, 0, s>>>(a.in, a.w, c);
    return 1;
}

int launch_sort(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s) {
    const uint32_t n = 2 * a.w;
    const uint32_t tiles = (n + kRadixTile - 1) / kRadixTile;
    RadixBufs rb{ix.keyA, ix.valA, ix.keyB, ix.valB, ix.hist, ix.look, ix.ctr};
    for (uint32_t p = 0; p < kPasses; ++p) k_radix_pass<<<tiles, kSortThreads, 0, s>>>(rb, n, p, a.seq + p);
    return (int)kPasses;
}

int launch_segment(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s) {
    const uint32_t n = 2 * a.w;
    const uint32_t tiles = (n + kTile - 1) / kTile;
    SegBufs sb{ix.keyA, ix.valA, ix.keyB, ix.valB, ix.hist, ix.vt, ix.vmask,
               reinterpret_cast<uint2 *>(ix.einfo), ix.vlist, ix.ctr};
    k_runs<<<tiles, kSortThreads, 0, s>>>(sb, n);
    k_fix<<<tiles, kSortThreads, 0, s>>>(sb, n);
    return 2;
}

int launch_update(const IndexBufs &ix, const StateBufs &st, const BatchArgs &a, cudaStream_t s) {
    if (st.count == 0) return 0;
    const uint64_t blocks = (st.count + 255) / 256;
    UpdateIdx u{ix.E, ix.einfo, ix.vt, ix.vmask, ix.valA, ix.valB, ix.hist, ix.pt, ix.pmask, ix.ctr};
    k_update<<<(uint32_t)blocks, 256, 0, s>>>(st.r1, st.r2, st.cf, st.p1, st.p2, st.count, a.first, a.seed, a.batch,
                                              a.m_prev, a.w, u, st.S + a.S_slot, st.stats);
    return 1;
}

int launch_clear(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s) {
    k_clear<<<grid_for(2ull * a.w, 256, 8), 256, 0, s>>>(ix.vt, ix.vlist, ix.pt, ix.pslot, a.w, ix.ctr);
    return 1;
}

int launch_init_tables(const IndexBufs &ix, cudaStream_t s) {
    const uint64_t vn = (uint64_t)ix.vmask + 1, pn = (uint64_t)ix.pmask + 1;
    k_init_tables<<<grid_for(std::max(vn, pn), 256, 16), 256, 0, s>>>(ix.vt, vn, ix.pt, pn);
    return 1;
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

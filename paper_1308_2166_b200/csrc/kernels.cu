// kernels.cu -- the per-batch hot path of bulkUpdateAll on sm_100a.
//
// Pipeline for one batch W:
//   k_stage        a1 + a3 : load W (coalesced 16-byte loads = 2 edges), validate, normalize to (lo, hi),
//                            insert both endpoints into the vertex table and the edge into the edge-pair
//                            hash -- one CAS round trip per probe, all three inserts in flight together --
//                            then take an arrival ticket per arc (atomicAdd on deg_W)
//   k_segment      a2      : one contiguous segment per vertex (block scan + one atomic per block); bins
//                            segments by length
//   k_scatter      a2      : every arc to segment start + ticket (unordered inside a segment)
//   k_order_tiny   a2      : segments of <= 16 arcs: one thread, register sorting network
//   k_order_mid    a2      : 17..256 arcs: one warp, shared-memory bitonic network
//   k_sort_chunks  a2      : longer: one block per <= 2048-arc chunk, shared-memory bitonic network
//   k_merge_chunks a2      : segments of > 2048 arcs: final slot = sum of ranks across sorted chunks
//   k_update       a4..a8  : ONE pass over the estimator SoA: Step 1 (level-1 reservoir), Step 2
//                            (chi^+ from ranks / degrees, level-2 pick by segment arithmetic), Step 3
//                            (closing-edge probe), block partial sums of chi over closed estimators
//   k_clear                : empties exactly the table slots this batch used
// After a2 the segment of vertex x holds x's arcs in increasing arrival position, i.e. Fig. 4's
// rankAll order (src asc, pos desc) reversed inside each src group: rank(x->y) = segEnd - 1 - slot.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "index.cuh"
#include "kernels.h"
#include "philox.cuh"

namespace tcb {

// ------------------------------------------------------------------------------------------------
// a1 + a3: staging and table inserts

struct VIns {  // an in-flight vertex insert
    uint32_t v, b, slot;
    bool done, claimed;
};

// One probe step of a vertex insert: reads the 8-key bucket, CASes the first free key if v is absent.
__device__ __forceinline__ void vins_step(uint32_t *vkey, uint32_t mask, VIns &s) {
    const uint4 *p = reinterpret_cast<const uint4 *>(vkey + s.b);
    const uint4 k0 = __ldcg(p), k1 = __ldcg(p + 1);
    int j = match4(k0, s.v);
    if (j < 0) {
        j = match4(k1, s.v);
        if (j >= 0) j += 4;
    }
    if (j >= 0) {
        s.slot = s.b + j;
        s.done = true;
        return;
    }
    int e = match4(k0, kEmptyV);
    if (e < 0) {
        e = match4(k1, kEmptyV);
        if (e >= 0) e += 4;
    }
    if (e < 0) {
        s.b = (s.b + kVBucket) & mask;  // bucket full without v: next bucket
        return;
    }
    const uint32_t old = atomicCAS(vkey + s.b + e, kEmptyV, s.v);
    if (old == kEmptyV || old == s.v) {
        s.slot = s.b + e;
        s.done = true;
        s.claimed = (old == kEmptyV);
    }
    // else: another vertex took that key slot; re-read the same bucket
}

struct PIns {
    unsigned long long key;
    uint32_t b, slot;
    bool done, dup;
};

__device__ __forceinline__ void pins_step(unsigned long long *pkey, uint32_t mask, PIns &s) {
    const ulonglong2 *p = reinterpret_cast<const ulonglong2 *>(pkey + s.b);
    const ulonglong2 a = __ldcg(p), c = __ldcg(p + 1);
    if (a.x == s.key || a.y == s.key || c.x == s.key || c.y == s.key) {
        s.done = true;
        s.dup = true;
        return;
    }
    const int e = a.x == kEmptyP ? 0 : a.y == kEmptyP ? 1 : c.x == kEmptyP ? 2 : c.y == kEmptyP ? 3 : -1;
    if (e < 0) {
        s.b = (s.b + kPBucket) & mask;
        return;
    }
    const unsigned long long old = atomicCAS(pkey + s.b + e, kEmptyP, s.key);
    if (old == kEmptyP) {
        s.slot = s.b + e;
        s.done = true;
    } else if (old == s.key) {
        s.done = true;
        s.dup = true;
    }
}

struct StageCtx {
    uint2 *E;
    uint4 *arcrec;
    uint32_t *pslot;
    uint32_t *vkey;
    uint2 *vinfo;
    uint32_t vmask;
    unsigned long long *pkey;
    uint32_t *ppos;
    uint32_t pmask;
    uint32_t *ctr;
};

__device__ __forceinline__ uint32_t stage_one(const StageCtx &c, uint2 e, uint32_t k) {
    if (e.x == kEmptyV || e.y == kEmptyV || e.x == e.y) {
        c.pslot[k] = kNoSlot;
        return (e.x == kEmptyV || e.y == kEmptyV) ? kErrInval : kErrLoop;
    }
    const uint32_t lo = min(e.x, e.y), hi = max(e.x, e.y);
    c.E[k] = make_uint2(lo, hi);
    VIns a{lo, hash_vertex(lo) & c.vmask & ~(kVBucket - 1), 0, false, false};
    VIns b{hi, hash_vertex(hi) & c.vmask & ~(kVBucket - 1), 0, false, false};
    const unsigned long long key = pair_key(lo, hi);
    PIns q{key, hash_pair(key) & c.pmask & ~(kPBucket - 1), kNoSlot, false, false};
    // the three inserts are independent: step them together so their round trips overlap
    while (!(a.done && b.done && q.done)) {
        if (!a.done) vins_step(c.vkey, c.vmask, a);
        if (!b.done) vins_step(c.vkey, c.vmask, b);
        if (!q.done) pins_step(c.pkey, c.pmask, q);
    }
    // arrival tickets: deg_W counters (two independent atomics)
    const uint32_t ta = atomicAdd(&c.vinfo[a.slot].x, 1u);
    const uint32_t tb = atomicAdd(&c.vinfo[b.slot].x, 1u);
    c.arcrec[k] = make_uint4(a.slot, ta, b.slot, tb);
    c.pslot[k] = q.slot;
    if (!q.dup) c.ppos[q.slot] = k;
    return q.dup ? kErrDup : 0u;
}

__global__ void __launch_bounds__(256) k_stage(const uint2 *__restrict__ in, uint32_t w, StageCtx c) {
    if (c.ctr[3] & (kErrInval | kErrLoop | kErrDup)) return;  // sticky error of an earlier async batch
    uint32_t bad = 0;
    const uint32_t stride = gridDim.x * blockDim.x;
    if ((reinterpret_cast<uintptr_t>(in) & 15u) == 0) {
        const uint32_t npairs = w >> 1;
        const uint4 *in4 = reinterpret_cast<const uint4 *>(in);
        for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < npairs; q += stride) {
            const uint4 two = __ldcs(in4 + q);
            bad |= stage_one(c, make_uint2(two.x, two.y), 2 * q);
            bad |= stage_one(c, make_uint2(two.z, two.w), 2 * q + 1);
        }
        if ((w & 1u) && blockIdx.x * blockDim.x + threadIdx.x == 0) bad |= stage_one(c, in[w - 1], w - 1);
    } else {
        for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < w; k += stride) bad |= stage_one(c, in[k], k);
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (bad && (threadIdx.x & 31u) == 0) atomicOr(&c.ctr[3], bad);
}

// ------------------------------------------------------------------------------------------------
// a2: segments

// Block-wide exclusive scan of a 64-bit value (256 threads); returns the exclusive prefix and sets total.
__device__ __forceinline__ unsigned long long block_scan_u64(unsigned long long v, unsigned long long &total,
                                                             unsigned long long *wsum /* [9] */) {
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    unsigned long long incl = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= (uint32_t)off) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (threadIdx.x < 8) {
        const unsigned long long wv = wsum[threadIdx.x];
        unsigned long long x = wv;
#pragma unroll
        for (int off = 1; off < 8; off <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffu, x, off);
            if (threadIdx.x >= (uint32_t)off) x += y;
        }
        wsum[threadIdx.x] = x - wv;
        if (threadIdx.x == 7) wsum[8] = x;
    }
    __syncthreads();
    total = wsum[8];
    const unsigned long long ex = wsum[warp] + incl - v;
    __syncthreads();
    return ex;
}

// Segment start of every vertex of W (the order of segments is irrelevant, only their contents).
// Walks the vertex table in tiles of 256 x 8 slots: the compact vertex list, the segment starts and
// the length bins (mid list, big-segment chunks) are appended with ONE atomic per tile and counter.
__global__ void __launch_bounds__(256) k_segment(const uint32_t *__restrict__ vkey, uint2 *vinfo, uint32_t nslots,
                                                 uint32_t *__restrict__ vlist, uint32_t *__restrict__ midlist,
                                                 uint4 *__restrict__ chunks, uint32_t *ctr) {
    if (ctr[3]) return;
    __shared__ unsigned long long wsum[9];
    __shared__ uint32_t base[4];
    const uint32_t tile_slots = 256u * kVBucket;
    for (uint32_t t0 = blockIdx.x * tile_slots; t0 < nslots; t0 += gridDim.x * tile_slots) {
        const uint32_t s0 = t0 + threadIdx.x * kVBucket;
        const uint4 *p = reinterpret_cast<const uint4 *>(vkey + s0);
        const uint4 k0 = p[0], k1 = p[1];
        const uint32_t keys[8] = {k0.x, k0.y, k0.z, k0.w, k1.x, k1.y, k1.z, k1.w};
        uint32_t deg[8];
        uint32_t nocc = 0, nmid = 0, degsum = 0, nch = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            deg[i] = keys[i] != kEmptyV ? vinfo[s0 + i].x : 0u;
            nocc += keys[i] != kEmptyV;
            degsum += deg[i];
            nmid += (deg[i] > kTinySeg && deg[i] <= kMidSeg);
            nch += deg[i] > kMidSeg ? (deg[i] + kChunk - 1) / kChunk : 0u;
        }
        unsigned long long tot_a, tot_b;
        const unsigned long long ex_a =
            block_scan_u64(((unsigned long long)degsum << 32) | nocc, tot_a, wsum);  // degsum fits: <= 2w
        const unsigned long long ex_b = block_scan_u64(((unsigned long long)nch << 32) | nmid, tot_b, wsum);
        if (threadIdx.x == 0) {
            base[0] = (uint32_t)tot_a ? atomicAdd(&ctr[0], (uint32_t)tot_a) : 0u;
            base[1] = (uint32_t)(tot_a >> 32) ? atomicAdd(&ctr[1], (uint32_t)(tot_a >> 32)) : 0u;
            base[2] = (uint32_t)tot_b ? atomicAdd(&ctr[4], (uint32_t)tot_b) : 0u;
            base[3] = (uint32_t)(tot_b >> 32) ? atomicAdd(&ctr[2], (uint32_t)(tot_b >> 32)) : 0u;
        }
        __syncthreads();
        uint32_t li = base[0] + (uint32_t)ex_a, st = base[1] + (uint32_t)(ex_a >> 32);
        uint32_t mi = base[2] + (uint32_t)ex_b, ci = base[3] + (uint32_t)(ex_b >> 32);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (keys[i] == kEmptyV) continue;
            const uint32_t s = s0 + i;
            vinfo[s].y = st;
            vlist[li++] = s;
            if (deg[i] > kMidSeg) {
                const uint32_t n = (deg[i] + kChunk - 1) / kChunk;
                for (uint32_t c = 0; c < n; ++c) chunks[ci++] = make_uint4(st, deg[i], c, 0u);
            } else if (deg[i] > kTinySeg) {
                midlist[mi++] = s;
            }
            st += deg[i];
        }
        __syncthreads();
    }
}

// every arc to segment start + ticket
__global__ void __launch_bounds__(256) k_scatter(const uint4 *__restrict__ arcrec, const uint2 *__restrict__ vinfo,
                                                 uint32_t *__restrict__ segU, uint32_t w, const uint32_t *ctr) {
    if (ctr[3]) return;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < w; k += gridDim.x * blockDim.x) {
        const uint4 a = arcrec[k];
        const uint32_t s0 = vinfo[a.x].y, s1 = vinfo[a.z].y;
        segU[s0 + a.y] = k << 1;
        segU[s1 + a.w] = (k << 1) | 1u;
    }
}

__device__ __forceinline__ void cswap(uint32_t &a, uint32_t &b) {
    const uint32_t x = min(a, b), y = max(a, b);
    a = x;
    b = y;
}

// Register bitonic sorter of N (power of two) keys, fully unrolled.
template <int N>
__device__ __forceinline__ void bitonic_regs(uint32_t (&x)[N]) {
#pragma unroll
    for (int size = 2; size <= N; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
#pragma unroll
            for (int i = 0; i < N; ++i) {
                const int j = i ^ stride;
                if (j > i) {
                    if ((i & size) == 0) cswap(x[i], x[j]);
                    else cswap(x[j], x[i]);
                }
            }
        }
    }
}

template <int N>
__device__ __forceinline__ void order_small(const uint32_t *__restrict__ segU, uint32_t *__restrict__ segS,
                                            uint2 *__restrict__ einfo2, uint32_t start, uint32_t deg) {
    uint32_t x[N];
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = (uint32_t)i < deg ? segU[start + i] : 0xFFFFFFFFu;
    bitonic_regs<N>(x);
    const uint32_t end = start + deg;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        if ((uint32_t)i < deg) {
            segS[start + i] = x[i];
            einfo2[x[i]] = make_uint2(start + i, end);
        }
    }
}

// segments of <= kTinySeg arcs: one thread each
__global__ void __launch_bounds__(256) k_order_tiny(const uint32_t *__restrict__ vlist, const uint2 *__restrict__ vinfo,
                                                    const uint32_t *__restrict__ segU, uint32_t *__restrict__ segS,
                                                    uint2 *__restrict__ einfo2, const uint32_t *ctr) {
    if (ctr[3]) return;
    const uint32_t D = ctr[0];
    for (uint32_t d = blockIdx.x * blockDim.x + threadIdx.x; d < D; d += gridDim.x * blockDim.x) {
        const uint2 inf = vinfo[vlist[d]];
        const uint32_t deg = inf.x, start = inf.y;
        if (deg == 1) {
            const uint32_t v = segU[start];
            segS[start] = v;
            einfo2[v] = make_uint2(start, start + 1);
        } else if (deg == 2) {
            uint32_t a = segU[start], b = segU[start + 1];
            cswap(a, b);
            segS[start] = a;
            segS[start + 1] = b;
            einfo2[a] = make_uint2(start, start + 2);
            einfo2[b] = make_uint2(start + 1, start + 2);
        } else if (deg <= 4) {
            order_small<4>(segU, segS, einfo2, start, deg);
        } else if (deg <= 8) {
            order_small<8>(segU, segS, einfo2, start, deg);
        } else if (deg <= kTinySeg) {
            order_small<16>(segU, segS, einfo2, start, deg);
        }
    }
}

// segments of kTinySeg+1 .. kMidSeg arcs: one warp each, bitonic network in shared memory
__global__ void __launch_bounds__(256) k_order_mid(const uint32_t *__restrict__ midlist, const uint2 *__restrict__ vinfo,
                                                   const uint32_t *__restrict__ segU, uint32_t *__restrict__ segS,
                                                   uint2 *__restrict__ einfo2, const uint32_t *ctr) {
    if (ctr[3]) return;
    __shared__ uint32_t sm[8][kMidSeg];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint32_t *s = sm[warp];
    const uint32_t n_mid = ctr[4];
    for (uint32_t q = blockIdx.x * 8u + warp; q < n_mid; q += gridDim.x * 8u) {
        const uint2 inf = vinfo[midlist[q]];
        const uint32_t deg = inf.x, start = inf.y;
        uint32_t P = 32;
        while (P < deg) P <<= 1;
        for (uint32_t i = lane; i < P; i += 32) s[i] = i < deg ? segU[start + i] : 0xFFFFFFFFu;
        __syncwarp();
        for (uint32_t size = 2; size <= P; size <<= 1) {
            for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                for (uint32_t i = lane; i < (P >> 1); i += 32) {
                    const uint32_t lo = 2 * i - (i & (stride - 1));
                    const uint32_t hi = lo + stride;
                    const uint32_t x = s[lo], y = s[hi];
                    if ((x > y) == ((lo & size) == 0)) {
                        s[lo] = y;
                        s[hi] = x;
                    }
                }
                __syncwarp();
            }
        }
        const uint32_t end = start + deg;
        for (uint32_t i = lane; i < deg; i += 32) {
            const uint32_t v = s[i];
            segS[start + i] = v;
            einfo2[v] = make_uint2(start + i, end);
        }
        __syncwarp();
    }
}

// longer segments: sort each chunk of <= kChunk arcs in shared memory (bitonic network)
__global__ void __launch_bounds__(512) k_sort_chunks(const uint4 *__restrict__ chunks, uint32_t *segU,
                                                     uint32_t *__restrict__ segS, uint2 *__restrict__ einfo2,
                                                     const uint32_t *ctr) {
    if (ctr[3]) return;
    __shared__ uint32_t sm[kChunk];
    const uint32_t nch = ctr[2];
    for (uint32_t c = blockIdx.x; c < nch; c += gridDim.x) {
        const uint4 d = chunks[c];
        const uint32_t start = d.x, deg = d.y, ci = d.z;
        const uint32_t base = start + ci * kChunk;
        const uint32_t n = min(kChunk, deg - ci * kChunk);
        uint32_t P = 2;
        while (P < n) P <<= 1;
        for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) sm[i] = i < n ? segU[base + i] : 0xFFFFFFFFu;
        __syncthreads();
        for (uint32_t size = 2; size <= P; size <<= 1) {
            for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                for (uint32_t i = threadIdx.x; i < (P >> 1); i += blockDim.x) {
                    const uint32_t lo = 2 * i - (i & (stride - 1));
                    const uint32_t hi = lo + stride;
                    const uint32_t x = sm[lo], y = sm[hi];
                    if ((x > y) == ((lo & size) == 0)) {
                        sm[lo] = y;
                        sm[hi] = x;
                    }
                }
                __syncthreads();
            }
        }
        if (deg <= kChunk) {
            for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
                const uint32_t v = sm[i];
                segS[start + i] = v;
                einfo2[v] = make_uint2(start + i, start + deg);
            }
        } else {
            for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) segU[base + i] = sm[i];
        }
        __syncthreads();
    }
}

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t *a, uint32_t n, uint32_t v) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(a + mid) < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// segments of > kChunk arcs: merge the sorted chunks by rank (values are distinct)
__global__ void __launch_bounds__(256) k_merge_chunks(const uint4 *__restrict__ chunks, const uint32_t *__restrict__ segU,
                                                      uint32_t *__restrict__ segS, uint2 *__restrict__ einfo2,
                                                      const uint32_t *ctr) {
    if (ctr[3]) return;
    const uint32_t nch = ctr[2];
    for (uint32_t c = blockIdx.x; c < nch; c += gridDim.x) {
        const uint4 d = chunks[c];
        const uint32_t start = d.x, deg = d.y, ci = d.z;
        if (deg <= kChunk) continue;
        const uint32_t nchunks = (deg + kChunk - 1) / kChunk;
        const uint32_t base = start + ci * kChunk;
        const uint32_t n = min(kChunk, deg - ci * kChunk);
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
            const uint32_t v = segU[base + i];
            uint32_t pos = i;
            for (uint32_t cj = 0; cj < nchunks; ++cj) {
                if (cj == ci) continue;
                pos += lower_bound_u32(segU + start + cj * kChunk, min(kChunk, deg - cj * kChunk), v);
            }
            segS[start + pos] = v;
            einfo2[v] = make_uint2(start + pos, start + deg);
        }
    }
}

// ------------------------------------------------------------------------------------------------
// a4..a8: the fused estimator update, one thread per estimator.

struct UpdateIdx {
    const uint2 *E;
    const uint4 *einfo;
    const uint32_t *vkey;
    const uint2 *vinfo;
    uint32_t vmask;
    const uint32_t *segS;
    const unsigned long long *pkey;
    const uint32_t *ppos;
    uint32_t pmask;
    const uint32_t *ctr;
};

__global__ void __launch_bounds__(256) k_update(uint2 *__restrict__ r1s, uint2 *__restrict__ r2s,
                                                uint32_t *__restrict__ cfs, uint64_t *__restrict__ p1s,
                                                uint64_t *__restrict__ p2s, uint64_t count, uint64_t first,
                                                uint64_t seed, uint32_t batch, uint64_t m_prev, uint32_t w,
                                                UpdateIdx ix, unsigned long long *S, unsigned long long *stats) {
    if (ix.ctr[3]) return;
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
        uint2 r1;
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
            c = cf_old & kCMask;
            closed = (cf_old & kClosedBit) != 0;
            // ---- Step 2a for a retained f1: rank(u->v) = deg_W(u) (footnote PAPER.md:818-821) ----
            const uint2 iu = vt_find(ix.vkey, ix.vinfo, ix.vmask, r1.x);
            const uint2 iv = vt_find(ix.vkey, ix.vinfo, ix.vmask, r1.y);
            ld = iu.x;
            rd = iv.x;
            endU = iu.y + iu.x;
            endV = iv.y + iv.x;
        }
        const uint32_t chi_p = ld + rd;  // |Gamma_W(f1)| = rank(u->v) + rank(v->u)
        bool r2new = false;
        uint2 r2 = make_uint2(kEmptyV, kEmptyV);
        uint32_t k2 = 0;
        const bool had_r2 = !fresh && c > 0;  // NBSI: chi == 0 <=> f2 empty
        if (chi_p) {
            // ---- Step 2b: keep f2 w.p. chi^-/(chi^-+chi^+), else phi names an edge ----
            const uint64_t d2 = bounded((uint64_t)c + chi_p, xhi, dc, 0x20000u);
            if (d2 >= c) {
                const uint32_t phi = (uint32_t)(d2 - c);
                const uint32_t end = phi < ld ? endU : endV;
                const uint32_t a = phi < ld ? phi : phi - ld;
                const uint32_t val = __ldg(ix.segS + (end - 1u - a));
                k2 = val >> 1;
                r2 = __ldg(ix.E + k2);
                r2new = true;
                closed = false;
            }
            c += chi_p;
        }
        // ---- Step 3: closing edge after f2 ----
        if ((r2new || had_r2) && !closed) {
            if (!r2new) r2 = __ldcs(r2s + t);
            const uint32_t x = (r1.x == r2.x || r1.x == r2.y) ? r1.y : r1.x;  // f1's endpoint not on f2
            const uint32_t z = (r2.x == r1.x || r2.x == r1.y) ? r2.y : r2.x;  // f2's endpoint not on f1
            const int64_t kk = pt_find(ix.pkey, ix.ppos, ix.pmask, pair_key(min(x, z), max(x, z)));
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
                atomicAdd(stats + 2, (unsigned long long)ix.ctr[0]);
                atomicAdd(stats + 3, 1ull);
            }
        }
    }
}

// Empty exactly the table slots this batch used (runs even when the batch was rejected).
__global__ void __launch_bounds__(256) k_clear(uint32_t *__restrict__ vkey, uint2 *__restrict__ vinfo,
                                               const uint32_t *__restrict__ vlist, unsigned long long *__restrict__ pkey,
                                               const uint32_t *__restrict__ pslot, uint32_t w, const uint32_t *ctr) {
    const uint32_t D = ctr[0];
    const uint32_t n = max(D, w);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (i < D) {
            const uint32_t s = vlist[i];
            vkey[s] = kEmptyV;
            vinfo[s] = make_uint2(0u, 0u);
        }
        if (i < w) {
            const uint32_t s = pslot[i];
            if (s != kNoSlot) pkey[s] = kEmptyP;
        }
    }
}

__global__ void k_init_tables(uint32_t *vkey, uint2 *vinfo, uint64_t vn, unsigned long long *pkey, uint64_t pn) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < max(vn, pn); i += (uint64_t)gridDim.x * blockDim.x) {
        if (i < vn) {
            vkey[i] = kEmptyV;
            vinfo[i] = make_uint2(0u, 0u);
        }
        if (i < pn) pkey[i] = kEmptyP;
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
    StageCtx c{ix.E, ix.arcrec, ix.pslot, ix.vkey, ix.vinfo, ix.vmask, ix.pkey, ix.ppos, ix.pmask, ix.ctr};
    k_stage<<<grid_for((a.w + 1) / 2, 256, 8), 256, 0, s>>>(a.in, a.w, c);
    return 1;
}

int launch_segment(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s) {
    const uint64_t nslots = (uint64_t)ix.vmask + 1;
    k_segment<<<grid_for(nslots / kVBucket, 256, 4), 256, 0, s>>>(ix.vkey, ix.vinfo, (uint32_t)nslots, ix.vlist,
                                                                  ix.midlist, ix.chunks, ix.ctr);
    return 1;
}

int launch_scatter(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s) {
    k_scatter<<<grid_for(a.w, 256, 8), 256, 0, s>>>(ix.arcrec, ix.vinfo, ix.segU, a.w, ix.ctr);
    return 1;
}

int launch_sort(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s) {
    uint2 *einfo2 = reinterpret_cast<uint2 *>(ix.einfo);
    k_order_tiny<<<grid_for(2ull * a.w, 256, 8), 256, 0, s>>>(ix.vlist, ix.vinfo, ix.segU, ix.segS, einfo2, ix.ctr);
    const uint32_t mid_bound = (uint32_t)(2ull * a.w / (kTinySeg + 1) + 1);
    k_order_mid<<<grid_for(mid_bound, 8, 8), 256, 0, s>>>(ix.midlist, ix.vinfo, ix.segU, ix.segS, einfo2, ix.ctr);
    const uint32_t chunk_bound =
        (uint32_t)std::min<uint64_t>(ix.chunk_cap, 2ull * a.w / (kMidSeg + 1) + 2ull * a.w / kChunk + 1);
    const uint32_t g = std::max<uint32_t>(1, std::min<uint32_t>(chunk_bound, sm_count() * 4));
    k_sort_chunks<<<g, 512, 0, s>>>(ix.chunks, ix.segU, ix.segS, einfo2, ix.ctr);
    k_merge_chunks<<<g, 256, 0, s>>>(ix.chunks, ix.segU, ix.segS, einfo2, ix.ctr);
    return 4;
}

int launch_update(const IndexBufs &ix, const StateBufs &st, const BatchArgs &a, cudaStream_t s) {
    if (st.count == 0) return 0;
    const uint64_t blocks = (st.count + 255) / 256;
    UpdateIdx u{ix.E, ix.einfo, ix.vkey, ix.vinfo, ix.vmask, ix.segS, ix.pkey, ix.ppos, ix.pmask, ix.ctr};
    k_update<<<(uint32_t)blocks, 256, 0, s>>>(st.r1, st.r2, st.cf, st.p1, st.p2, st.count, a.first, a.seed, a.batch,
                                              a.m_prev, a.w, u, st.S + a.S_slot, st.stats);
    return 1;
}

int launch_clear(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s) {
    k_clear<<<grid_for(2ull * a.w, 256, 8), 256, 0, s>>>(ix.vkey, ix.vinfo, ix.vlist, ix.pkey, ix.pslot, a.w, ix.ctr);
    return 1;
}

int launch_init_tables(const IndexBufs &ix, cudaStream_t s) {
    const uint64_t vn = (uint64_t)ix.vmask + 1, pn = (uint64_t)ix.pmask + 1;
    k_init_tables<<<grid_for(std::max(vn, pn), 256, 16), 256, 0, s>>>(ix.vkey, ix.vinfo, vn, ix.pkey, pn);
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

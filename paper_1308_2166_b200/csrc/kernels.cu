// kernels.cu -- the per-batch hot path of bulkUpdateAll on sm_100a.
//
// Pipeline for one batch W:
//   k_stage        a1 + a3 : load W (coalesced uint4 = 2 edges), validate, normalize to (lo, hi), insert
//                            both endpoints into the vertex table (deg_W by atomic ticket) and the edge
//                            into the edge-pair hash (128-bit CAS; a repeat is TC_EDUP)
//   k_segment      a2      : one contiguous segment per vertex (block scan + one atomic per block)
//   k_scatter      a2      : place every arc at segment start + its ticket (unordered inside a segment)
//   k_rank_small   a2      : segments of <= 32 arcs: arrival order by counting rank
//   k_sort_chunks  a2      : longer segments: bitonic sort of <= 2048-arc chunks in shared memory
//   k_merge_chunks a2      : segments of > 2048 arcs: final slot = sum of ranks across sorted chunks
//   k_update       a4..a8  : ONE pass over the estimator SoA: Step 1 (level-1 reservoir), Step 2
//                            (chi^+ from ranks / degrees, level-2 pick by segment arithmetic), Step 3
//                            (closing-edge probe), block partial sums of chi over closed estimators
// After a2 the segment of vertex x holds x's arcs in increasing arrival position, i.e. Fig. 4's
// rankAll order (src asc, pos desc) reversed inside each src group: rank(x->y) = segEnd - 1 - slot.
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

// Insert v (or find it) in the vertex table; returns its slot and an arrival ticket in [0, deg_W(v)).
__device__ __forceinline__ void vt_insert(VSlot *vt, uint32_t mask, uint32_t epoch, uint32_t v, uint32_t *vlist,
                                          uint32_t *nD, uint32_t &slot, uint32_t &ticket) {
    uint32_t h = hash_vertex(v) & mask;
    while (true) {
        const uint4 s = __ldcg(reinterpret_cast<const uint4 *>(vt) + h);
        if (s.y == epoch) {
            if (s.x == v) {
                slot = h;
                ticket = atomicAdd(&vt[h].deg, 1u);
                return;
            }
            h = (h + 1) & mask;
            continue;
        }
        const u128 cmp = pack4(s.x, s.y, s.z, s.w);
        const u128 old = atomicCAS(reinterpret_cast<u128 *>(vt + h), cmp, pack4(v, epoch, 1u, 0u));
        if (old == cmp) {
            slot = h;
            ticket = 0;
            vlist[atomicAdd(nD, 1u)] = h;
            return;
        }
        // lost the race for this slot: re-read it
    }
}

// Insert (lo, hi) -> k in the edge-pair hash; false if the pair is already present (duplicate).
__device__ __forceinline__ bool pt_insert(PSlot *pt, uint32_t mask, uint32_t epoch, uint32_t lo, uint32_t hi,
                                          uint32_t k) {
    uint32_t h = hash_pair(lo, hi) & mask;
    while (true) {
        const uint4 s = __ldcg(reinterpret_cast<const uint4 *>(pt) + h);
        if (s.w == epoch) {
            if (s.x == lo && s.y == hi) return false;
            h = (h + 1) & mask;
            continue;
        }
        const u128 cmp = pack4(s.x, s.y, s.z, s.w);
        const u128 old = atomicCAS(reinterpret_cast<u128 *>(pt + h), cmp, pack4(lo, hi, k, epoch));
        if (old == cmp) return true;
    }
}

__device__ __forceinline__ uint32_t stage_one(uint2 e, uint32_t k, uint2 *__restrict__ E, uint4 *__restrict__ arcrec,
                                              VSlot *vt, uint32_t vmask, PSlot *pt, uint32_t pmask, uint32_t epoch,
                                              uint32_t *vlist, uint32_t *nD) {
    if (e.x == kEmptyV || e.y == kEmptyV) return kErrInval;
    if (e.x == e.y) return kErrLoop;
    const uint32_t lo = min(e.x, e.y), hi = max(e.x, e.y);
    E[k] = make_uint2(lo, hi);
    uint4 rec;
    vt_insert(vt, vmask, epoch, lo, vlist, nD, rec.x, rec.y);
    vt_insert(vt, vmask, epoch, hi, vlist, nD, rec.z, rec.w);
    arcrec[k] = rec;
    return pt_insert(pt, pmask, epoch, lo, hi, k) ? 0u : kErrDup;
}

// a1 + a3: two edges per thread through one 16-byte load when the input is 16-byte aligned.
__global__ void __launch_bounds__(256) k_stage(const uint2 *__restrict__ in, uint32_t w, uint2 *__restrict__ E,
                                               uint4 *__restrict__ arcrec, VSlot *vt, uint32_t vmask, PSlot *pt,
                                               uint32_t pmask, uint32_t epoch, uint32_t *vlist, uint32_t *ctr) {
    if (ctr[3] & (kErrInval | kErrLoop | kErrDup)) return;  // sticky error of an earlier async batch
    uint32_t bad = 0;
    const uint32_t stride = gridDim.x * blockDim.x;
    const bool vec = (reinterpret_cast<uintptr_t>(in) & 15u) == 0;
    if (vec) {
        const uint32_t npairs = w >> 1;
        const uint4 *in4 = reinterpret_cast<const uint4 *>(in);
        for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < npairs; q += stride) {
            const uint4 two = __ldcs(in4 + q);
            bad |= stage_one(make_uint2(two.x, two.y), 2 * q, E, arcrec, vt, vmask, pt, pmask, epoch, vlist, ctr);
            bad |= stage_one(make_uint2(two.z, two.w), 2 * q + 1, E, arcrec, vt, vmask, pt, pmask, epoch, vlist, ctr);
        }
        if ((w & 1u) && blockIdx.x * blockDim.x + threadIdx.x == 0)
            bad |= stage_one(in[w - 1], w - 1, E, arcrec, vt, vmask, pt, pmask, epoch, vlist, ctr);
    } else {
        for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < w; k += stride)
            bad |= stage_one(in[k], k, E, arcrec, vt, vmask, pt, pmask, epoch, vlist, ctr);
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (bad && (threadIdx.x & 31u) == 0) atomicOr(&ctr[3], bad);
}

// a2: segment start of every vertex of W (order of segments is irrelevant, only their contents).
__global__ void __launch_bounds__(256) k_segment(VSlot *vt, const uint32_t *__restrict__ vlist, uint32_t *ctr,
                                                 uint4 *__restrict__ chunks) {
    if (ctr[3]) return;
    const uint32_t D = ctr[0];
    __shared__ uint32_t wsum[8];
    __shared__ uint32_t base_sh;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    for (uint32_t b0 = blockIdx.x * 256u; b0 < D; b0 += gridDim.x * 256u) {
        const uint32_t d = b0 + threadIdx.x;
        uint32_t slot = 0, deg = 0;
        if (d < D) {
            slot = vlist[d];
            deg = vt[slot].deg;
        }
        uint32_t incl = deg;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= (uint32_t)off) incl += y;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        if (threadIdx.x < 8) {
            const uint32_t v = wsum[threadIdx.x];
            uint32_t x = v;
#pragma unroll
            for (int off = 1; off < 8; off <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffu, x, off);
                if (threadIdx.x >= (uint32_t)off) x += y;
            }
            wsum[threadIdx.x] = x - v;
            if (threadIdx.x == 7) base_sh = atomicAdd(&ctr[1], x);
        }
        __syncthreads();
        if (d < D) {
            const uint32_t start = base_sh + wsum[warp] + incl - deg;
            vt[slot].start = start;
            if (deg > kSmallSeg) {
                const uint32_t nch = (deg + kChunk - 1) / kChunk;
                const uint32_t c0 = atomicAdd(&ctr[2], nch);
                for (uint32_t c = 0; c < nch; ++c) chunks[c0 + c] = make_uint4(start, deg, c, 0u);
            }
        }
        __syncthreads();
    }
}

// a2: every arc to segment start + ticket.
__global__ void __launch_bounds__(256) k_scatter(const uint4 *__restrict__ arcrec, const VSlot *__restrict__ vt,
                                                 uint32_t *__restrict__ segU, uint32_t w, const uint32_t *ctr) {
    if (ctr[3]) return;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < w; k += gridDim.x * blockDim.x) {
        const uint4 a = arcrec[k];
        const uint32_t s0 = vt[a.x].start, s1 = vt[a.z].start;
        segU[s0 + a.y] = k << 1;
        segU[s1 + a.w] = (k << 1) | 1u;
    }
}

// a2, short segments: slot of an arc = number of arcs of its segment that arrived before it.
__global__ void __launch_bounds__(256) k_rank_small(const uint4 *__restrict__ arcrec, const VSlot *__restrict__ vt,
                                                    const uint32_t *__restrict__ segU, uint32_t *__restrict__ segS,
                                                    uint2 *__restrict__ einfo2, uint32_t w, const uint32_t *ctr) {
    if (ctr[3]) return;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < w; k += gridDim.x * blockDim.x) {
        const uint4 a = arcrec[k];
#pragma unroll
        for (uint32_t side = 0; side < 2; ++side) {
            const uint32_t slot = side ? a.z : a.x;
            const uint4 s = __ldg(reinterpret_cast<const uint4 *>(vt) + slot);
            const uint32_t deg = s.z, start = s.w;
            if (deg > kSmallSeg) continue;
            const uint32_t val = (k << 1) | side;
            uint32_t p = 0;
            for (uint32_t i = 0; i < deg; ++i) p += (__ldg(segU + start + i) < val) ? 1u : 0u;
            segS[start + p] = val;
            einfo2[val] = make_uint2(start + p, start + deg);
        }
    }
}

// a2, long segments: sort each chunk of <= kChunk arcs in shared memory (bitonic network).
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
                    const bool asc = (lo & size) == 0;
                    const uint32_t x = sm[lo], y = sm[hi];
                    if ((x > y) == asc) {
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

// a2, segments of > kChunk arcs: merge the sorted chunks by rank (values are distinct).
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

// a4..a8: the fused estimator update, one thread per estimator.
__global__ void __launch_bounds__(256) k_update(uint2 *__restrict__ r1s, uint2 *__restrict__ r2s,
                                                uint32_t *__restrict__ cfs, uint64_t *__restrict__ p1s,
                                                uint64_t *__restrict__ p2s, uint64_t count, uint64_t first,
                                                uint64_t seed, uint32_t batch, uint64_t m_prev, uint32_t w,
                                                const uint2 *__restrict__ E, const uint4 *__restrict__ einfo,
                                                const VSlot *__restrict__ vt, uint32_t vmask,
                                                const uint32_t *__restrict__ segS, const PSlot *__restrict__ pt,
                                                uint32_t pmask, uint32_t epoch, const uint32_t *ctr,
                                                unsigned long long *S, unsigned long long *stats) {
    if (ctr[3]) return;
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
            r1 = __ldg(E + j);
            c = 0;
            closed = false;
            // ---- Step 2a for a fresh f1 = w_j: ld = rank(u->v), rd = rank(v->u) ----
            const uint4 inf = __ldg(einfo + j);
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
            vt_find(vt, vmask, epoch, r1.x, ld, endU);
            vt_find(vt, vmask, epoch, r1.y, rd, endV);
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
                const uint32_t val = __ldg(segS + (end - 1u - a));
                k2 = val >> 1;
                r2 = __ldg(E + k2);
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
            const int64_t kk = pt_find(pt, pmask, epoch, min(x, z), max(x, z));
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
                atomicAdd(stats + 2, (unsigned long long)ctr[0]);
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

int launch_stage(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s) {
    k_stage<<<grid_for((a.w + 1) / 2, 256, 8), 256, 0, s>>>(a.in, a.w, ix.E, ix.arcrec, ix.vt, ix.vmask, ix.pt,
                                                            ix.pmask, a.epoch, ix.vlist, ix.ctr);
    return 1;
}

int launch_segment(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s) {
    k_segment<<<grid_for(2ull * a.w, 256, 8), 256, 0, s>>>(ix.vt, ix.vlist, ix.ctr, ix.chunks);
    return 1;
}

int launch_scatter(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s) {
    k_scatter<<<grid_for(a.w, 256, 8), 256, 0, s>>>(ix.arcrec, ix.vt, ix.segU, a.w, ix.ctr);
    return 1;
}

int launch_sort(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s) {
    uint2 *einfo2 = reinterpret_cast<uint2 *>(ix.einfo);
    k_rank_small<<<grid_for(a.w, 256, 8), 256, 0, s>>>(ix.arcrec, ix.vt, ix.segU, ix.segS, einfo2, a.w, ix.ctr);
    const uint32_t chunk_bound = (uint32_t)std::min<uint64_t>(ix.chunk_cap, 2ull * a.w / (kSmallSeg + 1) + 2ull * a.w / kChunk + 1);
    const uint32_t g = std::max<uint32_t>(1, std::min<uint32_t>(chunk_bound, sm_count() * 4));
    k_sort_chunks<<<g, 512, 0, s>>>(ix.chunks, ix.segU, ix.segS, einfo2, ix.ctr);
    k_merge_chunks<<<g, 256, 0, s>>>(ix.chunks, ix.segU, ix.segS, einfo2, ix.ctr);
    return 3;
}

int launch_update(const IndexBufs &ix, const StateBufs &st, const BatchArgs &a, cudaStream_t s) {
    if (st.count == 0) return 0;
    const uint64_t blocks = (st.count + 255) / 256;
    k_update<<<(uint32_t)blocks, 256, 0, s>>>(st.r1, st.r2, st.cf, st.p1, st.p2, st.count, a.first, a.seed, a.batch,
                                              a.m_prev, a.w, ix.E, ix.einfo, ix.vt, ix.vmask, ix.segS, ix.pt,
                                              ix.pmask, a.epoch, ix.ctr, st.S + a.S_slot, st.stats);
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

// event.cu -- the event-driven estimator mode (reading R17, §10 row 4).
//
// The sequential neighborhood-sampling rule (batch size 1 of bulkUpdateAll is reservoir
// sampling) with both reservoir coins replaced by skip-sampled replacement points:
//   J = next_after(t1)  the stream time at which f1 is next replaced (P(J > s) = t1 / s),
//   K = next_after(chi) the adjacency count at which f2 is next replaced (P(K > k) = chi / k), K = 1 for a new f1.
// chi is never stored: chi = deg(u) + deg(v) - B with persistent vertex degrees and B = deg_t1(u) + deg_t1(v)
// (no edge but f1 touches both u and v in a simple graph).  A batch processes only the estimators it can change:
//   * f1 is replaced          <=> the batch holds stream time J             -> watch (kJKey, J)
//   * chi reaches K           <=> deg(u) + deg(v) reaches B + K             -> watches (u, du + a), (v, dv + b)
//     with a + b = Delta + 1, Delta = B + K - du - dv: one of them fires at or before the event (re-armed with
//     the halved remainder otherwise, O(log Delta) firings per event);
//   * the closing edge arrives <=> the batch holds the pair                 -> watch (closing pair)
// and processes each of them once, replaying every event of the batch in time order against the batch index
// (vertex segments in arrival order, the edge-pair table) -- the same tables the bulk pass probes.
//
// Random words: estimator i's 64-bit word stream n = 0, 1, ...: Philox4x32-10 block ctr = (i lo, i hi, n >> 1,
// 0xED5A0000), key = (seed lo, seed hi); word x | y << 32 for even n, z | w << 32 for odd n.  U[0, n) is Lemire's
// multiply-shift, a rejected word replaced by the next word.  next_after(t): t = 0 -> 1; else epoch k = trailing
// zeros of a word (0 -> INF), L = t 2^k (> HMAX -> INF), then proposals s = L + 1 + U[0, L) accepted when
// U[0, s-1) < L and U[0, s) < L + 1; s > HMAX -> INF.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "event.h"
#include "philox.cuh"

namespace tcb {

namespace {

constexpr uint32_t kFullMask = 0xffffffffu;

// ---- the random words of one estimator ----------------------------------------------------------------------
struct EdWords {
    uint32_t id_lo, id_hi, n;  // next word index
    PhiloxKey key;
    uint64_t spare;            // the odd word of the last block (valid when n is odd and have_spare)
    bool have_spare;
};

__device__ __forceinline__ uint64_t ed_word(EdWords &w) {
    const uint32_t n = w.n++;
    if ((n & 1u) && w.have_spare) {
        w.have_spare = false;
        return w.spare;
    }
    const uint4 o = philox4x32_10(make_uint4(w.id_lo, w.id_hi, n >> 1, 0xED5A0000u), w.key);
    if (n & 1u) return (uint64_t)o.z | ((uint64_t)o.w << 32);
    w.spare = (uint64_t)o.z | ((uint64_t)o.w << 32);
    w.have_spare = true;
    return (uint64_t)o.x | ((uint64_t)o.y << 32);
}

__device__ __forceinline__ uint64_t ed_uniform(uint64_t n, EdWords &w) {
    uint64_t x = ed_word(w);
    uint64_t lo = x * n;
    uint64_t hi = __umul64hi(x, n);
    if (lo < n) {
        const uint64_t thr = (0ull - n) % n;
        while (lo < thr) {
            x = ed_word(w);
            lo = x * n;
            hi = __umul64hi(x, n);
        }
    }
    return hi;
}

__device__ uint32_t ed_next_after(uint32_t t, EdWords &w) {
    if (t == 0) return 1u;
    const uint64_t x = ed_word(w);
    if (x == 0) return kEdInf;
    const int k = __ffsll((long long)x) - 1;
    if (k >= 31) return kEdInf;
    const uint64_t L = (uint64_t)t << k;
    if (L > kEdHMax) return kEdInf;
    for (;;) {
        const uint64_t s = L + 1 + ed_uniform(L, w);
        if (ed_uniform(s - 1, w) >= L) continue;
        if (ed_uniform(s, w) >= L + 1) continue;
        return s <= kEdHMax ? (uint32_t)s : kEdInf;
    }
}

// ---- hash tables ----------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t pv_find(const EdDev &e, uint32_t x) {
    uint32_t i = hash_vertex(x) & e.pv_mask;
    for (uint32_t n = 0; n <= e.pv_mask; ++n) {
        const uint32_t k = e.pv[i].x;
        if (k == x) return i;
        if (k == kEmptyV) return kEdNil;
        i = (i + 1) & e.pv_mask;
    }
    return kEdNil;
}

__device__ uint32_t pv_insert(const EdDev &e, uint32_t x, uint32_t *ixctr) {
    uint32_t i = hash_vertex(x) & e.pv_mask;
    for (uint32_t n = 0; n <= e.pv_mask; ++n) {
        const uint32_t k = *reinterpret_cast<volatile uint32_t *>(&e.pv[i].x);
        if (k == x) return i;
        if (k == kEmptyV) {
            const uint32_t prev = atomicCAS(&e.pv[i].x, kEmptyV, x);
            if (prev == kEmptyV) {
                atomicAdd(&e.ctr[kEdPVN], 1u);
                return i;
            }
            if (prev == x) return i;
        }
        i = (i + 1) & e.pv_mask;
    }
    atomicOr(&ixctr[kCtrErr], kErrInternal);  // a full table: never a hang
    return kEdNil;
}

__device__ __forceinline__ uint64_t key64(uint32_t k0, uint32_t k1) { return ((uint64_t)k1 << 32) | k0; }

__device__ __forceinline__ uint32_t map_find(const uint4 *map, uint32_t mask, uint32_t k0, uint32_t k1) {
    const uint64_t key = key64(k0, k1);
    uint32_t i = (uint32_t)hash_pair64(key) & mask;
    for (uint32_t n = 0; n <= mask; ++n) {
        const uint4 s = map[i];
        if (s.x == k0 && s.y == k1) return i;
        if (s.x == kEmptyV && s.y == kEmptyV) return kEdNil;
        i = (i + 1) & mask;
    }
    return kEdNil;
}

__device__ uint32_t map_insert(uint4 *map, uint32_t mask, uint32_t k0, uint32_t k1, uint32_t *ixctr) {
    const uint64_t key = key64(k0, k1);
    uint32_t i = (uint32_t)hash_pair64(key) & mask;
    {  // most keys are new and their home slot free: claim it in one round trip
        const unsigned long long prev = atomicCAS(reinterpret_cast<unsigned long long *>(&map[i]), ~0ull,
                                                  (unsigned long long)key);
        if (prev == ~0ull || prev == key) return i;
    }
    for (uint32_t n = 0; n <= mask; ++n) {
        unsigned long long *kp = reinterpret_cast<unsigned long long *>(&map[i]);
        const unsigned long long cur = *reinterpret_cast<volatile unsigned long long *>(kp);
        if (cur == key) return i;
        if (cur == ~0ull) {
            const unsigned long long prev = atomicCAS(kp, ~0ull, (unsigned long long)key);
            if (prev == ~0ull || prev == key) return i;
        }
        i = (i + 1) & mask;
    }
    atomicOr(&ixctr[kCtrErr], kErrInternal);
    return kEdNil;
}

// Watch versions, one per kind, packed in one word per estimator: a node is live while its kind's version is the
// estimator's current one.  A stale node that looks live (the 10/11-bit field wrapped) only queues the estimator
// once more -- processing an estimator without events in the batch is harmless -- so the check is a filter, and
// correctness needs only that a live watch is never missed.
enum WatchKind : uint32_t { kWJ = 0, kWT = 1, kWP = 2 };
__device__ __forceinline__ uint32_t ver_of(uint32_t ver, uint32_t kind) {
    return kind == kWJ ? (ver & 0x3FFu) : kind == kWT ? ((ver >> 10) & 0x7FFu) : (ver >> 21);
}
__device__ __forceinline__ uint32_t ver_bump(uint32_t ver, uint32_t kind) {
    const uint32_t f = ver_of(ver, kind) + 1u;
    return kind == kWJ ? ((ver & ~0x3FFu) | (f & 0x3FFu))
                       : kind == kWT ? ((ver & ~(0x7FFu << 10)) | ((f & 0x7FFu) << 10)) : ((ver & 0x1FFFFFu) | (f << 21));
}

// One slot per active lane of the calling (possibly divergent) warp: lanes with want get consecutive indices from
// *ctr (one atomic per warp), others get kEdNil.
__device__ __forceinline__ uint32_t warp_take(uint32_t *ctr, bool want) {
    const uint32_t mask = __activemask();
    const uint32_t b = __ballot_sync(mask, want);
    if (!b) return kEdNil;
    const uint32_t lane = threadIdx.x & 31u, leader = __ffs(b) - 1u;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(ctr, (uint32_t)__popc(b));
    base = __shfl_sync(mask, base, leader);
    return want ? base + (uint32_t)__popc(b & ((1u << lane) - 1u)) : kEdNil;
}

// n[lane] <= 7 consecutive slots per active lane (one atomic per warp): returns the lane's first slot.
__device__ __forceinline__ uint32_t warp_take_n(uint32_t *ctr, uint32_t n) {
    const uint32_t mask = __activemask();
    const uint32_t lane = threadIdx.x & 31u, lt = (1u << lane) - 1u;
    const uint32_t b0 = __ballot_sync(mask, n & 1u), b1 = __ballot_sync(mask, n & 2u), b2 = __ballot_sync(mask, n & 4u);
    const uint32_t total = __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
    if (!total) return 0u;
    const uint32_t leader = __ffs(mask) - 1u;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(ctr, total);
    base = __shfl_sync(mask, base, leader);
    return base + __popc(b0 & lt) + 2 * __popc(b1 & lt) + 4 * __popc(b2 & lt);
}

// Watch lists are stacks of 64-byte chunks of kChunkNodes nodes {estimator, kind << 30 | version} with the next chunk
// in word 14, so a list is walked one DRAM access per chunk.  The key's slot holds {head chunk, fill of the head}
// as one 64-bit word (slot .z = head, .w = fill); a full or missing head gets a fresh chunk by CAS.
constexpr uint32_t kChunkNodes = 7;

// The slow path of a watch: key slot s known, spare chunk taken; push the node (CAS loop on {head, fill}).
__device__ void watch_push(const EdDev &e, uint4 *map, uint32_t s, uint2 node, uint32_t spare, uint32_t *ixctr) {
    unsigned long long *hf = reinterpret_cast<unsigned long long *>(&map[s].z);
    for (uint32_t it = 0; it < 1024u; ++it) {
        const unsigned long long old = *reinterpret_cast<volatile unsigned long long *>(hf);
        const uint32_t head = (uint32_t)old, fill = (uint32_t)(old >> 32);
        if (head != kEdNil && fill < kChunkNodes) {
            if (atomicCAS(hf, old, old + (1ull << 32)) == old) {
                reinterpret_cast<uint2 *>(e.pool + 4ull * head)[fill] = node;
                return;
            }
        } else {
            reinterpret_cast<uint32_t *>(e.pool + 4ull * spare)[14] = head;
            if (atomicCAS(hf, old, (1ull << 32) | spare) == old) {
                reinterpret_cast<uint2 *>(e.pool + 4ull * spare)[0] = node;
                return;
            }
        }
    }
    atomicOr(&ixctr[kCtrErr], kErrInternal);  // never: a bounded retry loop instead of a possible hang
}

// Arm up to 4 watches of one estimator.  Their round trips are independent, so each step is issued for all of
// them before any result is used: claim the keys' home slots (most keys are new), then install each spare chunk
// on a fresh key's {head, fill} word; only a taken home slot or an existing list takes the looping paths.
struct WatchReq {
    uint4 *map;
    uint32_t mask, k0, k1, kind, spare;
};

__device__ __forceinline__ void watch_many(const EdDev &e, const WatchReq *rq, uint32_t n, uint32_t est, uint32_t ver,
                                           uint32_t *ixctr) {
    uint32_t slot[4];
    unsigned long long prev[4];
#pragma unroll
    for (uint32_t i = 0; i < 4; ++i) {
        if (i >= n) continue;
        slot[i] = (uint32_t)hash_pair64(key64(rq[i].k0, rq[i].k1)) & rq[i].mask;
        prev[i] = atomicCAS(reinterpret_cast<unsigned long long *>(&rq[i].map[slot[i]]), ~0ull,
                            (unsigned long long)key64(rq[i].k0, rq[i].k1));
    }
#pragma unroll
    for (uint32_t i = 0; i < 4; ++i) {
        if (i >= n) continue;
        if (prev[i] != ~0ull && prev[i] != key64(rq[i].k0, rq[i].k1))
            slot[i] = map_insert(rq[i].map, rq[i].mask, rq[i].k0, rq[i].k1, ixctr);
        if (rq[i].spare >= e.pool_cap) {
            atomicOr(&ixctr[kCtrErr], kErrInternal);
            slot[i] = kEdNil;
        }
        if (slot[i] == kEdNil) continue;
        reinterpret_cast<uint32_t *>(e.pool + 4ull * rq[i].spare)[14] = kEdNil;
        // a key just created has the cleared {NIL, ~0} word: install the chunk directly
        prev[i] = atomicCAS(reinterpret_cast<unsigned long long *>(&rq[i].map[slot[i]].z), ~0ull,
                            (1ull << 32) | rq[i].spare);
    }
#pragma unroll
    for (uint32_t i = 0; i < 4; ++i) {
        if (i >= n || slot[i] == kEdNil) continue;
        const uint2 node = make_uint2(est, (rq[i].kind << 30) | ver_of(ver, rq[i].kind));
        if (prev[i] == ~0ull) reinterpret_cast<uint2 *>(e.pool + 4ull * rq[i].spare)[0] = node;
        else watch_push(e, rq[i].map, slot[i], node, rq[i].spare, ixctr);
    }
}

// detach the list at slot s and queue its live estimators (each at most once per batch)
__device__ void fire(const EdDev &e, uint4 *map, uint32_t s, uint32_t tag, uint32_t *ixctr) {
    const unsigned long long old = atomicExch(reinterpret_cast<unsigned long long *>(&map[s].z), (unsigned long long)kEdNil);
    uint32_t c = (uint32_t)old, n = min((uint32_t)(old >> 32), kChunkNodes);
    for (uint32_t hops = 0; c != kEdNil && hops < e.pool_cap; ++hops) {
        const uint4 *ch = e.pool + 4ull * c;
        const uint4 q0 = ch[0], q1 = ch[1], q2 = ch[2], q3 = ch[3];
        const uint32_t w[16] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x, q2.y, q2.z, q2.w, q3.x, q3.y, q3.z, q3.w};
        uint2 vs[kChunkNodes];
#pragma unroll
        for (uint32_t j = 0; j < kChunkNodes; ++j)  // the versions of all nodes of the chunk in flight together
            if (j < n) vs[j] = e.vs[w[2 * j]];
#pragma unroll
        for (uint32_t j = 0; j < kChunkNodes; ++j) {
            if (j >= n) continue;
            const uint32_t est = w[2 * j], kv = w[2 * j + 1];
            const bool want = (kv & 0x3FFFFFFFu) == ver_of(vs[j].x, kv >> 30) && vs[j].y != tag &&
                              atomicExch(&e.vs[est].y, tag) != tag;
            const uint32_t q = warp_take(&e.ctr[kEdQueue], want);
            TC_CHECK(!want || (q < e.count && est < e.count), ixctr);
            if (want) e.queue[q] = est;
        }
        c = w[14];
        n = kChunkNodes;
    }
}

// ---- the batch index as the event mode reads it --------------------------------------------------------------
struct EdIdx {
    Lookup L;
    const uint2 *segS;   // arcs {k << 1 | side, neighbour} grouped by vertex, arrival order
    const uint2 *apos;   // edge k -> partition positions of its two arcs
    const uint2 *pslot;  // partition position -> {slot in segS, segment end}
    uint32_t *ctr;
    const BatchDesc *d;
    uint32_t w;
};

__device__ __forceinline__ uint32_t arc_vertex(const uint2 *E, uint32_t val) {
    const uint2 e = E[val >> 1];
    return (val & 1u) ? e.y : e.x;
}

// a vertex as this batch sees it
struct VInfo {
    uint32_t dold, pvs, dW, start;  // degree before the batch, pv slot, arcs in the batch, segment start
};

__device__ __forceinline__ VInfo vinfo_of(const EdDev &e, uint32_t x, uint2 r) {
    VInfo v;
    if (r.x) {
        const uint4 s = e.seg[r.y];
        v.dold = s.x;
        v.pvs = s.y;
        v.dW = r.x;
        v.start = r.y;
    } else {
        const uint32_t p = pv_find(e, x);
        v.pvs = p;
        v.dold = p == kEdNil ? 0u : e.pv[p].y;
        v.dW = 0;
        v.start = 0;
    }
    return v;
}

__device__ __forceinline__ VInfo vinfo(const EdIdx &I, const EdDev &e, uint32_t x) {
    VertProbe P;
    vt_issue(I.L, x, P);
    return vinfo_of(e, x, vt_resolve(I.L, P, x));  // {deg_W, segment start} or {0, 0}
}

// both endpoints, their probes issued together
__device__ __forceinline__ void vinfo2(const EdIdx &I, const EdDev &e, uint32_t x, uint32_t y, VInfo &ix, VInfo &iy) {
    VertProbe P, Q;
    vt_issue(I.L, x, P);
    vt_issue(I.L, y, Q);
    const uint2 rx = vt_resolve(I.L, P, x), ry = vt_resolve(I.L, Q, y);
    ix = vinfo_of(e, x, rx);
    iy = vinfo_of(e, y, ry);
}

// arcs of vertex v in the batch with batch index <= kmax (kmax = -1: none)
__device__ __forceinline__ uint32_t cnt_le(const EdIdx &I, const VInfo &v, int32_t kmax) {
    if (kmax < 0) return 0u;
    if (kmax >= (int32_t)I.w - 1) return v.dW;  // the whole batch: no search
    uint32_t a = 0, b = v.dW;
    while (a < b) {
        const uint32_t mid = (a + b) >> 1;
        if ((int32_t)(I.segS[v.start + mid].x >> 1) <= kmax) a = mid + 1;
        else b = mid;
    }
    return a;
}

// cnt_le of two vertices at once, the two binary searches interleaved so that their loads overlap
__device__ __forceinline__ uint2 cnt_le2(const EdIdx &I, const VInfo &u, const VInfo &v, int32_t kmax) {
    if (kmax < 0) return make_uint2(0u, 0u);
    if (kmax >= (int32_t)I.w - 1) return make_uint2(u.dW, v.dW);
    uint32_t a0 = 0, b0 = u.dW, a1 = 0, b1 = v.dW;
    while (a0 < b0 || a1 < b1) {
        const uint32_t m0 = (a0 + b0) >> 1, m1 = (a1 + b1) >> 1;
        const uint32_t x0 = a0 < b0 ? I.segS[u.start + m0].x : 0u, x1 = a1 < b1 ? I.segS[v.start + m1].x : 0u;
        if (a0 < b0) {
            if ((int32_t)(x0 >> 1) <= kmax) a0 = m0 + 1;
            else b0 = m0;
        }
        if (a1 < b1) {
            if ((int32_t)(x1 >> 1) <= kmax) a1 = m1 + 1;
            else b1 = m1;
        }
    }
    return make_uint2(a0, a1);
}

// batch index of the n-th (n >= 1) arc of u or v after batch index kq (the caller knows it exists): the two
// segments are sorted by batch index and disjoint, so a binary search over how many come from u's (merge path)
// a0, b0: the arcs of u and v at or before kq (cnt_le, computed once per f1 epoch)
__device__ int32_t kth_after(const EdIdx &I, const VInfo &u, const VInfo &v, uint32_t a0, uint32_t b0, uint32_t n) {
    const uint32_t la = u.dW - a0, lb = v.dW - b0;
    const uint2 *A = I.segS + u.start + a0, *Bs = I.segS + v.start + b0;
    uint32_t lo = n > lb ? n - lb : 0u, hi = min(n, la);
    while (lo < hi) {  // smallest i whose A[i] comes after B[n - i - 1]
        const uint32_t i = (lo + hi) >> 1;
        if ((A[i].x >> 1) < (Bs[n - i - 1].x >> 1)) lo = i + 1;
        else hi = i;
    }
    const int32_t ka = lo ? (int32_t)(A[lo - 1].x >> 1) : -1, kb = n - lo ? (int32_t)(Bs[n - lo - 1].x >> 1) : -1;
    return max(ka, kb);
}

// ---- kernels ---------------------------------------------------------------------------------------------------
#ifdef TC_ED_CLOCKS  // timing instrumentation of k_ed_process (tools/dbg, never in the product build)
__device__ uint32_t g_edclk[1 << 22][8];
__device__ uint32_t g_edclk_n;
#define TC_EDCLK_BEGIN                                                 \
    const long long clk0_ = clock64();                                 \
    const uint32_t ci_ = atomicAdd(&g_edclk_n, 1u) & ((1u << 22) - 1u); \
    g_edclk[ci_][7] = events;
#define TC_EDCLK(k) g_edclk[ci_][k] = (uint32_t)(clock64() - clk0_);
#else
#define TC_EDCLK_BEGIN
#define TC_EDCLK(k)
#endif
// The per-batch kernels are latency chains with little data each (a few thousand items over 148 SMs): items are
// dealt lane-major -- item i to warp i mod W, lane i / W for the W warps of the grid -- so that a small batch puts
// one or two items in each of many warps rather than 32 divergent lanes in a few.
struct Spread {
    uint32_t first, step;
};
__device__ __forceinline__ Spread spread() {
    const uint32_t nw = gridDim.x * (blockDim.x >> 5), wid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    return Spread{(threadIdx.x & 31u) * nw + wid, 32u * nw};
}


// Persistent vertices of the batch: find-or-insert, degree limit (reading R17c), per-segment info, and S's growth
// from every closed estimator whose f1 touches a batch vertex (sum over batch arcs of ncl(x)).
__global__ void __launch_bounds__(256) k_ed_pre(EdIdx I, EdDev e, unsigned long long *S, unsigned long long *stats) {
    const BatchDesc d = *I.d;
    if (I.ctr[kCtrErr]) {  // rejected (this batch or an earlier asynchronous one): record the first, change nothing
        if (blockIdx.x == 0 && threadIdx.x == 0 && I.ctr[kCtrFailB] == 0xFFFFFFFFu) I.ctr[kCtrFailB] = d.batch;
        return;
    }
    unsigned long long grow = 0;
    uint32_t nv = 0;  // distinct vertices (the bench's byte model: tc_stats out[2], out[3])
    const Spread sp = spread();
    for (uint32_t s = sp.first; s < 2 * I.w; s += sp.step) {
        const uint32_t val = I.segS[s].x;
        const uint32_t x = arc_vertex(I.L.E, val);
        if (s > 0 && arc_vertex(I.L.E, I.segS[s - 1].x) == x) continue;  // not the first arc of x's segment
        VertProbe P;
        vt_issue(I.L, x, P);
        const uint32_t dW = vt_resolve(I.L, P, x).x;
        ++nv;
        const uint32_t p = pv_insert(e, x, I.ctr);
        if (p == kEdNil) continue;
        const uint4 pv = e.pv[p];
        if ((uint64_t)pv.y + dW > kEdDegMax) atomicOr(&I.ctr[kCtrErr], kErrOvf);
        e.seg[s] = make_uint4(pv.y, p, dW, s);
        grow += (unsigned long long)dW * pv.z;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        grow += __shfl_xor_sync(kFullMask, grow, off);
        nv += __shfl_xor_sync(kFullMask, nv, off);
    }
    if ((threadIdx.x & 31u) == 0) {
        if (grow) atomicAdd(S + d.slot, grow);
        if (nv) atomicAdd(stats + 2, (unsigned long long)nv);
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(stats + 3, 1ull);
    }
}

// The fast path (no vertex degree can reach the limit in this batch, so nothing after the index can reject it):
// k_ed_pre's vertex work and k_ed_trigger's lookups in ONE kernel over 4w items -- arc slot s < 2w: the vertex's
// persistent record (inserted at its segment's first slot, with the segment record and S's growth) and the degree
// watch (x, deg_old(x) + rank + 1) that the arc reaches; edge item: the time and pair watches.  The degrees
// themselves are applied by k_ed_process (nothing reads a batch vertex's persistent degree before that).
__global__ void __launch_bounds__(256) k_ed_front(EdIdx I, EdDev e, unsigned long long *S, unsigned long long *stats) {
    const BatchDesc d = *I.d;
    if (I.ctr[kCtrErr]) {  // rejected (this batch or an earlier asynchronous one): record the first, change nothing
        if (blockIdx.x == 0 && threadIdx.x == 0 && I.ctr[kCtrFailB] == 0xFFFFFFFFu) I.ctr[kCtrFailB] = d.batch;
        return;
    }
    const bool full = e.ctr[kEdFull] != 0;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    if (full) {  // a full sweep: every estimator is processed and re-armed into cleared maps
        const uint4 empty = make_uint4(kEmptyV, kEmptyV, kEdNil, kEmptyV);
        for (uint64_t i = tid; i <= e.a_mask; i += nth) e.amap[i] = empty;
        for (uint64_t i = tid; i <= e.p_mask; i += nth) e.pmap[i] = empty;
        if (tid == 0) {
            for (uint32_t i = 0; i < kEdStripes; ++i) e.ctr[kEdStripe0 + i] = 0u;
            atomicAdd(&e.ctr[kEdSweeps], 1u);
        }
    }
    const uint32_t tag = d.batch + 1u;
    const uint32_t t0 = (uint32_t)d.m_prev + 1u;  // stream time of batch edge 0
    unsigned long long grow = 0;
    uint32_t nv = 0;
    const Spread sp = spread();
    for (uint32_t i = sp.first; i < 4 * I.w; i += sp.step) {
        uint32_t sl = kEdNil;
        uint4 *map = e.amap;
        if (i < 2 * I.w) {
            const uint32_t s = i;
            const uint32_t x = arc_vertex(I.L.E, I.segS[s].x);
            const bool first = s == 0 || arc_vertex(I.L.E, I.segS[s - 1].x) != x;
            VertProbe P;
            vt_issue(I.L, x, P);
            const uint2 r = vt_resolve(I.L, P, x);  // {deg_W, segment start}
            TC_CHECK(r.x > 0 && r.y <= s && s < r.y + r.x, I.ctr);
            uint32_t dold;
            if (first) {
                const uint32_t p = pv_insert(e, x, I.ctr);
                if (p == kEdNil) continue;
                const uint4 pv = e.pv[p];
                dold = pv.y;
                e.seg[s] = make_uint4(pv.y, p, r.x, s);
                grow += (unsigned long long)r.x * pv.z;
                ++nv;
            } else {
                const uint32_t p = full ? kEdNil : pv_find(e, x);  // a vertex new in this batch has no watches
                dold = p == kEdNil ? 0u : e.pv[p].y;
            }
            if (!full && dold) sl = map_find(e.amap, e.a_mask, x, dold + (s - r.y) + 1u);
        } else if (!full) {
            const uint32_t j = i - 2 * I.w, k = j >> 1;
            if (j & 1u) {
                const uint2 ed = I.L.E[k];
                map = e.pmap;
                sl = map_find(e.pmap, e.p_mask, ed.x, ed.y);
            } else {
                sl = map_find(e.amap, e.a_mask, kJKey, t0 + k);
            }
        }
        if (sl != kEdNil) fire(e, map, sl, tag, I.ctr);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        grow += __shfl_xor_sync(kFullMask, grow, off);
        nv += __shfl_xor_sync(kFullMask, nv, off);
    }
    if ((threadIdx.x & 31u) == 0) {
        if (grow) atomicAdd(S + d.slot, grow);
        if (nv) atomicAdd(stats + 2, (unsigned long long)nv);
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(stats + 3, 1ull);
    }
}

// Watches that fire in this batch -> the queue.  A full sweep instead clears the watch maps (every estimator is
// processed and re-armed).
__global__ void __launch_bounds__(256) k_ed_trigger(EdIdx I, EdDev e) {
    if (I.ctr[kCtrErr]) return;
    const BatchDesc d = *I.d;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    if (e.ctr[kEdFull]) {
        const uint4 empty = make_uint4(kEmptyV, kEmptyV, kEdNil, kEmptyV);
        for (uint64_t i = tid; i <= e.a_mask; i += nth) e.amap[i] = empty;
        for (uint64_t i = tid; i <= e.p_mask; i += nth) e.pmap[i] = empty;
        if (tid == 0) {
            for (uint32_t i = 0; i < kEdStripes; ++i) e.ctr[kEdStripe0 + i] = 0u;
            atomicAdd(&e.ctr[kEdSweeps], 1u);
        }
        return;
    }
    const uint32_t tag = d.batch + 1u;
    const uint32_t t0 = (uint32_t)d.m_prev + 1u;  // stream time of batch edge 0
    const Spread sp = spread();
    for (uint32_t i = sp.first; i < 4 * I.w; i += sp.step) {  // item (edge k, kind): time, pair, lo arc, hi arc
        const uint32_t k = i >> 2, kind = i & 3u;
        uint32_t sl;
        uint4 *map = e.amap;
        if (kind == 0) {
            sl = map_find(e.amap, e.a_mask, kJKey, t0 + k);
        } else if (kind == 1) {
            const uint2 ed = I.L.E[k];
            map = e.pmap;
            sl = map_find(e.pmap, e.p_mask, ed.x, ed.y);
        } else {
            const uint2 ed = I.L.E[k];
            const uint32_t x = kind == 3 ? ed.y : ed.x;
            const uint2 ap = I.apos[k];
            const uint2 ps = I.pslot[kind == 3 ? ap.y : ap.x];  // {slot, segment end}
            VertProbe P;
            vt_issue(I.L, x, P);
            const uint2 r = vt_resolve(I.L, P, x);  // {deg_W, start}
            TC_CHECK(r.x > 0 && r.y <= ps.x && ps.x < r.y + r.x && ps.x < 2 * I.w, I.ctr);
            const uint32_t theta = e.seg[r.y].x + (ps.x - r.y) + 1u;  // x's degree once this arc has arrived
            sl = map_find(e.amap, e.a_mask, x, theta);
        }
        if (sl != kEdNil) fire(e, map, sl, tag, I.ctr);
    }
}

// Each queued estimator (every estimator in a full sweep): replay its events of this batch in time order, update
// S and the closed counts, re-arm its watches.
__global__ void __launch_bounds__(256) k_ed_process(EdIdx I, EdDev e, unsigned long long *S) {
    if (I.ctr[kCtrErr]) return;
    const BatchDesc d = *I.d;
    const bool full = e.ctr[kEdFull] != 0;
    const uint32_t nq = full ? (uint32_t)e.count : e.ctr[kEdQueue];
    const uint32_t P0 = (uint32_t)d.m_prev, Pend = P0 + I.w;
    Lookup L = I.L;
    L.ptag = d.ptag;
    unsigned long long dS = 0;
    uint32_t visited = 0, events = 0;
    if (d.pad & 4u) {  // the fast path: the batch's vertex degrees (k_ed_front left them to this kernel; the
                       // estimators below read the persistent degree of non-batch vertices only)
        for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < 2 * I.w; s += gridDim.x * blockDim.x) {
            const uint32_t x = arc_vertex(I.L.E, I.segS[s].x);
            if (s > 0 && arc_vertex(I.L.E, I.segS[s - 1].x) == x) continue;
            const uint4 sg = e.seg[s];
            e.pv[sg.y].y = sg.x + sg.z;
        }
    }
    const Spread sp = full ? Spread{blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x} : spread();
    for (uint32_t q = sp.first; q < nq; q += sp.step) {
        const uint32_t t = full ? q : e.queue[q];
        TC_CHECK(t < e.count, I.ctr);
        TC_EDCLK_BEGIN
        ++visited;
        const uint64_t gid = e.first + t;
        EdWords W{(uint32_t)gid, (uint32_t)(gid >> 32), e.ev[t], PhiloxKey{(uint32_t)e.seed, (uint32_t)(e.seed >> 32)},
                  0ull, false};
        uint32_t J = e.J[t], t1 = e.t1[t], u = e.u[t], v = e.v[t], B = e.B[t], K = e.K[t], t2 = e.t2[t], y = e.y[t],
                 fl = e.fl[t];
        const uint32_t uo = u, vo = v, Bo = B, t1o = t1, J_o = J, t2o = t2;
        const bool closed_o = (fl & 1u) != 0;
        // the batch in time order, one f1 epoch at a time: f2 events (clause 3) of the current f1 up to the next f1
        // replacement (clause 1) inside the batch, then that replacement -- the random words are used in event
        // order, as the per-edge rule uses them
        VInfo iu, iv;
        if (t1) vinfo2(I, e, u, v, iu, iv);
        TC_EDCLK(0)
        int32_t kq = -1;  // events of the current f1 are after batch index kq
        for (;;) {
            const bool jin = J != kEdInf && J <= Pend;
            const int32_t kh = jin ? (int32_t)(J - P0) - 2 : (int32_t)I.w - 1;  // the epoch's last batch index
            if (t1 && K != kEdInf) {
                const uint2 ch = cnt_le2(I, iu, iv, kh);
                const uint32_t chi_h = iu.dold + ch.x + iv.dold + ch.y - B;
                if (K <= chi_h) {  // chi reaches K at an arc of this epoch
                    // every replacement of the epoch draws the next K (the words are used in event order), but
                    // only the last one's arc is the epoch's f2: locate that one alone
                    uint32_t Klast;
                    do {
                        Klast = K;
                        K = ed_next_after(K, W);
                        ++events;
                    } while (K != kEdInf && K <= chi_h);
                    const uint2 cq = cnt_le2(I, iu, iv, kq);
                    const uint32_t cu = cq.x, cv = cq.y;
                    const uint32_t chi_q = iu.dold + cu + iv.dold + cv - B;
                    const int32_t k2 = kth_after(I, iu, iv, cu, cv, Klast - chi_q);
                    TC_CHECK(k2 > kq && k2 <= kh, I.ctr);
                    const uint2 ed = L.E[k2];
                    const bool at_u = ed.x == u || ed.y == u;
                    const uint32_t sh = at_u ? u : v;
                    y = ed.x == sh ? ed.y : ed.x;
                    t2 = P0 + 1u + (uint32_t)k2;
                    fl = at_u ? 0u : 2u;  // a new f2 is not closed
                }
            }
            if (!jin) break;
            t1 = J;  // clause 1: f1 <- e_J
            J = ed_next_after(t1, W);
            ++events;
            kq = (int32_t)(t1 - P0 - 1u);
            const uint2 ed = L.E[kq];
 
            u = ed.x;
            v = ed.y;
            vinfo2(I, e, u, v, iu, iv);
            const uint2 cb = cnt_le2(I, iu, iv, kq);
            B = iu.dold + cb.x + iv.dold + cb.y;
            K = 1u;
            t2 = 0u;
            y = kEmptyV;
            fl = 0u;
        }
        TC_EDCLK(1)
        uint32_t du_end = 0, dv_end = 0;
        if (t1) {
            du_end = iu.dold + iu.dW;
            dv_end = iv.dold + iv.dW;
            if (t2 && !(fl & 1u)) {  // clause 4: the closing edge in this batch, after f2
                const uint32_t z = (fl & 2u) ? u : v;
                const int64_t kc = pt_find(L, min(z, y), max(z, y));
                if (kc >= 0 && P0 + 1u + (uint32_t)kc > t2) fl |= 1u;
            }
        }
        const bool closed = (fl & 1u) != 0;
        TC_EDCLK(2)
        // S and the closed counts: the old contribution at the end of the batch out, the new one in
        if (closed_o) {
            uint32_t c_old;
            if (t1 == t1o) {
                c_old = du_end + dv_end - Bo;
            } else {
                VInfo a, b;
                vinfo2(I, e, uo, vo, a, b);
                c_old = a.dold + a.dW + b.dold + b.dW - Bo;
                atomicSub(&e.pv[a.pvs].z, 1u);
                atomicSub(&e.pv[b.pvs].z, 1u);
            }
            dS -= c_old;
            if (t1 == t1o && !closed) {
                atomicSub(&e.pv[iu.pvs].z, 1u);
                atomicSub(&e.pv[iv.pvs].z, 1u);
            }
        }
        if (closed) {
            dS += du_end + dv_end - B;
            if (!(closed_o && t1 == t1o)) {
                atomicAdd(&e.pv[iu.pvs].z, 1u);
                atomicAdd(&e.pv[iv.pvs].z, 1u);
            }
        }
        TC_EDCLK(3)
        // re-arm: the degree watches always (their split depends on the degrees now); the time and pair watches only
        // when they changed (the old node is still armed otherwise), or after a full sweep cleared the maps
        uint32_t ver = e.vs[t].x;
        const bool armJ = (full || J != J_o) && J != kEdInf, armT = t1 && K != kEdInf,
                   newP = full || t2 != t2o || closed != closed_o, armP = newP && t2 && !closed;
        const uint32_t stripe = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) % kEdStripes;
        const uint32_t nch = (armJ ? 1u : 0u) + (armT ? 2u : 0u) + (armP ? 1u : 0u);
        const uint32_t l = warp_take_n(&e.ctr[kEdStripe0 + stripe], nch), stripe_cap = e.pool_cap / kEdStripes;
        uint32_t chunk = l + nch <= stripe_cap ? stripe * stripe_cap + l : e.pool_cap;  // past the stripe: kErrInternal
        WatchReq rq[4];
        uint32_t nrq = 0;
        if (full || J != J_o) {
            ver = ver_bump(ver, kWJ);
            if (armJ) rq[nrq++] = WatchReq{e.amap, e.a_mask, kJKey, J, kWJ, chunk++};
        }
        ver = ver_bump(ver, kWT);
        if (armT) {
            // chi reaches K once deg(u) + deg(v) has grown by delta more: split delta + 1 between u and v in
            // proportion to their degrees (a proxy of their arrival rates), so that the first watch to fire tends to
            // be close to the event itself; any split with a, b >= 1 and a + b = delta + 1 is exact
            const uint32_t delta = B + K - du_end - dv_end;  // >= 1
            uint32_t a = (uint32_t)((uint64_t)(delta + 1u) * du_end / ((uint64_t)du_end + dv_end));
            a = min(max(a, 1u), delta);
            const uint32_t b = delta + 1u - a;
            rq[nrq++] = WatchReq{e.amap, e.a_mask, u, du_end + a, kWT, chunk++};
            rq[nrq++] = WatchReq{e.amap, e.a_mask, v, dv_end + b, kWT, chunk++};
        }
        if (newP) {
            ver = ver_bump(ver, kWP);
            if (armP) {
                const uint32_t z = (fl & 2u) ? u : v;
                rq[nrq++] = WatchReq{e.pmap, e.p_mask, min(z, y), max(z, y), kWP, chunk++};
            }
        }
        watch_many(e, rq, nrq, t, ver, I.ctr);
        TC_EDCLK(4)
#ifdef TC_ED_CLOCKS
        g_edclk[ci_][6] = events;
#endif
        e.vs[t].x = ver;
        e.J[t] = J;
        e.t1[t] = t1;
        e.u[t] = u;
        e.v[t] = v;
        e.B[t] = B;
        e.K[t] = t1 ? K : kEdInf;
        e.t2[t] = t2;
        e.y[t] = y;
        e.fl[t] = fl;
        e.ev[t] = W.n;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        dS += __shfl_xor_sync(kFullMask, dS, off);
        visited += __shfl_xor_sync(kFullMask, visited, off);
        events += __shfl_xor_sync(kFullMask, events, off);
    }
    if ((threadIdx.x & 31u) == 0) {
        if (dS) atomicAdd(S + d.slot, dS);
        if (visited) atomicAdd(&e.ctr[kEdVisited], visited);
        if (events) atomicAdd(&e.ctr[kEdEvents], events);
    }
}

// The batch's degrees into the persistent table.
__global__ void __launch_bounds__(256) k_ed_post(EdIdx I, EdDev e) {
    if (I.ctr[kCtrErr]) return;
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < 2 * I.w; s += gridDim.x * blockDim.x) {
        const uint32_t x = arc_vertex(I.L.E, I.segS[s].x);
        if (s > 0 && arc_vertex(I.L.E, I.segS[s - 1].x) == x) continue;
        const uint4 sg = e.seg[s];
        e.pv[sg.y].y = sg.x + sg.z;
    }
}

__global__ void k_ed_init(EdDev e) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t t = tid; t < e.count; t += nth) {
        e.J[t] = 1u;
        e.t1[t] = 0u;
        e.u[t] = kEmptyV;
        e.v[t] = kEmptyV;
        e.B[t] = 0u;
        e.K[t] = kEdInf;
        e.t2[t] = 0u;
        e.y[t] = kEmptyV;
        e.fl[t] = 0u;
        e.vs[t] = make_uint2(0u, 0u);
        e.ev[t] = 0u;
    }
    const uint4 empty = make_uint4(kEmptyV, kEmptyV, kEdNil, kEmptyV);
    for (uint64_t i = tid; i <= e.a_mask; i += nth) e.amap[i] = empty;
    for (uint64_t i = tid; i <= e.p_mask; i += nth) e.pmap[i] = empty;
    for (uint64_t i = tid; i <= e.pv_mask; i += nth) e.pv[i] = make_uint4(kEmptyV, 0u, 0u, 0u);
    if (tid < (uint64_t)kEdWords) e.ctr[tid] = 0u;
}

__global__ void k_ed_set_thr(uint32_t *ctr, uint32_t thr) { ctr[kEdThr] = thr; }

__global__ void k_ed_rehash(uint4 *old_pv, uint64_t old_n, uint4 *pv, uint32_t mask, uint32_t *err) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < old_n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 s = old_pv[i];
        if (s.x == kEmptyV) continue;
        uint32_t j = hash_vertex(s.x) & mask;
        uint32_t n = 0;
        for (; n <= mask; ++n) {
            if (atomicCAS(&pv[j].x, kEmptyV, s.x) == kEmptyV) {
                pv[j].y = s.y;
                pv[j].z = s.z;
                break;
            }
            j = (j + 1) & mask;
        }
        if (n > mask) atomicOr(err, 1u);
    }
}

__global__ void k_ed_fill_pv(uint4 *pv, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        pv[i] = make_uint4(kEmptyV, 0u, 0u, 0u);
}

__global__ void k_ed_export(EdDev e, uint2 *r1, uint32_t *p1, uint2 *r2, uint32_t *p2, uint32_t *cf) {
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < e.count; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t t1 = e.t1[t];
        if (!t1) {
            r1[t] = r2[t] = make_uint2(kEmptyV, kEmptyV);
            p1[t] = p2[t] = kEmptyV;
            cf[t] = 0u;
            continue;
        }
        const uint32_t u = e.u[t], v = e.v[t];
        const uint32_t pu = pv_find(e, u), pv = pv_find(e, v);
        const uint32_t chi = e.pv[pu].y + e.pv[pv].y - e.B[t];
        const uint32_t fl = e.fl[t], t2 = e.t2[t];
        r1[t] = make_uint2(u, v);
        p1[t] = t1 - 1u;
        if (t2) {
            const uint32_t sh = (fl & 2u) ? v : u, y = e.y[t];
            r2[t] = make_uint2(min(sh, y), max(sh, y));
            p2[t] = t2 - 1u;
        } else {
            r2[t] = make_uint2(kEmptyV, kEmptyV);
            p2[t] = kEmptyV;
        }
        cf[t] = chi | ((fl & 1u) ? kClosedBit : 0u);
    }
}

uint32_t grid_of(uint64_t items, uint32_t per_sm) {
    const uint64_t want = (items + 255) / 256;
    const uint64_t cap = (uint64_t)sm_count() * per_sm;
    return (uint32_t)std::max<uint64_t>(1, std::min(want, cap));
}

uint64_t pow2_at_least(uint64_t x) {
    uint64_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

}  // namespace

bool ed_alloc(EdDev &e, uint64_t count, uint64_t first, uint64_t seed, uint64_t pv_cap) {
    e = EdDev();
    e.count = count;
    e.first = first;
    e.seed = seed;
    const uint64_t n = std::max<uint64_t>(count, 1);
    // watch chunks (64 B, 7 nodes; every armed watch takes one): a sweep arms at most 4 per estimator, a batch at
    // most 4 per estimator it visits; a rebuild is due once more than 12 n are in use, so 16 n + slack always
    // suffice.  Every key owns at least one chunk, so the maps (load <= 1/2) get 2 slots per chunk.  (~1.5 KB per
    // estimator in all: the rebuilds -- a full sweep, O(r) -- stay rare.)
    const uint64_t pool = 16 * n + 32 * 1024;
    if (pool > 0x7FFFFFF0ull) return false;
    e.pool_cap = (uint32_t)pool;
    const uint64_t acap = pow2_at_least(2 * pool), pcap = acap;
    const uint64_t vcap = pow2_at_least(std::max<uint64_t>(pv_cap, 1024));
    if (acap > (1ull << 32) || pcap > (1ull << 32) || vcap > (1ull << 32)) return false;
    e.a_mask = (uint32_t)(acap - 1);
    e.p_mask = (uint32_t)(pcap - 1);
    e.pv_mask = (uint32_t)(vcap - 1);
    uint32_t **soa[] = {&e.J, &e.t1, &e.u, &e.v, &e.B, &e.K, &e.t2, &e.y, &e.fl, &e.ev, &e.queue};
    bool ok = true;
    for (uint32_t **p : soa) ok = ok && cudaMalloc(p, 4 * n) == cudaSuccess;
    ok = ok && cudaMalloc(&e.vs, 8 * n) == cudaSuccess &&
         cudaMalloc(&e.pool, 64 * pool) == cudaSuccess && cudaMalloc(&e.amap, 16 * acap) == cudaSuccess &&
         cudaMalloc(&e.pmap, 16 * pcap) == cudaSuccess && cudaMalloc(&e.pv, 16 * vcap) == cudaSuccess &&
         cudaMalloc(&e.ctr, 4 * kEdWords) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        ed_free(e);
    }
    return ok;
}

void ed_free(EdDev &e) {
    void *bufs[] = {e.J, e.t1, e.u, e.v, e.B, e.K, e.t2, e.y, e.fl, e.vs, e.ev, e.queue,
                    e.pool, e.amap, e.pmap, e.pv, e.ctr, e.seg};
    for (void *p : bufs) cudaFree(p);
    e = EdDev();
}

bool ed_alloc_seg(EdDev &e, uint64_t wcap) {
    cudaFree(e.seg);
    e.seg = nullptr;
    if (cudaMalloc(&e.seg, 16 * 2 * std::max<uint64_t>(wcap, 1)) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return true;
}

int launch_ed_init(const EdDev &e, cudaStream_t s) {
    const uint64_t items = std::max<uint64_t>({e.count, (uint64_t)e.a_mask + 1, (uint64_t)e.p_mask + 1,
                                               (uint64_t)e.pv_mask + 1});
    k_ed_init<<<grid_of(items, 16), 256, 0, s>>>(e);
    // rebuild threshold: more than 12 chunks per estimator in use in any stripe (see ed_alloc)
    const uint64_t n = std::max<uint64_t>(e.count, 1);
    k_ed_set_thr<<<1, 1, 0, s>>>(e.ctr, (uint32_t)((12 * n + 1024) / kEdStripes));
    return 2;
}

int ed_rehash_pv(EdDev &e, uint64_t new_cap, cudaStream_t s) {
    new_cap = pow2_at_least(new_cap);
    if (new_cap > (1ull << 32)) return -1;
    uint4 *pv = nullptr;
    if (cudaMalloc(&pv, 16 * new_cap) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    uint32_t *err = nullptr;
    if (cudaMalloc(&err, 4) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(pv);
        return -1;
    }
    cudaMemsetAsync(err, 0, 4, s);
    k_ed_fill_pv<<<grid_of(new_cap, 16), 256, 0, s>>>(pv, new_cap);
    const uint64_t old_n = (uint64_t)e.pv_mask + 1;
    k_ed_rehash<<<grid_of(old_n, 16), 256, 0, s>>>(e.pv, old_n, pv, (uint32_t)(new_cap - 1), err);
    uint32_t h = 0;
    const bool ok = cudaMemcpyAsync(&h, err, 4, cudaMemcpyDeviceToHost, s) == cudaSuccess &&
                    cudaStreamSynchronize(s) == cudaSuccess && h == 0;
    cudaFree(err);
    if (!ok) {
        cudaGetLastError();
        cudaFree(pv);
        return -1;
    }
    cudaFree(e.pv);
    e.pv = pv;
    e.pv_mask = (uint32_t)(new_cap - 1);
    return 0;
}

static EdIdx ed_idx(const IndexBufs &ix, const BatchArgs &a) {
    return EdIdx{Lookup{ix.E, ix.vt, ix.vslice, a.g.bv, ix.pt, pair_groups(a.g.w), 0u}, ix.segS, ix.apos, ix.pslot,
                 ix.ctr, ix.desc, a.g.w};
}

int launch_ed_batch(const IndexBufs &ix, const BatchArgs &a, const EdDev &e, unsigned long long *stats, bool post,
                    cudaStream_t s, const KRec &kr) {
    const EdIdx I = ed_idx(ix, a);
    const uint32_t g_arcs = grid_of(2ull * a.g.w, 8), g_spread = std::max<uint32_t>(g_arcs, (uint32_t)sm_count() * 4);
    const uint32_t g_items = std::max<uint32_t>(grid_of(4ull * a.g.w, 8), (uint32_t)sm_count() * 4);
    if (!post) {  // fast path: vertex work and watch lookups in one kernel, the degrees applied by k_ed_process
        kr.beg(K_ED_FRONT, s);
        k_ed_front<<<g_items, 256, 0, s>>>(I, e, a.S, stats);
        kr.end(K_ED_FRONT, s);
        kr.beg(K_ED_PROCESS, s);
        k_ed_process<<<(uint32_t)sm_count() * 4, 256, 0, s>>>(I, e, a.S);
        kr.end(K_ED_PROCESS, s);
        return 2;
    }
    kr.beg(K_ED_PRE, s);
    k_ed_pre<<<g_spread, 256, 0, s>>>(I, e, a.S, stats);
    kr.end(K_ED_PRE, s);
    kr.beg(K_ED_TRIGGER, s);
    k_ed_trigger<<<g_items, 256, 0, s>>>(I, e);
    kr.end(K_ED_TRIGGER, s);
    kr.beg(K_ED_PROCESS, s);
    k_ed_process<<<(uint32_t)sm_count() * 4, 256, 0, s>>>(I, e, a.S);
    kr.end(K_ED_PROCESS, s);
    kr.beg(K_ED_POST, s);
    k_ed_post<<<g_arcs, 256, 0, s>>>(I, e);
    kr.end(K_ED_POST, s);
    return 4;
}

#ifdef TC_ED_CLOCKS
extern "C" int tc_debug_ed_clocks(uint32_t *out, uint32_t cap, int reset) {
    uint32_t n = 0;
    cudaMemcpyFromSymbol(&n, g_edclk_n, 4);
    n = n < cap ? n : cap;
    cudaMemcpyFromSymbol(out, g_edclk, 32ull * n);
    if (reset) {
        const uint32_t z = 0;
        cudaMemcpyToSymbol(g_edclk_n, &z, 4);
    }
    return (int)n;
}
#endif

int launch_ed_export(const EdDev &e, const StateBufs &st, cudaStream_t s) {
    if (!e.count) return 0;
    k_ed_export<<<grid_of(e.count, 16), 256, 0, s>>>(e, st.r1, st.p1, st.r2, st.p2, st.cf);
    return 1;
}

}  // namespace tcb

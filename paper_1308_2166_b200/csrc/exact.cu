// exact.cu -- tc_exact_triangles (include/tc.h): tau = |T(G)|, the number of triangles of a simple
// undirected graph (definition, §2), on the GPU.  It is the ground truth of the accuracy
// study (the paper's MD% methodology) -- not part of the
// per-batch estimator path, and independent of it (no shared kernels or tables).
//
// Method (degree-ordered wedge closing, restated from the textbook "forward" algorithm):
//   1. every edge {u, v} becomes two arcs; the arcs are sorted by (source, target) (CUB radix sort on a
//      packed key of 2b bits, b = bits of the largest id), which groups each vertex's neighbours, sorted;
//      equal neighbouring keys are duplicate edges (TC_EDUP);
//   2. rank(x) = (deg x, x); each edge keeps the one arc that points up in rank (the oriented graph has
//      out-degrees <= sqrt(2m)), compacted stably, so every out-list stays sorted;
//   3. each triangle {a, b, c} with rank a < b < c is counted exactly once, by the arc a -> b, as the
//      element c of N+(a) ∩ N+(b).  Sources with long out-lists go vertex-centric: a CTA puts N+(a) into
//      a shared-memory hash set and probes it with every N+(b), b in N+(a); the other arcs intersect by
//      binary search, thread per arc (a warp per arc when both lists are long).
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "../../include/tc.h"

namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr uint32_t kErrInval = 1u, kErrLoop = 2u, kErrDup = 4u;
constexpr uint32_t kHeavy = 48;  // shorter-list length above which an arc goes to the warp kernel
constexpr uint32_t kBigDeg = 32;                       // sources with longer out-lists: vertex-centric kernel
constexpr uint32_t kSetMax = 1u << 15;                 // largest shared-memory set (slots; 128 KB)
constexpr uint32_t kSetDegMax = kSetMax / 4 * 3;       // ... holds out-lists up to load 3/4
constexpr int kVThreads = 512;
constexpr int kThreads = 256;

inline uint32_t grid_for(uint64_t n, int per_sm_ctas = 8) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t need = (n + kThreads - 1) / kThreads;
    const uint64_t cap = (uint64_t)sms * per_sm_ctas;
    return (uint32_t)(need < cap ? (need ? need : 1) : cap);
}

// err bits and the largest vertex id
__global__ void __launch_bounds__(kThreads) kx_scan_edges(const uint2 *__restrict__ E, uint64_t m, uint32_t *w) {
    uint32_t bad = 0, mx = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint2 e = E[i];
        if (e.x == kFull || e.y == kFull) bad |= kErrInval;
        else if (e.x == e.y) bad |= kErrLoop;
        mx = max(mx, max(e.x == kFull ? 0u : e.x, e.y == kFull ? 0u : e.y));
    }
    bad = __reduce_or_sync(kFull, bad);
    mx = __reduce_max_sync(kFull, mx);
    if ((threadIdx.x & 31u) == 0) {
        if (bad) atomicOr(&w[0], bad);
        atomicMax(&w[1], mx);
    }
}

__global__ void __launch_bounds__(kThreads) kx_arcs(const uint2 *__restrict__ E, uint64_t m, uint32_t b,
                                                    uint64_t *__restrict__ keys) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint2 e = E[i];
        reinterpret_cast<ulonglong2 *>(keys)[i] =
            make_ulonglong2(((uint64_t)e.x << b) | e.y, ((uint64_t)e.y << b) | e.x);
    }
}

// head[j] = arc j starts its source's run; duplicate arcs (equal keys) flag TC_EDUP
__global__ void __launch_bounds__(kThreads) kx_heads(const uint64_t *__restrict__ keys, uint64_t n, uint32_t b,
                                                     uint32_t *__restrict__ head, uint32_t *w) {
    uint32_t dup = 0;
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[j];
        const uint64_t p = j ? keys[j - 1] : ~0ull;
        head[j] = (j == 0 || (k >> b) != (p >> b)) ? 1u : 0u;
        dup |= (j && k == p) ? kErrDup : 0u;
    }
    dup = __reduce_or_sync(kFull, dup);
    if (dup && (threadIdx.x & 31u) == 0) atomicOr(&w[0], dup);
}

// vertex table: for the run heads, off[vid] = first arc, vert[vid] = the vertex id
__global__ void __launch_bounds__(kThreads) kx_runs(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ head,
                                                    const uint32_t *__restrict__ vinc, uint64_t n, uint32_t b,
                                                    uint32_t *__restrict__ off, uint32_t *__restrict__ vert) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
        if (head[j]) {
            const uint32_t v = vinc[j] - 1u;
            off[v] = (uint32_t)j;
            vert[v] = (uint32_t)(keys[j] >> b);
        }
        if (j == n - 1) off[vinc[j]] = (uint32_t)n;  // off[D] = n
    }
}

__device__ __forceinline__ uint32_t find_vid(const uint32_t *__restrict__ vert, uint32_t D, uint32_t x) {
    uint32_t lo = 0, hi = D;  // vert is strictly increasing; x is present
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(vert + mid) <= x) lo = mid;
        else hi = mid;
    }
    return lo;
}

// orientation: keep arc u -> v iff (deg u, u) < (deg v, v); dst[j] = vid of v
__global__ void __launch_bounds__(kThreads) kx_orient(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ vinc,
                                                      const uint32_t *__restrict__ off, const uint32_t *__restrict__ vert,
                                                      uint64_t n, uint32_t b, uint32_t *__restrict__ keep,
                                                      uint32_t *__restrict__ dst) {
    const uint64_t mask = (1ull << b) - 1ull;
    const uint32_t D = vinc[n - 1];
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[j];
        const uint32_t u = (uint32_t)(k >> b), v = (uint32_t)(k & mask);
        const uint32_t vu = vinc[j] - 1u, vv = find_vid(vert, D, v);
        const uint32_t du = off[vu + 1] - off[vu], dv = off[vv + 1] - off[vv];
        keep[j] = (du < dv || (du == dv && u < v)) ? 1u : 0u;
        dst[j] = vv;
    }
}

__global__ void __launch_bounds__(kThreads) kx_compact(const uint32_t *__restrict__ keep, const uint32_t *__restrict__ kpos,
                                                       const uint32_t *__restrict__ dst, const uint32_t *__restrict__ vinc,
                                                       uint64_t n, uint32_t *__restrict__ adj, uint32_t *__restrict__ src) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
        if (keep[j]) {
            const uint32_t q = kpos[j];
            adj[q] = dst[j];
            src[q] = vinc[j] - 1u;
        }
    }
}

// out-list starts: offp[vid] = kept arcs before the vertex's first arc; offp[D] = m
__global__ void __launch_bounds__(kThreads) kx_outoff(const uint32_t *__restrict__ off, const uint32_t *__restrict__ kpos,
                                                      const uint32_t *__restrict__ pD, uint64_t m, uint32_t *__restrict__ offp) {
    const uint32_t D = *pD;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v <= D; v += (uint64_t)gridDim.x * blockDim.x)
        offp[v] = v < D ? kpos[off[v]] : (uint32_t)m;
}

// elements of S[0, ns) present in L[0, nl) (both sorted, distinct)
__device__ __forceinline__ uint32_t count_in(const uint32_t *__restrict__ S, uint32_t ns, const uint32_t *__restrict__ L,
                                             uint32_t nl, uint32_t s0, uint32_t ds) {
    uint32_t c = 0, lo = 0;
    for (uint32_t i = s0; i < ns; i += ds) {
        const uint32_t x = __ldg(S + i);
        uint32_t a = lo, z = nl;  // first L[k] >= x, searching from the last hit on (S ascends)
        while (a < z) {
            const uint32_t mid = (a + z) >> 1;
            if (__ldg(L + mid) < x) a = mid + 1;
            else z = mid;
        }
        if (a < nl && __ldg(L + a) == x) ++c;
        if (ds == 1) lo = a;
    }
    return c;
}

__global__ void __launch_bounds__(kThreads) kx_count(const uint32_t *__restrict__ adj, const uint32_t *__restrict__ src,
                                                     const uint32_t *__restrict__ offp, uint64_t m,
                                                     unsigned long long *tau, uint32_t *heavy, uint32_t *nheavy) {
    uint32_t c = 0;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < m; q += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t a = src[q], x = adj[q];
        const uint32_t a0 = offp[a], a1 = offp[a + 1], x0 = offp[x], x1 = offp[x + 1];
        const uint32_t na = a1 - a0, nx = x1 - x0;
        if (na > kBigDeg && na <= kSetDegMax) continue;  // kx_count_vertex's source
        if (min(na, nx) > kHeavy) {
            heavy[atomicAdd(nheavy, 1u)] = (uint32_t)q;
            continue;
        }
        c += na <= nx ? count_in(adj + a0, na, adj + x0, nx, 0, 1) : count_in(adj + x0, nx, adj + a0, na, 0, 1);
    }
    c = __reduce_add_sync(kFull, c);
    if ((threadIdx.x & 31u) == 0 && c) atomicAdd(tau, (unsigned long long)c);
}

// warp per heavy arc: lanes stride over the shorter list
__global__ void __launch_bounds__(kThreads) kx_count_heavy(const uint32_t *__restrict__ adj, const uint32_t *__restrict__ src,
                                                           const uint32_t *__restrict__ offp, const uint32_t *__restrict__ heavy,
                                                           const uint32_t *__restrict__ nheavy, unsigned long long *tau) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t nh = *nheavy;
    uint32_t c = 0;
    for (uint32_t h = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; h < nh; h += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t q = heavy[h];
        const uint32_t a = src[q], x = adj[q];
        const uint32_t a0 = offp[a], a1 = offp[a + 1], x0 = offp[x], x1 = offp[x + 1];
        const uint32_t na = a1 - a0, nx = x1 - x0;
        c += na <= nx ? count_in(adj + a0, na, adj + x0, nx, lane, 32) : count_in(adj + x0, nx, adj + a0, na, lane, 32);
    }
    c = __reduce_add_sync(kFull, c);
    if (lane == 0 && c) atomicAdd(tau, (unsigned long long)c);
}

// the sources kx_count_vertex takes (kBigDeg < out-degree <= kSetDegMax), and the largest out-degree
__global__ void __launch_bounds__(kThreads) kx_bigsrc(const uint32_t *__restrict__ offp, const uint32_t *__restrict__ pD,
                                                      uint32_t *__restrict__ list, uint32_t *w) {
    const uint32_t D = *pD;
    uint32_t mx = 0;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < D; v += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t deg = offp[v + 1] - offp[v];
        mx = max(mx, deg);
        if (deg > kBigDeg && deg <= kSetDegMax) list[atomicAdd(&w[6], 1u)] = (uint32_t)v;
    }
    mx = __reduce_max_sync(kFull, mx);
    if ((threadIdx.x & 31u) == 0) atomicMax(&w[7], mx);
}

// CTA per listed source a (taken by ticket): N+(a) into a shared-memory hash set, then warps over x in N+(a)
// and lanes over N+(x), counting the members (or, when N+(x) is much the longer list, binary-searching
// N+(a)'s members in it) -- every triangle whose lowest vertex is a, once.
__global__ void __launch_bounds__(kVThreads) kx_count_vertex(const uint32_t *__restrict__ adj, const uint32_t *__restrict__ offp,
                                                             const uint32_t *__restrict__ list, uint32_t *w, uint32_t S,
                                                             unsigned long long *tau) {
    extern __shared__ uint32_t set[];
    __shared__ uint32_t s_i;
    constexpr uint32_t NW = kVThreads / 32;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t nbig = w[6];
    uint32_t c = 0;
    while (true) {
        if (threadIdx.x == 0) s_i = atomicAdd(&w[8], 1u);
        __syncthreads();
        const uint32_t i = s_i;
        __syncthreads();  // s_i is read by all before thread 0 takes the next ticket
        if (i >= nbig) break;
        const uint32_t a = list[i], a0 = offp[a], na = offp[a + 1] - a0;
        uint32_t T = 1;
        while (T < 2 * na && T < S) T <<= 1;
        const uint32_t mask = T - 1u, sh = 32u - (31u - __clz(T));
        for (uint32_t j = threadIdx.x; j < T; j += kVThreads) set[j] = kFull;
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < na; j += kVThreads) {
            const uint32_t y = adj[a0 + j];
            uint32_t h = T > 1 ? (y * 0x9E3779B1u) >> sh : 0u;
            while (atomicCAS(&set[h], kFull, y) != kFull) h = (h + 1u) & mask;
        }
        __syncthreads();
        for (uint32_t j = warp; j < na; j += NW) {
            const uint32_t x = adj[a0 + j], x0 = offp[x], nx = offp[x + 1] - x0;
            if (nx > na * (32u - __clz(nx))) {  // N+(x) much longer: binary-search N+(a)'s members in it
                c += count_in(adj + a0, na, adj + x0, nx, lane, 32);
                continue;
            }
            for (uint32_t t = lane; t < nx; t += 32) {
                const uint32_t y = __ldg(adj + x0 + t);
                uint32_t h = T > 1 ? (y * 0x9E3779B1u) >> sh : 0u;
                while (true) {
                    const uint32_t k = set[h];
                    if (k == y) {
                        ++c;
                        break;
                    }
                    if (k == kFull) break;
                    h = (h + 1u) & mask;
                }
            }
        }
        __syncthreads();
    }
    c = __reduce_add_sync(kFull, c);
    if (lane == 0 && c) atomicAdd(tau, (unsigned long long)c);
}

struct Scratch {
    cudaStream_t s = nullptr;
    void *p[10] = {};
    ~Scratch() {
        for (void *q : p)
            if (q) cudaFree(q);
        if (s) cudaStreamDestroy(s);
    }
};

}  // namespace

#define XK(call)                                                                                \
    do {                                                                                        \
        const cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) {                                                                \
            if (getenv("TC_DEBUG")) fprintf(stderr, "exact.cu:%d: %s\n", __LINE__, cudaGetErrorString(e_)); \
            cudaGetLastError();                                                                 \
            return TC_ECUDA;                                                                    \
        }                                                                                       \
    } while (0)
#define XA(ptr, bytes)                                        \
    do {                                                      \
        if (cudaMalloc(&(ptr), (bytes)) != cudaSuccess) {     \
            cudaGetLastError();                               \
            return TC_ENOMEM;                                 \
        }                                                     \
    } while (0)

extern "C" int tc_exact_triangles(const tc_edge *edges, uint64_t m, uint64_t *tau, double *device_ms) {
    if (!tau || (m && !edges) || m >= (1ull << 31)) return TC_EINVAL;
    *tau = 0;
    if (device_ms) *device_ms = 0.0;
    if (m == 0) return TC_OK;
    Scratch x;
    XK(cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking));
    const cudaStream_t s = x.s;
    const uint64_t n = 2 * m;
    // buffers: E (m uint2), keys + alt (n u64 each), keep | kpos (2n u32), off / vert / offp (n + 1 u32 each),
    // words; after the sort the alternate key buffer holds head | vinc, and the sorted keys (once dead)
    // adj | src | heavy (m u32 each)
    uint2 *E = nullptr;
    uint64_t *keys = nullptr, *alt = nullptr;
    uint32_t *w = nullptr;  // [0] error bits, [1] max id, [2] heavy count, [3] D; [4..5] tau
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, edges) != cudaSuccess) {
        cudaGetLastError();
        attr.type = cudaMemoryTypeUnregistered;
    }
    int dev = 0;
    XK(cudaGetDevice(&dev));
    const bool on_device = (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged) && attr.device == dev;
    if (attr.type == cudaMemoryTypeDevice && attr.device != dev) return TC_EINVAL;
    if (on_device) {
        E = reinterpret_cast<uint2 *>(const_cast<tc_edge *>(edges));
    } else {
        XA(x.p[0], 8 * m);
        E = static_cast<uint2 *>(x.p[0]);
        XK(cudaMemcpyAsync(E, edges, 8 * m, cudaMemcpyHostToDevice, s));
    }
    XA(x.p[1], 8 * n);
    XA(x.p[2], 8 * n);
    XA(x.p[3], 64);
    XA(x.p[8], 8 * n);        // keep | kpos
    XA(x.p[5], 4 * (n + 1));  // off, vert, offp: D + 1 <= n + 1 entries each
    XA(x.p[6], 4 * (n + 1));
    XA(x.p[7], 4 * (n + 1));
    uint32_t *off = static_cast<uint32_t *>(x.p[5]), *vert = static_cast<uint32_t *>(x.p[6]),
             *offp = static_cast<uint32_t *>(x.p[7]);
    keys = static_cast<uint64_t *>(x.p[1]);
    alt = static_cast<uint64_t *>(x.p[2]);
    w = static_cast<uint32_t *>(x.p[3]);
    cudaEvent_t e0, e1;
    XK(cudaEventCreate(&e0));
    if (cudaEventCreate(&e1) != cudaSuccess) {
        cudaEventDestroy(e0);
        return TC_ECUDA;
    }
    struct EvGuard {
        cudaEvent_t a, b;
        ~EvGuard() {
            cudaEventDestroy(a);
            cudaEventDestroy(b);
        }
    } eg{e0, e1};
    XK(cudaEventRecord(e0, s));
    XK(cudaMemsetAsync(w, 0, 64, s));
    kx_scan_edges<<<grid_for(m), kThreads, 0, s>>>(E, m, w);
    uint32_t hw[2];
    XK(cudaMemcpyAsync(hw, w, 8, cudaMemcpyDeviceToHost, s));
    XK(cudaStreamSynchronize(s));
    if (hw[0] & kErrInval) return TC_EINVAL;
    if (hw[0] & kErrLoop) return TC_ESELFLOOP;
    const uint32_t b = 32 - __builtin_clz(hw[1] | 1u);  // bits of the largest id (>= 1)
    kx_arcs<<<grid_for(m), kThreads, 0, s>>>(E, m, b, keys);
    // 1. sort the arcs by (source, target)
    cub::DoubleBuffer<uint64_t> db(keys, alt);
    size_t tmp_bytes = 0;
    XK(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, db, (int64_t)n, 0, (int)(2 * b), s));
    size_t scan_bytes = 0;
    XK(cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, (uint32_t *)nullptr, (uint32_t *)nullptr, (int64_t)n, s));
    XA(x.p[4], (tmp_bytes > scan_bytes ? tmp_bytes : scan_bytes) + 256);
    void *tmp = x.p[4];
    size_t tb = tmp_bytes;
    XK(cub::DeviceRadixSort::SortKeys(tmp, tb, db, (int64_t)n, 0, (int)(2 * b), s));
    const uint64_t *sk = db.Current();
    uint32_t *fr = reinterpret_cast<uint32_t *>(db.Alternate());  // two n-u32 arrays
    uint32_t *head = fr, *vinc = fr + n;
    kx_heads<<<grid_for(n), kThreads, 0, s>>>(sk, n, b, head, w);
    tb = scan_bytes;
    XK(cub::DeviceScan::InclusiveSum(tmp, tb, head, vinc, (int64_t)n, s));
    kx_runs<<<grid_for(n), kThreads, 0, s>>>(sk, head, vinc, n, b, off, vert);
    // 2. orientation by (degree, id), stable compaction
    uint32_t *keep = static_cast<uint32_t *>(x.p[8]), *dst = head;  // head is dead after kx_runs
    kx_orient<<<grid_for(n), kThreads, 0, s>>>(sk, vinc, off, vert, n, b, keep, dst);
    uint32_t *kpos = keep + n;
    tb = scan_bytes;
    XK(cub::DeviceScan::ExclusiveSum(tmp, tb, keep, kpos, (int64_t)n, s));
    // the sorted keys are dead: adj | src | heavy live in their memory
    uint32_t *adj = reinterpret_cast<uint32_t *>(const_cast<uint64_t *>(sk)), *src = adj + m, *heavy = adj + 2 * m;
    kx_compact<<<grid_for(n), kThreads, 0, s>>>(keep, kpos, dst, vinc, n, adj, src);
    kx_outoff<<<grid_for(n + 1), kThreads, 0, s>>>(off, kpos, vinc + n - 1, m, offp);
    // 3. wedge closing: sources with long out-lists vertex-centric (a shared-memory set of N+(a)), the rest
    //    arc by arc (binary search; a warp per arc when both lists are long)
    unsigned long long *dtau = reinterpret_cast<unsigned long long *>(w + 4);
    uint32_t *big = keep;  // keep | kpos are dead after kx_outoff: the source list
    kx_bigsrc<<<grid_for(n + 1), kThreads, 0, s>>>(offp, vinc + n - 1, big, w);
    kx_count<<<grid_for(m), kThreads, 0, s>>>(adj, src, offp, m, dtau, heavy, w + 2);
    kx_count_heavy<<<grid_for(32ull * m, 8), kThreads, 0, s>>>(adj, src, offp, heavy, w + 2, dtau);
    uint32_t hb[2];
    XK(cudaMemcpyAsync(hb, w + 6, 8, cudaMemcpyDeviceToHost, s));
    XK(cudaStreamSynchronize(s));
    if (hb[0]) {
        uint32_t S = 1;
        while (S < 2 * std::min(hb[1], kSetDegMax) && S < kSetMax) S <<= 1;
        XK(cudaFuncSetAttribute(kx_count_vertex, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(4 * S)));
        int dev2 = 0, sms = 148, per = 1;
        XK(cudaGetDevice(&dev2));
        XK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev2));
        XK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kx_count_vertex, kVThreads, 4 * S));
        const uint32_t grid = std::min<uint32_t>(hb[0], (uint32_t)(sms * std::max(per, 1)));
        kx_count_vertex<<<grid, kVThreads, 4 * S, s>>>(adj, offp, big, w, S, dtau);
    }
    XK(cudaEventRecord(e1, s));
    unsigned long long ht = 0;
    XK(cudaMemcpyAsync(&ht, dtau, 8, cudaMemcpyDeviceToHost, s));
    XK(cudaMemcpyAsync(hw, w, 4, cudaMemcpyDeviceToHost, s));
    XK(cudaStreamSynchronize(s));
    XK(cudaGetLastError());
    if (hw[0] & kErrDup) return TC_EDUP;  // the count above is then meaningless
    float ms = 0.f;
    XK(cudaEventElapsedTime(&ms, e0, e1));
    if (device_ms) *device_ms = ms;
    *tau = ht;
    return TC_OK;
}

// event.h -- the event-driven estimator mode (reading R17, §10 row 4).
// Host-side, internal.
//
// Per estimator the mode keeps the sequential neighborhood-sampling state plus the two
// skip-sampled replacement points: J, the time at which f1 is next replaced, and K, the adjacency count at which
// f2 is next replaced; chi is kept lazily as deg(u) + deg(v) - B with persistent vertex degrees.  A batch visits
// only the estimators it can change, found through watch lists keyed by the exact event that would change them:
//   (kJKey, J)           -- the batch contains stream time J;
//   (x, theta)           -- vertex x reaches degree theta (the two halves of the remaining adjacency count);
//   closing pair (a, b)  -- the batch contains the closing edge of (f1, f2).
// Batches early in the stream (m < 8 w, where most estimators change anyway) and every batch after
// the watch-node pool passed its threshold are full sweeps: every estimator is processed and all watch lists are
// rebuilt.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace tcb {

constexpr uint32_t kEdInf = 0xFFFFFFFFu;   // "never" (beyond HMAX = 2^31 - 1)
constexpr uint32_t kEdHMax = 0x7FFFFFFFu;
constexpr uint32_t kEdDegMax = (1u << 30) - 1u;  // reading R17c
constexpr uint32_t kEdNil = 0xFFFFFFFFu;
constexpr uint32_t kJKey = 0xFFFFFFFFu;    // the reserved vertex id: (kJKey, t) watches stream time t

// counters (EdDev::ctr)
constexpr int kEdPool = 0;     // (unused: the chunk pool is striped, kEdStripe0 ..)
constexpr int kEdQueue = 1;    // estimators queued in this batch
constexpr int kEdFull = 2;     // this batch is a full sweep (set by k_desc)
constexpr int kEdPVN = 3;      // vertices in the persistent table
constexpr int kEdThr = 4;      // per-stripe chunk threshold of a rebuild
constexpr int kEdVisited = 5;  // estimators processed (all batches)
constexpr int kEdEvents = 6;   // f1 / f2 replacements (all batches)
constexpr int kEdSweeps = 7;   // full sweeps
constexpr int kEdStripe0 = 8;  // chunks in use per stripe: the pool is 32 stripes of pool_cap / 32 chunks, warp w
constexpr uint32_t kEdStripes = 32;  // allocating from stripe w mod 32 (one hot counter would serialise them)
constexpr int kEdWords = kEdStripe0 + (int)kEdStripes;

struct EdDev {
    // estimator SoA: J, f1 = (u, v) at time t1 (0: none), B = deg_t1(u) + deg_t1(v), K, f2 at time t2 = (shared,
    // y) with fl bit 1 = "shared is v", fl bit 0 = closed; ev = random words used; vs = {watch versions (time,
    // degree, pair: 10 / 11 / 11 bits), last batch the estimator was queued in}
    uint32_t *J, *t1, *u, *v, *B, *K, *t2, *y, *fl, *ev;
    uint2 *vs;
    uint64_t count, first, seed;
    uint4 *pv;        // persistent vertices {id, degree, closed estimators with it as an f1 endpoint, 0}
    uint32_t pv_mask;
    uint4 *amap;      // {key lo, key hi, head, 0}: (vertex, degree threshold) and (kJKey, time) watches
    uint32_t a_mask;
    uint4 *pmap;      // closing-pair watches
    uint32_t p_mask;
    uint4 *pool;      // watch chunks: 64 B = 7 nodes {estimator, kind << 30 | version} + the next chunk (word 14)
    uint32_t pool_cap;  // chunks (kEdStripes stripes of pool_cap / kEdStripes)
    uint32_t *queue;  // [count] estimators to process in this batch
    uint4 *seg;       // [2 wcap] at each vertex segment's first slot: {degree before the batch, pv slot, degree in
                      // the batch, segment start}
    uint32_t *ctr;
};

// Device allocations of the mode for `count` estimators (pool, maps, SoA) and an initial vertex capacity.
bool ed_alloc(EdDev &e, uint64_t count, uint64_t first, uint64_t seed, uint64_t pv_cap);
void ed_free(EdDev &e);
bool ed_alloc_seg(EdDev &e, uint64_t wcap);  // with the index (2 wcap entries)
// Fresh state: every estimator empty with J = 1, empty tables, counters zero.
int launch_ed_init(const EdDev &e, cudaStream_t s);
// Re-insert the persistent vertices into a table of new_cap slots (replaces e.pv / e.pv_mask on success).
int ed_rehash_pv(EdDev &e, uint64_t new_cap, cudaStream_t s);
// The kernels of a batch (after the index).  Fast path (no vertex degree can reach the limit; descriptor pad bit
// 2): k_ed_front (vertex records + every watch lookup) and k_ed_process (which also applies the degrees).  When
// `post` (the limit can be reached, so the batch may still be rejected after the index): k_ed_pre checks it,
// k_ed_trigger looks the watches up, k_ed_process, and k_ed_post applies the degrees once the batch is accepted.  stats: the bulk state's event counters
// (tc_stats): out[2] += distinct vertices of the batch, out[3] += 1.
int launch_ed_batch(const IndexBufs &ix, const BatchArgs &a, const EdDev &e, unsigned long long *stats, bool post,
                    cudaStream_t s, const KRec &kr);
// The NBSI view of the state (r1, p1, r2, p2, chi | closed) into the bulk state buffers.
int launch_ed_export(const EdDev &e, const StateBufs &st, cudaStream_t s);

}  // namespace tcb

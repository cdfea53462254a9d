// kernels.h -- launch wrappers of the per-batch pipeline (kernels.cu).  Host-side, internal.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "index.cuh"

namespace tcb {

struct IndexBufs {
    uint64_t wcap = 0;             // edges the buffers hold
    uint64_t tiles_cap = 0;        // count/scatter tiles
    uint2 *E = nullptr;            // [wcap] normalised edges
    uint4 *arcs = nullptr;         // [2 wcap] vertex-bucketed arcs {vertex, k<<1|side, neighbour, 0}, arrival
                                   // order per bucket
    uint4 *arcs2 = nullptr;        // [2 wcap] arcs of the split sub-buckets (when Geometry::bs > 0)
    uint32_t *vstart2 = nullptr;   // [2^15 + 1] sub-bucket starts
    uint2 *scratch = nullptr;      // [2 wcap] sort scratch of oversized vertex buckets
    uint2 *segS = nullptr;         // [2 wcap] arcs {k<<1|side, neighbour} grouped by vertex
    uint2 *apos = nullptr;         // [wcap] partition positions of edge k's arcs {lo side, hi side} (k_scatter)
    uint2 *pslot = nullptr;        // [2 wcap] by partition position: {slot in segS, segment end} (vertex kernels)
    VSlot *vt = nullptr;           // [4 wcap] vertex-table slices (bucket b at 2 * start_b)
    uint2 *vslice = nullptr;       // [4096] {offset, size}
    uint32_t *vperm = nullptr;     // [4096] vertex buckets in processing order (oversized first)
    uint32_t *vdefer = nullptr;    // [4096] large buckets k_vhub hands to k_vbig
    uint2 *pt = nullptr;           // [4 ceil(wcap / 2)] pair slots {k, fp}, groups of 4
    uint32_t *cntV = nullptr;      // [4096 * tiles] per-(bucket, tile) arc counts
    uint32_t *offV = nullptr;      // [4096 * tiles] the tile's offset inside the bucket
    uint16_t *arank = nullptr;     // [2 wcap] rank of each arc among its tile's arcs of the same vertex bucket
    uint32_t *vstart = nullptr;    // [4097] vertex-bucket totals -> exclusive prefix
    uint32_t *ctr = nullptr;       // device counters (index.cuh kCtr*)
    uint32_t *filt = nullptr;      // [kFilterWords] small-batch filter over the batch's vertices
    uint32_t *pf = nullptr;        // [pf_words(wcap)] large-batch pair filter (index.cuh)
    uint2 *stage = nullptr;        // [wcap] H2D staging for host batches (two buffers, alternating)
    uint2 *stage2 = nullptr;
    BatchDesc *desc = nullptr;     // the per-batch descriptor (k_desc writes it; every kernel reads it)
};

constexpr int kNStats = 7;

// Split estimator pass (tc_tune TC_TUNE_SPLIT_KERNELS): one kernel per step of SURVEY.md §8(a) -- Ku1 level-1
// resample (a4), Ku2 adjacency count (a5), Ku3 level-2 select (a6), Ku4 closing-edge lookup (a7), Kr aggregation
// (a8) -- with each step's values kept per estimator for per-step parity and per-step timing.
struct StepBufs {
    uint64_t count = 0;
    uint32_t *j = nullptr;     // Step 1: replacement index in W, 0xFFFFFFFF = f1 retained
    uint64_t *xhi = nullptr;   // the Philox word of Step 2's draw
    uint32_t *chim = nullptr;  // chi^- (after Step 1)
    uint32_t *ld = nullptr, *rd = nullptr;      // rank(u->v), rank(v->u): chi^+ = ld + rd
    uint32_t *endU = nullptr, *endV = nullptr;  // segment ends of u and v
    uint64_t *d2 = nullptr;    // Step 2's draw over chi^- + chi^+ (UINT64_MAX: no draw)
    uint32_t *k2 = nullptr;    // batch position of the new f2 (0xFFFFFFFF: f2 kept)
};

struct StateBufs {
    uint64_t count = 0;
    uint2 *r1 = nullptr, *r2 = nullptr;
    uint32_t *cf = nullptr;  // chi in bits 0..30, closed flag in bit 31
    uint32_t *p1 = nullptr, *p2 = nullptr;  // 0-based global positions (< 2^31, reading R13); 0xFFFFFFFF = empty
    unsigned long long *S = nullptr;      // [2] closed-sum accumulators (double-buffered by batch parity)
    unsigned long long *stats = nullptr;  // [kNStats] fresh f1, replaced f2 of retained f1, sum of D, batches,
                                          // estimators the small-batch pass skipped, arcs / vertices of the
                                          // large-bucket kernels
};

// Bucket geometry of one batch (host-computed from w and the tuning knobs).
struct Geometry {
    uint32_t w;
    uint32_t tiles;    // ceil(w / kTileEdges)
    uint32_t bv;       // vertex bucket bits (= bp1 + bs)
    uint32_t bp1;      // partition bits (<= 12): the buckets of k_count / k_scatter
    uint32_t bs;       // split bits (k_split: each partition bucket into 2^bs sub-buckets; 0 = no split)
    uint32_t vcap;     // vertex buckets larger than this go to k_vhub (<= 2048)
    uint32_t sortcap;  // k_vbig: buckets larger than this take the chunked global-memory path (<= kVChunk)
    bool small_index;  // the whole index by one CTA (k_small_index; w <= kSmallIndexMax)
};

constexpr uint32_t kSmallIndexMaxBits = 8;  // k_small_index: at most 256 CTAs
constexpr uint32_t kSmallIndexMax = 4096;  // k_small_index: one CTA per vertex bucket of ~Tuning::small_index_arcs arcs (a bucket may
                                           // hold all 2 w arcs: hash path caps 4096 / 8192 at 256 / 512 threads)

// Launch-time values of a push.  The per-batch values (input pointer, m, batch index, pair tag, S slot) are
// NOT here: the kernels read them from the device descriptor (BatchDesc), so a captured graph of the launch
// sequence depends only on the batch shape (w and the flags below).
struct BatchArgs {
    uint64_t first;   // global id of local estimator 0
    uint64_t seed;
    unsigned long long *S;  // the two S accumulators (slot from the descriptor)
    bool small;       // small-batch estimator pass (filters built by k_pairs, k_update skips untouched estimators)
    Geometry g;
    bool pfilt = false;  // the pair filter: k_pairs fills it, Step 3 of k_update reads it before the pair table
};

// Batches of at most this many edges take the filtered small-batch estimator pass (filter load <= 1/16)
constexpr uint32_t kSmallBatchMax = 8192;  // measured break-even ~16384 on C5

struct Tuning {
    uint32_t small = 0;            // 0 auto (w <= kSmallBatchMax), 1 never, 2 always
    uint32_t vbucket_arcs = 1024;  // target arcs per vertex bucket
    uint32_t vcap = 2048;
    uint32_t sortcap = kVChunk;
    uint32_t split = 0;            // 1: the estimator pass as the split per-step kernels
    uint32_t small_index = 0;      // 0 auto (w <= kSmallIndexMax), 1 never, 2 always when w <= kSmallIndexMax
    uint32_t event_checked = 0;    // event mode: 1 = always the four-kernel path that checks the degree limit
    uint32_t pair_filter = 0;      // 0 auto (w >= kPairFilterMin), 1 never, 2 always (bulk fused pass, partitioned index)
    uint32_t small_index_arcs = 64;   // k_small_index: target arcs per CTA (vertex bucket), at most 2^kSmallIndexMaxBits CTAs
};

// Batches of at least kPairFilterMin (index.cuh) edges get the pair filter (below it the pair table is mostly
// L2-resident)

Geometry make_geometry(uint32_t w, const Tuning &t);

// Per-kernel profiling (tc_profile_kernels): ids match include/tc.h TC_KERNEL_*.
enum KernelId { K_COUNT = 0, K_SCAN_COLS, K_SCAN_TOT, K_SCATTER, K_SPLIT, K_PAIRS, K_VHUB, K_VBIG, K_VHASH, K_UPDATE,
                K_U1, K_U2, K_U3, K_U4, K_R, K_SMALL, K_ED_PRE, K_ED_TRIGGER, K_ED_PROCESS, K_ED_POST, K_ED_FRONT, K_NKERNELS };
struct KRec {
    cudaEvent_t *ev = nullptr;  // 2 K_NKERNELS events (begin, end) or null: no profiling
    uint32_t *used = nullptr;   // bit k set once kernel k's events were recorded in this push
    void beg(int k, cudaStream_t s) const {
        if (ev) cudaEventRecord(ev[2 * k], s);
    }
    void end(int k, cudaStream_t s) const {
        if (ev) {
            cudaEventRecord(ev[2 * k + 1], s);
            *used |= 1u << k;
        }
    }
};

// Each returns the number of kernel launches issued.
int launch_partition(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s, const KRec &kr = KRec());  // a1
int launch_pairs(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s, const KRec &kr = KRec());      // a3
int launch_vertices(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s, const KRec &kr = KRec());   // a2
int launch_small_index(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s, const KRec &kr = KRec());  // a1-a3
int launch_vertices_big(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s, const KRec &kr = KRec());  // a2 > vcap
#ifndef TC_BIG_CTAS
#define TC_BIG_CTAS 64
#endif
constexpr uint32_t kBigCTAs = TC_BIG_CTAS;
int launch_update(const IndexBufs &ix, const StateBufs &st, const BatchArgs &a, cudaStream_t s, const KRec &kr = KRec());
int launch_update_split(const IndexBufs &ix, const StateBufs &st, const StepBufs &sb, const BatchArgs &a, cudaStream_t s,
                        const KRec &kr = KRec());

// the push's first node; edctr: the event mode's counters (null in the bulk mode)
int launch_desc(const IndexBufs &ix, const BatchArgs &a, const BatchDesc &d, uint32_t *edctr, cudaStream_t s);
const void *desc_kernel();                                                  // its function (graph node lookup)

int launch_init_state(const StateBufs &st, cudaStream_t s);
int launch_group_sums(const StateBufs &st, uint64_t first, uint64_t N, uint32_t groups, unsigned long long *out,
                      cudaStream_t s);  // groups over global ids (first = global id of local 0, N = r)

int launch_test_draws(const uint64_t *n, const uint64_t *x, const uint64_t *id, const uint32_t *b, const uint32_t *base,
                      uint64_t seed, uint64_t count, uint64_t *out, cudaStream_t s);
int launch_test_philox(const uint32_t *ctr, const uint32_t *key, uint64_t count, uint32_t *out, cudaStream_t s);

int sm_count();
int set_kernel_attributes();  // dynamic shared memory limits on the current device

}  // namespace tcb

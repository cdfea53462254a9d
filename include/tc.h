/*
 * tc.h -- C ABI of the B200 bulk neighborhood-sampling triangle estimator
 *         (Tangwongsan, Pavan, Tirthapura, arXiv:1308.2166; "coordinated bulk parallel").
 *
 * The library maintains r independent estimators, each a tuple (f1, f2, f3, chi) satisfying
 * the neighborhood sampling invariant NBSI (§3.1), over a stream of undirected
 * simple-graph edges that arrives in batches W (§4.1).  One call to
 * tc_push_batch() is one run of bulkUpdateAll: Step 1 level-1 reservoir
 * (PAPER.md:520-538), Step 2 level-2 edges and chi, Step 3 closing edges
 * (PAPER.md:835-845), for all estimators of this handle, on the GPU.
 *
 * Conventions (all calls):
 *  - Vertex ids are uint32; 0xFFFFFFFF is reserved (it encodes "empty") and is rejected.
 *    The paper's batch is "an array of a pair of int's".
 *  - Estimator ids are global, 0 .. r-1; a handle owns a contiguous shard [first, first+count)
 *    (tc_create owns all of them).  All randomness is Philox4x32-10 keyed by (seed) with counter
 *    (id, batch index, draw word) -- DESIGN.md reading R7 -- so a shard's states do not depend on
 *    how the estimators are split across handles / GPUs.
 *  - Errors: functions returning int return TC_OK (0) or a negative TC_E* code.  A rejected batch
 *    leaves every estimator and the counters unchanged (all-or-nothing).
 *  - Not thread-safe per handle (single writer); distinct handles are independent.
 *  - Stream: every handle owns one CUDA stream on its device; all device work is issued on it.
 */
#ifndef TC_B200_H
#define TC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tc_ctx tc_ctx; /* opaque, owned by the library */

/* One stream element: an undirected edge {u, v}, any orientation.  8 bytes, layout == CUDA uint2. */
typedef struct {
    uint32_t u, v;
} tc_edge;

enum {
    TC_OK = 0,
    TC_EINVAL = -1,      /* bad argument, or a vertex id 0xFFFFFFFF in the batch            */
    TC_ENOMEM = -2,      /* device or host allocation failed                                */
    TC_ESELFLOOP = -3,   /* u == v in the batch (the graph is simple)          */
    TC_EDUP = -4,        /* the same undirected pair twice in one batch  */
    TC_EOVERFLOW = -5,   /* chi overflow (reading R13), or the library limit m <= 2^31-1    */
    TC_ECUDA = -6,       /* a CUDA call failed; the handle is poisoned                      */
    TC_ENCCL = -7,       /* NCCL unavailable or failed; the communicator is aborted and the
                            handle poisoned                                                 */
    TC_ESTATE = -8,      /* handle poisoned by an earlier asynchronous error               */
    TC_EPARSE = -9,      /* malformed edge-list line (tc_parse_edges / tc_ingest_file)      */
    TC_EIO = -10,        /* the edge-list file cannot be opened or read                     */
    TC_EINTERNAL = -11   /* a bounds check of a -DTC_CHECKED build failed (never in release) */
};

/* tc_create -- r estimators (ids 0..r-1) on the current CUDA device, all "empty" (f1 = f2 = f3 =
 * empty, chi = 0), m = 0.  seed keys the Philox stream.  Returns NULL on failure (r == 0, no device,
 * out of memory); tc_last_error() then says why. */
tc_ctx *tc_create(uint64_t r, uint64_t seed);

/* tc_create_shard -- estimators [first, first+count) of r, on CUDA device `device` (-1 = current).
 * w_max_hint preallocates the per-batch index for batches up to that many edges (0 = grow on
 * demand).  count may be 0 (an idle shard still tracks m).  NULL on failure. */
tc_ctx *tc_create_shard(uint64_t r, uint64_t seed, uint64_t first, uint64_t count, int device,
                        uint64_t w_max_hint);

/* ------------------------------------------------------------------------------------------- */
/* Multi-GPU: estimators are independent, so GPU g of G owns the contiguous global ids
 * [floor(g r / G), floor((g+1) r / G)) and runs the whole per-batch update for them; all randomness is keyed
 * by the GLOBAL id, so the union of the shards is bit-identical to one unsharded run.  The only exchanges are
 * the batch (ncclBroadcast from rank 0, 8 w bytes, on a communication stream into one of two receive
 * buffers, so batch b+1's broadcast overlaps batch b's kernels) and, per estimate, an ncclAllReduce of the
 * exact u64 partial sums.  NCCL is loaded at run time (libnccl.so.2) on first use.                      */

/* tc_nccl_unique_id -- write a new ncclUniqueId (128 bytes, NCCL_UNIQUE_ID_BYTES) to id; rank 0 calls it and
 * passes the bytes to every rank out of band (e.g. a torch.distributed broadcast).  TC_ENCCL if NCCL is
 * unavailable. */
int tc_nccl_unique_id(void *id);

/* tc_create_rank -- one process per GPU ("torchrun mode"): this rank's shard of r estimators on CUDA device
 * `device` (-1 = current) and an NCCL communicator of `world` ranks (ncclCommInitRank with the 128-byte
 * nccl_unique_id from tc_nccl_unique_id on rank 0; a collective: every rank calls it).  On such a handle:
 *  - tc_push_batch / tc_push_batch_after are collective: every rank calls them with the same w, rank 0 passes
 *    the edges (host or its device), the other ranks pass edges = NULL (ignored otherwise); the library
 *    broadcasts the batch and every rank updates its shard.  A bad batch is rejected identically everywhere.
 *  - tc_closed_sum, tc_estimate, tc_closed_sum_async, tc_group_sums and tc_estimate_mom are collective and
 *    return the values over ALL r estimators on every rank.
 *  - tc_get_state / tc_set_state address the local shard (local ids 0 .. count-1); tc_rank_info tells which.
 *  - waits poll ncclCommGetAsyncError: an NCCL failure, or no progress for TC_NCCL_TIMEOUT_S seconds
 *    (environment, default 600), aborts the communicator and poisons the handle with TC_ENCCL.
 * NULL on failure (tc_last_error: TC_EINVAL, TC_ENOMEM, TC_ECUDA, TC_ENCCL). */
tc_ctx *tc_create_rank(uint64_t r, uint64_t seed, int rank, int world, const void *nccl_unique_id, int device,
                       uint64_t w_max_hint);

/* tc_config -- options of tc_create_ex (zero-initialise, then set what you need). */
typedef struct {
    int ngpus;            /* GPUs this process drives (<= 1: one GPU, a plain handle)                        */
    const int *devices;   /* ngpus CUDA device ids, or NULL for 0 .. ngpus-1 (the current device if ngpus <= 1) */
    int strict_errors;    /* 1: strict mode (each push synchronises); 0: asynchronous errors (tc_set_async)   */
    int graphs;           /* 1: each push as one CUDA graph per GPU (tc_set_graphs)                           */
    uint64_t w_max_hint;  /* preallocate the per-batch index for batches of up to this many edges             */
} tc_config;

/* tc_create_ex -- one process drives cfg->ngpus GPUs (ncclCommInitAll): one handle whose shards live on the
 * listed devices.  tc_push_batch takes the edges (host, or device memory of devices[0]) and broadcasts them;
 * tc_estimate / tc_closed_sum / tc_group_sums / tc_estimate_mom cover all r estimators; tc_get_state
 * addresses GLOBAL ids across the shards; tc_counters, tc_sync, tc_reset, tc_set_async, tc_set_graphs,
 * tc_tune apply to every shard; tc_set_state, tc_set_counters, tc_closed_sum_async, tc_profile* and tc_stats
 * are not available on a multi-GPU handle (TC_EINVAL).  NULL on failure (tc_last_error says why). */
tc_ctx *tc_create_ex(uint64_t r, uint64_t seed, const tc_config *cfg);

/* tc_rank_info -- rank and world of a rank handle (0 and 1 otherwise; world = ngpus for a tc_create_ex group)
 * and the global id of its first estimator and how many it owns. */
int tc_rank_info(tc_ctx *ctx, int *rank, int *world, uint64_t *first, uint64_t *count);

/* tc_push_batch -- bulkUpdateAll on the next w edges of the stream.
 *  edges: w tc_edge in arrival order.  Host memory (pageable or pinned) or device memory on the
 *         handle's device.  Host buffers are copied before the call returns (uploaded on a copy stream
 *         into one of two staging buffers, so the upload overlaps the previous batch's kernels when
 *         asynchronous errors are enabled); a device buffer must
 *         stay valid and unmodified until the next synchronising call (tc_sync, tc_estimate*,
 *         tc_get_state) when asynchronous errors are enabled, else until this call returns.
 *  w == 0: no-op (the batch index does not advance); w > 2^28 -> TC_EINVAL.
 *  Rejects the whole batch (state and counters unchanged) with, in this priority order:
 *  TC_EINVAL (an id 0xFFFFFFFF), TC_ESELFLOOP, TC_EDUP, TC_EOVERFLOW.  Edges that repeat an edge of
 *  an EARLIER batch are not detected (each edge arrives once).
 *  LIBRARY LIMIT: stream positions are stored in 32 bits on the device, so a batch that would take m past
 *  2^31 - 1 edges is rejected with TC_EOVERFLOW (reading R13).  This is a restriction of this
 *  library, not of the method (the oracle keeps u64 positions); below it chi <= m - 1 cannot overflow its
 *  31 bits either.  In asynchronous mode this limit is checked before enqueueing and returned at once.
 *  In the default strict mode the call synchronises and returns the batch's status; with
 *  tc_set_async(ctx, 1) it returns TC_OK after enqueueing, a failure is reported by the next
 *  synchronising call, and the handle is then poisoned (TC_ESTATE) -- its state and counters stay
 *  those of the last accepted batch (tc_get_state, tc_counters and tc_reset still work on it). */
int tc_push_batch(tc_ctx *ctx, const tc_edge *edges, uint64_t w);

/* tc_push_batch_after -- tc_push_batch for a DEVICE batch produced by work queued on producer_stream (a
 * cudaStream_t as void*; NULL = no ordering, i.e. tc_push_batch): the handle's stream first waits for
 * everything enqueued on producer_stream so far (an event; no host synchronisation), so the batch may still
 * be being written when the call is made.  Same arguments, semantics and errors as tc_push_batch. */
int tc_push_batch_after(tc_ctx *ctx, const tc_edge *edges, uint64_t w, void *producer_stream);

/* tc_estimate -- the mean of the coarse estimates X_i = chi_i * m if f3_i != empty else 0
 * (Lemma unbiased-est), over ALL r estimators, computed as
 * (double)m * (double)S / (double)r with S = sum of chi_i over this handle's closed estimators
 * (exact uint64).  For a shard (count < r) this is the shard's contribution; shards add up.
 * Synchronises.  0.0 before any edge. */
int tc_estimate(tc_ctx *ctx, double *out);

/* tc_reset -- back to the state right after creation (all estimators empty, m = 0, no batch), keeping
 * the allocations; clears a poisoned handle.  Synchronises. */
int tc_reset(tc_ctx *ctx);

/* tc_destroy -- frees the handle and its device memory; NULL-safe. */
void tc_destroy(tc_ctx *ctx);

/* ------------------------------------------------------------------------------------------- */
/* Extensions: shards, state readback, aggregation, streams, profiling.                         */

/* tc_closed_sum -- S for this handle (exact uint64; shards all-reduce it).  Synchronises. */
int tc_closed_sum(tc_ctx *ctx, uint64_t *S);

/* tc_estimate_mom -- median of means over `groups` contiguous groups of ALL r estimators, group g = global ids
 * [floor(g*r/G), floor((g+1)*r/G)), group mean (double)m * (double)S_g / (double)|g|, lower median;
 * PAPER.md:373-376, 887-888 (reading R9).  1 <= groups <= r.  TC_EINVAL on a lone shard
 * (tc_create_shard with count < r: it has only part of every group).  Synchronises. */
int tc_estimate_mom(tc_ctx *ctx, uint32_t groups, double *out);

/* tc_required_estimators -- the number of estimators that suffices for an (eps, delta)-approximation
 * (Theorem mdelta-suffices): r = ceil(96 / eps^2 * (m * Delta / tau) * ln(1 / delta)),
 * natural log (reading R10), evaluated in fp64.  m: stream edges, Delta: maximum degree, tau: a
 * lower bound on the triangle count.  Host-only (no device work).  TC_EINVAL unless 0 < eps, 0 < delta < 1,
 * tau > 0 and m * Delta < 2^64; TC_EOVERFLOW if r does not fit 64 bits. */
int tc_required_estimators(double eps, double delta, uint64_t m, uint64_t Delta, uint64_t tau, uint64_t *r);

/* tc_closed_sum_async -- enqueue, on the handle's stream after the last pushed batch, the copy of that
 * batch's S (exact uint64) to *S (host memory; pinned keeps the call asynchronous).  Returns without
 * waiting: *S is valid once the stream has passed that point (tc_sync, or any synchronising call), and
 * only if that call reports TC_OK (in asynchronous mode a rejected batch leaves garbage there).  The
 * estimate is then m * S / r with m after that batch (tc_estimate's expression).  Lets a pipeline read
 * every batch's result without a host synchronisation per batch. */
int tc_closed_sum_async(tc_ctx *ctx, uint64_t *S);

/* tc_group_sums -- S_g (exact uint64, host array of `groups`, 1 <= groups <= r) over contiguous groups of the
 * GLOBAL estimator ids g = [floor(g r / G), floor((g+1) r / G)): a shard handle reports the part of its own
 * estimators (groups it does not intersect are 0; shard vectors add up), a rank handle or a tc_create_ex
 * group the total. */
int tc_group_sums(tc_ctx *ctx, uint32_t groups, uint64_t *S_g);

/* tc_get_state -- copy local estimators [first, first+count) to HOST arrays (SoA):
 *  r1, r2: 2*count uint32 (lo, hi) with lo < hi, (0xFFFFFFFF, 0xFFFFFFFF) = empty;
 *  p1, p2: count uint64 0-based global stream positions (UINT64_MAX = empty);
 *  c: count uint32 chi;  closed: count uint8 (f3 != empty).  Any pointer may be NULL.
 * Synchronises. */
int tc_get_state(tc_ctx *ctx, uint64_t first, uint64_t count, uint32_t *r1, uint64_t *p1,
                 uint32_t *r2, uint64_t *p2, uint32_t *c, uint8_t *closed);

/* tc_set_state -- checkpoint restore: overwrite local estimators [first, first+count)
 * from HOST arrays in tc_get_state's layout (all pointers required when count > 0).  Validated first
 * (TC_EINVAL and nothing written unless every r1 / r2 is empty with position UINT64_MAX or has lo < hi and
 * a position < 2^31 - 1, c < 2^31 and closed in {0, 1}, and the NBSI invariants the estimator pass relies
 * on hold: an empty f1 has an empty f2, c = 0 and closed = 0; c == 0 iff f2 is empty;
 * closed implies f2 present; f2 shares exactly one endpoint with f1 and p1 < p2).  The closed sum S is recomputed.  Together with
 * tc_set_counters this resumes a stream exactly: the next push draws with the restored batch index.
 * Synchronises. */
int tc_set_state(tc_ctx *ctx, uint64_t first, uint64_t count, const uint32_t *r1, const uint64_t *p1,
                 const uint32_t *r2, const uint64_t *p2, const uint32_t *c, const uint8_t *closed);

/* tc_set_counters -- restore m (< 2^31) and the number of accepted non-empty batches (0 iff m = 0);
 * recomputes S.  Synchronises. */
int tc_set_counters(tc_ctx *ctx, uint64_t m, uint32_t batches);

/* tc_counters -- m (edges accepted so far) and the number of accepted non-empty batches.  In asynchronous
 * mode it synchronises first, so that a batch rejected after it was enqueued is not counted (on a handle
 * poisoned that way it returns the counters of the last accepted batch, matching tc_get_state). */
int tc_counters(tc_ctx *ctx, uint64_t *m, uint32_t *batches);

/* tc_set_async -- 0 = strict (default: each push synchronises and reports its status);
 * 1 = asynchronous (sticky error, reported at the next synchronising call). */
int tc_set_async(tc_ctx *ctx, int async_errors);

/* tc_set_graphs -- 1: each push runs as one CUDA graph: the launch sequence is captured once per batch shape
 * (w, and the small-batch / split passes) and relaunched for every later batch of that shape with only its
 * first node's arguments changed (the per-batch descriptor: input pointer, m, batch index, pair tag, S slot),
 * so a push costs one small host call plus the graph launch; up to 4 shapes are kept (least recently used
 * evicted; index growth and tc_tune drop them).  0 (default): plain stream launches.  Results are identical;
 * only launch overhead differs. */
int tc_set_graphs(tc_ctx *ctx, int enable);

/* tc_graph_captures -- how many graphs the handle has captured so far (a steady stream: one per shape). */
int tc_graph_captures(tc_ctx *ctx, uint64_t *captures);

/* tc_tune -- index-geometry knobs (tests / tuning).  Results never depend on them; only speed does.
 *  TC_TUNE_VBUCKET_ARCS  target arcs per vertex bucket (default 1024; the bucket count is a power of two
 *                        <= 4096 chosen from 2w / target)
 *  TC_TUNE_VBUCKET_CAP   vertex buckets with more arcs than this (1..2048, default 2048) leave the common
 *                        shared-memory hash path for the large-bucket kernel (hub peeling, then the hash
 *                        path for up to 4095 remaining arcs, else a radix sort on the vertex hash)
 *  TC_TUNE_VBUCKET_SORT_CAP  large-bucket kernel: buckets with more arcs than this (1..6144, default 6144)
 *                        are sorted in chunks through global memory instead of in shared memory
 *  TC_TUNE_SMALL_BATCH   the estimator pass for small batches: 0 = auto (default; batches
 *                        of at most 8192 edges), 1 = never, 2 = always.  It reads r1, r2, chi of every
 *                        estimator, tests f1's endpoints against a bit filter of the batch's vertices (no
 *                        false negatives) and runs Steps 1-3 only for estimators whose f1 is replaced or has
 *                        an endpoint in the batch, writing only the fields that change.
 *  TC_TUNE_SPLIT_KERNELS 1: the estimator pass runs as one kernel per step of SURVEY.md §8(a) -- k_u1_resample
 *                        (Step 1, a4), k_u2_count (Step 2a, a5), k_u3_select (Step 2b, a6), k_u4_close (Step 3,
 *                        a7), k_r_reduce (aggregation, a8) -- instead of the fused k_update, keeping every step's
 *                        values per estimator (tc_get_steps) for per-step parity and per-step timing; 0 (default):
 *                        fused.  The states are identical either way.
 *  TC_TUNE_SMALL_INDEX   batches of at most 4096 edges build the whole index in ONE kernel (one CTA per vertex
 *                        bucket of ~64 arcs, TC_TUNE_SMALL_INDEX_ARCS: validation, pair table, grouping) instead of the eight launches of
 *                        the partitioned build: 0 = auto (default), 1 = never, 2 = always (same).
 *  TC_TUNE_SMALL_INDEX_ARCS  target arcs per k_small_index CTA (16..8192, default 64; at most 256 CTAs).  Same
 *                        results (the segment order in segS may differ; every probe goes through the tables).
 *  TC_TUNE_EVENT_CHECKED event mode: 1 = every batch through the four-kernel path that checks the vertex degree
 *                        limit before applying anything (k_ed_pre, k_ed_trigger, k_ed_process, k_ed_post); 0
 *                        (default) = that path only when a degree could reach the limit (m + w > 2^30 - 1),
 *                        else the two-kernel path (k_ed_front, k_ed_process).  Same results.
 *  TC_TUNE_PAIR_FILTER   bulk mode, fused estimator pass: a Bloom filter over the batch's pairs (16 bits per edge,
 *                        filled by the pair-table kernel) that Step 3's closing-edge probe
 *                        reads before the edge-pair table; it has no false negatives.  0 = auto (default;
 *                        batches of at least 2^21 edges, where the table no longer stays in L2), 1 = never,
 *                        2 = always (partitioned index).  Same results.
 * Returns TC_EINVAL for an unknown knob or a value out of range.  Synchronises. */
enum { TC_TUNE_VBUCKET_ARCS = 0, TC_TUNE_VBUCKET_CAP = 2, TC_TUNE_VBUCKET_SORT_CAP = 4, TC_TUNE_SMALL_BATCH = 6,
       TC_TUNE_SPLIT_KERNELS = 8, TC_TUNE_SMALL_INDEX = 10, TC_TUNE_EVENT_CHECKED = 12, TC_TUNE_PAIR_FILTER = 14,
       TC_TUNE_SMALL_INDEX_ARCS = 16 };
int tc_tune(tc_ctx *ctx, int knob, uint64_t value);

/* tc_set_mode -- the estimator update rule (reading R17, §10 row 4).
 *  TC_MODE_BULK  (default) the paper's bulkUpdateAll (§4): every estimator takes one Step-1
 *                draw per batch, O(r + w) work per batch.
 *  TC_MODE_EVENT the sequential neighborhood-sampling rule (batch size 1 of bulkUpdateAll is
 *                reservoir sampling) with skip-sampled reservoirs: each estimator draws, when
 *                f1 (f2) is taken, the stream time J (the adjacency count K) of its next replacement, with
 *                P(J > s) = t1/s (P(K > k) = chi/k) -- exactly the per-edge coins' law, so NBSI holds after every
 *                batch and E[X] = tau as in the bulk mode, but the random draws differ (the two modes' states are
 *                different samples of the same law).  A batch processes only the estimators it changes (watch
 *                lists keyed by J, by (vertex, degree threshold) and by the closing pair; O(w + events) per
 *                batch after the first few), and the state after a stream prefix does not depend on the batching.
 *                chi is kept as deg(u) + deg(v) - B with persistent vertex degrees; a batch that would give a
 *                vertex degree > 2^30 - 1 is rejected with TC_EOVERFLOW (reading R17c).  tc_set_state and
 *                tc_set_counters return TC_EINVAL in this mode.
 * Only on a handle that has seen no batch (fresh or after tc_reset), else TC_EINVAL.  The event mode allocates
 * about 2.1 KB per estimator of watch tables (16 64-byte watch chunks, two maps of 16-byte slots at load <= 1/2)
 * plus 32 bytes per distinct vertex seen (table load <= 1/2).  Synchronises. */
enum { TC_MODE_BULK = 0, TC_MODE_EVENT = 1 };
int tc_set_mode(tc_ctx *ctx, int mode);

/* tc_get_event_state -- event mode: for local estimators [first, first+count), HOST arrays (any may be NULL):
 * J = the 1-based stream time of the next f1 replacement, K = the adjacency count at which f2 is next replaced
 * (0xFFFFFFFF: beyond 2^31 - 1, i.e. never; K = 0xFFFFFFFF also for an estimator without f1), ev = random words
 * used.  The NBSI fields come from tc_get_state.  TC_EINVAL in the bulk mode.  Synchronises. */
int tc_get_event_state(tc_ctx *ctx, uint64_t first, uint64_t count, uint32_t *J, uint32_t *K, uint32_t *ev);

/* tc_event_counters -- event mode, totals since the mode was set / the last reset: out[0] estimators processed,
 * out[1] f1 and f2 replacements, out[2] full sweeps, out[3] distinct vertices seen.  Returns 4 (TC_EINVAL in the
 * bulk mode).  Synchronises. */
int tc_event_counters(tc_ctx *ctx, uint64_t *out, int n);

/* tc_get_steps -- with TC_TUNE_SPLIT_KERNELS on: the per-step values of the last batch for local estimators
 * [first, first+count), HOST arrays (any may be NULL): j = Step 1's replacement index in W (0xFFFFFFFF: f1
 * retained), chim = chi^- after Step 1, ld / rd = rank(u->v) / rank(v->u) (chi^+ = ld + rd; u = min endpoint,
 * reading R1), d2 = Step 2's draw over chi^- + chi^+ (UINT64_MAX: no draw), k2 = batch position of the new f2
 * (0xFFFFFFFF: kept).  TC_EINVAL if the split pass was never enabled.  Synchronises. */
int tc_get_steps(tc_ctx *ctx, uint64_t first, uint64_t count, uint32_t *j, uint32_t *chim, uint32_t *ld, uint32_t *rd,
                 uint64_t *d2, uint32_t *k2);

/* tc_sync -- wait for all queued work; returns the first asynchronous error, if any. */
int tc_sync(tc_ctx *ctx);

/* tc_stream -- the handle's cudaStream_t (as void*), for events recorded by the caller. */
void *tc_stream(tc_ctx *ctx);

/* Profiling: when enabled, CUDA events bracket each kernel phase of every push (the pair phase on the
 * handle's second stream, where it overlaps the vertex phase).  tc_profile_read fills, for phase p < n
 * (TC_PHASE_*): total milliseconds and launch count since the last reset, and returns the number of
 * phases.  Synchronises. */
enum {
    TC_PHASE_PARTITION = 0, /* a1: validation, bucket histograms, scans, stable scatter of arcs / edges  */
    TC_PHASE_PAIRS = 1,     /* a3: edge-pair table (duplicates -> TC_EDUP), on the second stream         */
    TC_PHASE_VERTICES = 2,  /* a2: per-bucket grouping of arcs by vertex, ranks / segment ends, vertex table */
    TC_PHASE_UPDATE = 3,    /* a4-a8: the fused estimator update (Steps 1-3 + partial sums)              */
    TC_NPHASES = 4
};
int tc_profile(tc_ctx *ctx, int enable);
int tc_profile_read(tc_ctx *ctx, double *ms, uint64_t *launches, int n);

/* tc_profile_kernels -- the same per KERNEL (CUDA events around each launch; profiled pushes run as plain
 * stream launches, never as a graph): total milliseconds and launch count of kernel k < n since the last
 * tc_profile() call; returns the number of kernel ids.  Synchronises.  tc_kernel_name(k): its name (static
 * string, "" for an unknown id). */
int tc_profile_kernels(tc_ctx *ctx, double *ms, uint64_t *launches, int n);
const char *tc_kernel_name(int k);

/* tc_stats -- event counts since the last tc_profile() call (for the bench's byte model):
 * out[0] estimators whose f1 was replaced, out[1] retained-f1 estimators whose f2 was replaced,
 * out[2] sum over batches of the number of distinct vertices in W, out[3] batches, out[4] estimators the
 * small-batch pass skipped as untouched (TC_TUNE_SMALL_BATCH), out[5] arcs and out[6] distinct vertices
 * grouped by the large-bucket kernels (k_vhub / k_vbig).  Returns 7. */
int tc_stats(tc_ctx *ctx, uint64_t *out, int n);

/* Number of kernel launches issued by the last successful push (for the bench's gpu_launches). */
int tc_last_launches(tc_ctx *ctx, uint32_t *launches);

/* ------------------------------------------------------------------------------------------- */
/* Ground truth for the accuracy study (MD% methodology PAPER.md:993-1003).   */

/* tc_exact_triangles -- tau = |T(G)|, the exact number of triangles of the simple undirected graph
 * whose m edges are `edges` (§2: T(G) the triangles, tau = |T(G)|), computed on the
 * current CUDA device by degree-ordered wedge closing (exact.cu).  edges: host or device memory, any
 * orientation, m < 2^31; read only, owned by the caller.  Independent of every estimator handle (it
 * allocates and frees its own device scratch, about 80 bytes per edge, on its own stream).
 * *tau receives the count; device_ms (may be NULL) the device time of the computation from the first
 * kernel to the last (CUDA events; the host->device copy of host edges is excluded).
 * Errors: TC_EINVAL (tau NULL, edges NULL with m > 0, m >= 2^31, or a vertex id 0xFFFFFFFF),
 * TC_ESELFLOOP (u == v), TC_EDUP (the same undirected pair twice), TC_ENOMEM, TC_ECUDA.  On error *tau
 * is 0.  Synchronises. */
int tc_exact_triangles(const tc_edge *edges, uint64_t m, uint64_t *tau, double *device_ms);

/* ------------------------------------------------------------------------------------------- */
/* Ingestion in front of the path: SNAP-format text edge lists, the format of
 * the paper's datasets ("a list of edges in plain text", Table 1; streamed "as they are read from
 * disk"; I/O timed apart from processing).                  */

/* Line format: blank lines and lines whose first non-blank character is '#' or '%' are skipped; an
 * edge line is  <u> <whitespace> <v>  with u, v decimal ids <= 0xFFFFFFFE (spaces / tabs, '\r' allowed),
 * optionally followed by whitespace and further columns, which are ignored.  u == v is TC_ESELFLOOP
 * unless TC_INGEST_SKIP_LOOPS is set (then the line is skipped).  Duplicate pairs are NOT removed: the
 * file must list a simple graph, each edge once (a repeat inside one batch fails the push with TC_EDUP). */
enum { TC_INGEST_SKIP_LOOPS = 1 };

/* tc_parse_edges -- parse text[0, len) (host memory) into out[0, cap) (host).  Complete lines only,
 * unless final != 0 (then a last line without '\n' counts too); stops early when out is full (the
 * line that did not fit is not consumed).  *n_edges = edges written, *consumed = bytes consumed (a
 * prefix of whole lines), *lines = lines consumed.  On TC_EPARSE / TC_ESELFLOOP, *consumed stops before
 * the bad line and *lines counts it (so the caller's running count + *lines is its 1-based number).
 * Host-only (no device work). */
int tc_parse_edges(const char *text, uint64_t len, int final, int flags, tc_edge *out, uint64_t cap,
                   uint64_t *n_edges, uint64_t *consumed, uint64_t *lines);

typedef struct {
    uint64_t edges;       /* edges pushed (accepted)                                             */
    uint64_t batches;     /* tc_push_batch calls that succeeded                                  */
    uint64_t lines;       /* lines read                                                          */
    uint64_t error_line;  /* 1-based line of a parse error / self-loop, else 0                    */
    double io_s;          /* reader thread busy time: file reads + parsing (the paper's "I/O")   */
    double push_s;        /* time inside tc_push_batch (staging copy + update; strict mode: sync) */
    double wait_s;        /* time the pushing thread waited for a parsed batch (I/O-bound part)  */
    double wall_s;        /* whole call                                                          */
} tc_ingest_stats;

/* tc_ingest_file -- stream the SNAP-format edge list at `path` through tc_push_batch in batches of w
 * edges (the last one may be short), in file order.  A reader thread reads and parses into one of two
 * pinned host batch buffers while the calling thread pushes the other, so file I/O and parsing overlap
 * the GPU update.  Returns the first error: TC_EIO, TC_EPARSE / TC_ESELFLOOP (stats->error_line says
 * where; batches before it may already have been pushed -- stats->edges of them), or any tc_push_batch
 * code.  Synchronises at the end (tc_sync).  stats may be NULL. */
int tc_ingest_file(tc_ctx *ctx, const char *path, uint64_t w, int flags, tc_ingest_stats *stats);

/* ------------------------------------------------------------------------------------------- */
/* Test hooks (not on the path): the estimator pass's own device functions on chosen inputs, on the
 * current CUDA device, host arrays in and out, synchronous.                                     */

/* tc_test_draws -- out[i] = the device bounded uniform (Lemire multiply-shift with rejection, DESIGN.md
 * reading R8) of n[i] (> 0) from the first 64-bit word x[i], retries drawn from Philox4x32-10 with key
 * seed and counter (id[i].lo32, id[i].hi32, b[i], base[i] + t) (reading R7), exactly as the estimator pass
 * calls it.  TC_EINVAL on a NULL array or an n[i] = 0. */
int tc_test_draws(const uint64_t *n, const uint64_t *x, const uint64_t *id, const uint32_t *b,
                  const uint32_t *base, uint64_t seed, uint64_t count, uint64_t *out);

/* tc_test_philox -- out[4i..4i+3] = the device Philox4x32-10 block of counter ctr[4i..4i+3] and key
 * key[2i..2i+1]. */
int tc_test_philox(const uint32_t *ctr, const uint32_t *key, uint64_t count, uint32_t *out);

/* tc_strerror -- a static, never-NULL description of a TC_* code (owned by the library). */
const char *tc_strerror(int code);
int tc_last_error(void); /* thread-local code of the last failed tc_create* */

#ifdef __cplusplus
}
#endif
#endif /* TC_B200_H */

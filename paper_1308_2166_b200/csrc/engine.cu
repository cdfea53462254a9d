// engine.cu -- host side of the C ABI declared in include/tc.h: handle, device memory, the per-batch
// launch sequence, error handling and readback.  No PyTorch types; plain pointers and sizes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>
#include <array>
#include <vector>

#include <chrono>
#include <thread>

#include "../../include/tc.h"
#include "event.h"
#include "kernels.h"
#include "nccl_api.h"

using namespace tcb;

namespace {
thread_local int g_last_error = TC_OK;

uint64_t next_pow2(uint64_t x) {
    uint64_t p = 1;
    while (p < x) p <<= 1;
    return p;
}
}  // namespace

struct tc_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;   // second stream: the edge-pair table, concurrently with the vertex buckets
    cudaStream_t side2 = nullptr;  // third stream: the large vertex buckets
    cudaStream_t copy = nullptr;   // host-batch uploads, so batch b+1's H2D overlaps batch b's kernels
    cudaEvent_t copied[2] = {nullptr, nullptr}, stage_free[2] = {nullptr, nullptr};
    int stage_next = 0;            // staging buffer of the next host batch
    cudaEvent_t fork = nullptr, join = nullptr, fork2 = nullptr, join2 = nullptr;
    uint64_t r = 0, seed = 0, first = 0, count = 0;
    uint64_t m = 0;
    uint32_t b = 0;
    uint32_t ptag = 0;  // edge-pair table tag of the last push
    uint32_t pf_zeroed[2] = {0, 0};  // pair filters: leading words known to be zero (k_count zeroes the other one)
    int async_errors = 0;
    int poisoned = 0;  // 0 or the TC_E* code that poisoned the handle
    int S_slot = -1;   // accumulator slot holding S of the last accepted batch (-1: none yet)
    // asynchronous mode: m before each batch enqueued since the last clean settle (batch indices
    // async_b0, async_b0 + 1, ...), so that a rejected batch found later can be rolled back to
    std::vector<uint64_t> async_mprev;
    uint32_t async_b0 = 0;
    uint32_t last_launches = 0;
    StateBufs st;
    IndexBufs ix;
    uint32_t *h_err = nullptr;  // pinned
    cudaEvent_t copy_done = nullptr;
    cudaEvent_t produced = nullptr;  // tc_push_batch_after: the producer stream's work so far
    // profiling
    int prof = 0;
    // begin / end events of each phase, then of each kernel (KernelId), one set per profiled push (read and
    // recycled at the next sync); ev_kused: which kernels the push launched
    std::vector<std::array<cudaEvent_t, 2 * TC_NPHASES + 2 * K_NKERNELS>> ev_pool;
    std::vector<uint32_t> ev_kused;
    size_t ev_used = 0;
    double prof_ms[TC_NPHASES] = {};
    uint64_t prof_launch[TC_NPHASES] = {};
    double prof_kms[K_NKERNELS] = {};
    uint64_t prof_klaunch[K_NKERNELS] = {};
    // CUDA graphs of the per-batch launch sequence, one per batch shape (w, small-batch pass, split pass):
    // captured once, then relaunched with only the descriptor node's arguments changed (BatchDesc)
    int use_graph = 0;  // opt-in (tc_set_graphs)
    struct GraphEntry {
        uint64_t key = 0, last_use = 0;
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        cudaGraphNode_t desc_node = nullptr;
        uint32_t launches = 0;
    };
    std::vector<GraphEntry> graphs;
    uint64_t graph_clock = 0;
    uint64_t graph_captures = 0;  // how many captures (tests: a steady stream captures once per shape)
    Tuning tune;
    // multi-GPU: a rank handle (tc_create_rank, or a peer of a tc_create_ex group) owns the
    // global estimator ids [first, first + count) of r and an NCCL communicator; every batch is broadcast from
    // rank 0 into one of two receive buffers on the comm stream (batch b+1's broadcast overlaps batch b's
    // kernels) and the exact partial sums are all-reduced when an estimate is asked for
    ncclComm_t nccl = nullptr;
    int rank = 0, world = 1;
    int nccl_dead = 0;             // the communicator was aborted after an error
    cudaStream_t comm = nullptr;
    uint2 *bcast[2] = {nullptr, nullptr};
    cudaEvent_t bc_done = nullptr, bc_free[2] = {nullptr, nullptr}, inready = nullptr;
    int bc_next = 0;
    unsigned long long *d_red = nullptr;  // device scratch of the all-reduces (grown on demand)
    uint64_t d_red_words = 0;
    double nccl_timeout_s = 600.0;
    StepBufs steps;  // split estimator pass (TC_TUNE_SPLIT_KERNELS): per-step values of the last batch
    // a tc_create_ex handle over several GPUs of this process: the peers (rank handles) do all the work
    std::vector<tc_ctx *> peers;
    // event-driven mode (tc_set_mode TC_MODE_EVENT): its device tables, and an upper bound
    // on the persistent vertex count (exact at m = ed_m_known, + 2 per edge pushed since) that decides when the
    // vertex table must grow
    int mode = TC_MODE_BULK;
    EdDev ed;
    uint64_t ed_pv_known = 0, ed_m_known = 0;
};

// what a call on a poisoned handle returns: the CUDA / NCCL failure itself, else TC_ESTATE (a rejected batch)
static int poisoned_code(const tc_ctx *c) {
    if (!c->poisoned) return TC_OK;
    return (c->poisoned == TC_ECUDA || c->poisoned == TC_ENCCL) ? c->poisoned : TC_ESTATE;
}

static int fail_cuda(tc_ctx *c) {
    cudaGetLastError();
    if (c) c->poisoned = TC_ECUDA;
    return TC_ECUDA;
}

#define CK2(c, call)                                   \
    do {                                               \
        if ((call) != cudaSuccess) return fail_cuda(c); \
    } while (0)

#define CK(call)                                   \
    do {                                           \
        if ((call) != cudaSuccess) return fail_cuda(ctx); \
    } while (0)

static void free_steps(StepBufs &sb) {
    void *bufs[] = {sb.j, sb.xhi, sb.chim, sb.ld, sb.rd, sb.endU, sb.endV, sb.d2, sb.k2};
    for (void *p : bufs) cudaFree(p);
    sb = StepBufs();
}

static bool alloc_steps(StepBufs &sb, uint64_t count) {
    const uint64_t n = std::max<uint64_t>(count, 1);
    sb.count = count;
    const bool ok = cudaMalloc(&sb.j, 4 * n) == cudaSuccess && cudaMalloc(&sb.xhi, 8 * n) == cudaSuccess &&
                    cudaMalloc(&sb.chim, 4 * n) == cudaSuccess && cudaMalloc(&sb.ld, 4 * n) == cudaSuccess &&
                    cudaMalloc(&sb.rd, 4 * n) == cudaSuccess && cudaMalloc(&sb.endU, 4 * n) == cudaSuccess &&
                    cudaMalloc(&sb.endV, 4 * n) == cudaSuccess && cudaMalloc(&sb.d2, 8 * n) == cudaSuccess &&
                    cudaMalloc(&sb.k2, 4 * n) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        free_steps(sb);
    }
    return ok;
}

static void free_index(IndexBufs &ix) {
    void *bufs[] = {ix.arcs2, ix.vstart2, ix.E, ix.apos, ix.pslot, ix.segS, ix.pt, ix.vt, ix.vslice, ix.arcs, ix.scratch, ix.vperm, ix.vdefer,
                    ix.cntV, ix.offV, ix.arank, ix.vstart, ix.ctr, ix.stage, ix.stage2, ix.filt, ix.pf, ix.desc};
    for (void *p : bufs) cudaFree(p);
    ix = IndexBufs();
}

constexpr uint64_t kMaxBuckets = 1ull << kMaxBucketBits;
constexpr uint64_t kMaxBatch = 1ull << 28;  // 32-bit table offsets (vertex slices < 8 w slots)
constexpr uint64_t kStartWords = kMaxBuckets + 8;  // vstart: bucket sizes -> prefixes (+ grand total)

// (Re)allocate the per-batch index for batches of up to w edges.
static void drop_graphs(tc_ctx *ctx) {
    for (auto &g : ctx->graphs) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        if (g.graph) cudaGraphDestroy(g.graph);
    }
    ctx->graphs.clear();
}

extern "C" {
static int settle(tc_ctx *ctx);
}

static int grow_index(tc_ctx *ctx, uint64_t w) {
    if (w <= ctx->ix.wcap) return TC_OK;
    // the counters hold the only copy of the sticky asynchronous error word: surface it first
    const int rc = settle(ctx);
    if (rc != TC_OK) return rc;
    CK(cudaStreamSynchronize(ctx->copy));
    drop_graphs(ctx);  // the captured graphs hold the old buffers' addresses
    free_index(ctx->ix);
    IndexBufs &ix = ctx->ix;
    const uint64_t cap = std::max<uint64_t>(next_pow2(w), 1024);
    ix.tiles_cap = (cap + kTileEdges - 1) / kTileEdges;
    bool ok = cudaMalloc(&ix.E, 8 * cap) == cudaSuccess && cudaMalloc(&ix.apos, 8 * cap) == cudaSuccess &&
              cudaMalloc(&ix.pslot, 16 * cap) == cudaSuccess &&
              cudaMalloc(&ix.segS, 16 * cap) == cudaSuccess &&
              cudaMalloc(&ix.pt, 32ull * pair_groups_alloc((uint32_t)cap)) == cudaSuccess &&
              cudaMalloc(&ix.vt, 16 * 4 * cap) == cudaSuccess &&  // slices at 2 * (bucket start), <= 2 n_b slots
              cudaMalloc(&ix.vslice, 8 * kMaxBuckets) == cudaSuccess;
    ok = ok && cudaMalloc(&ix.arcs, 32 * cap) == cudaSuccess && cudaMalloc(&ix.vstart2, 4 * kStartWords) == cudaSuccess &&
         cudaMalloc(&ix.arcs2, 32 * cap) == cudaSuccess && cudaMalloc(&ix.scratch, 32 * cap) == cudaSuccess &&
         cudaMalloc(&ix.vperm, 4 * kMaxBuckets) == cudaSuccess && cudaMalloc(&ix.vdefer, 4 * kMaxBuckets) == cudaSuccess &&
         cudaMalloc(&ix.cntV, 4ull * (1u << kMaxPartBits) * ix.tiles_cap) == cudaSuccess &&
         cudaMalloc(&ix.offV, 4ull * (1u << kMaxPartBits) * ix.tiles_cap) == cudaSuccess &&
         cudaMalloc(&ix.arank, 4 * cap) == cudaSuccess && cudaMalloc(&ix.vstart, 4 * kStartWords) == cudaSuccess &&
         cudaMalloc(&ix.ctr, 4 * kCtrWords) == cudaSuccess && cudaMalloc(&ix.stage, 8 * cap) == cudaSuccess &&
         cudaMalloc(&ix.stage2, 8 * cap) == cudaSuccess && cudaMalloc(&ix.filt, 4ull * kFilterWords) == cudaSuccess &&
         cudaMalloc(&ix.pf, 8ull * pf_words((uint32_t)cap)) == cudaSuccess &&  // two filters
         cudaMalloc(&ix.desc, sizeof(BatchDesc)) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        free_index(ix);
        return TC_ENOMEM;
    }
    if (ctx->nccl) {  // receive buffers of the per-batch broadcast
        for (int i = 0; i < 2; ++i) {
            cudaFree(ctx->bcast[i]);
            ctx->bcast[i] = nullptr;
            if (cudaMalloc(&ctx->bcast[i], 8 * cap) != cudaSuccess) {
                cudaGetLastError();
                free_index(ix);
                return TC_ENOMEM;
            }
        }
    }
    if (ctx->mode == TC_MODE_EVENT && !ed_alloc_seg(ctx->ed, cap)) {
        free_index(ix);
        return TC_ENOMEM;
    }
    ix.wcap = cap;
    CK(cudaMemsetAsync(ix.ctr, 0, 4 * kCtrWords, ctx->stream));
    CK(cudaMemsetAsync(ix.ctr + kCtrFailB, 0xFF, 4, ctx->stream));
    CK(cudaMemsetAsync(ix.pt, 0, 32ull * pair_groups_alloc((uint32_t)cap), ctx->stream));  // tag 0: free
    CK(cudaMemsetAsync(ix.pf, 0, 8ull * pf_words((uint32_t)cap), ctx->stream));
    ctx->pf_zeroed[0] = ctx->pf_zeroed[1] = pf_words((uint32_t)cap);
    ctx->ptag = 0;
    return TC_OK;
}

static void destroy_ctx(tc_ctx *ctx) {
    if (!ctx) return;
    for (tc_ctx *p : ctx->peers) destroy_ctx(p);
    if (!ctx->peers.empty()) {
        delete ctx;
        return;
    }
    cudaSetDevice(ctx->device);
    if (ctx->comm) cudaStreamSynchronize(ctx->comm);
    if (ctx->nccl) {
        if (ctx->nccl_dead) nccl().CommAbort(ctx->nccl);
        else nccl().CommDestroy(ctx->nccl);
    }
    for (int i = 0; i < 2; ++i) {
        cudaFree(ctx->bcast[i]);
        if (ctx->bc_free[i]) cudaEventDestroy(ctx->bc_free[i]);
    }
    if (ctx->bc_done) cudaEventDestroy(ctx->bc_done);
    if (ctx->inready) cudaEventDestroy(ctx->inready);
    if (ctx->comm) cudaStreamDestroy(ctx->comm);
    cudaFree(ctx->d_red);
    free_steps(ctx->steps);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    ed_free(ctx->ed);
    free_index(ctx->ix);
    cudaFree(ctx->st.r1);
    cudaFree(ctx->st.r2);
    cudaFree(ctx->st.cf);
    cudaFree(ctx->st.p1);
    cudaFree(ctx->st.p2);
    cudaFree(ctx->st.S);
    cudaFree(ctx->st.stats);
    if (ctx->h_err) cudaFreeHost(ctx->h_err);
    if (ctx->copy_done) cudaEventDestroy(ctx->copy_done);
    if (ctx->produced) cudaEventDestroy(ctx->produced);
    for (auto &set : ctx->ev_pool)
        for (auto &e : set)
            if (e) cudaEventDestroy(e);
    drop_graphs(ctx);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    if (ctx->side2) cudaStreamDestroy(ctx->side2);
    if (ctx->copy) cudaStreamDestroy(ctx->copy);
    for (int i = 0; i < 2; ++i) {
        if (ctx->copied[i]) cudaEventDestroy(ctx->copied[i]);
        if (ctx->stage_free[i]) cudaEventDestroy(ctx->stage_free[i]);
    }
    if (ctx->join2) cudaEventDestroy(ctx->join2);
    if (ctx->fork2) cudaEventDestroy(ctx->fork2);
    if (ctx->fork) cudaEventDestroy(ctx->fork);
    if (ctx->join) cudaEventDestroy(ctx->join);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

extern "C" {

tc_ctx *tc_create_shard(uint64_t r, uint64_t seed, uint64_t first, uint64_t count, int device, uint64_t w_max_hint) {
    g_last_error = TC_OK;
    if (r == 0 || first > r || count > r - first || w_max_hint > kMaxBatch) {
        g_last_error = TC_EINVAL;
        return nullptr;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        g_last_error = TC_ECUDA;
        return nullptr;
    }
    if (device < 0) cudaGetDevice(&device);
    if (device >= ndev || cudaSetDevice(device) != cudaSuccess) {
        cudaGetLastError();
        g_last_error = TC_EINVAL;
        return nullptr;
    }
    tc_ctx *ctx = new (std::nothrow) tc_ctx();
    if (!ctx) {
        g_last_error = TC_ENOMEM;
        return nullptr;
    }
    static uint64_t attrs = 0;  // devices whose kernel attributes (dynamic shared memory) are set
    if (!(attrs >> (device & 63) & 1)) {
        if (set_kernel_attributes() != 0) {
            cudaGetLastError();
            delete ctx;
            g_last_error = TC_ECUDA;
            return nullptr;
        }
        attrs |= 1ull << (device & 63);
    }
    ctx->device = device;
    ctx->r = r;
    ctx->seed = seed;
    ctx->first = first;
    ctx->count = count;
    ctx->st.count = count;
    const uint64_t n = std::max<uint64_t>(count, 1);
    bool ok = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&ctx->side2, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&ctx->copied[0], cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&ctx->copied[1], cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&ctx->stage_free[0], cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&ctx->stage_free[1], cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&ctx->join2, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&ctx->fork2, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&ctx->fork, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&ctx->join, cudaEventDisableTiming) == cudaSuccess &&
              cudaMalloc(&ctx->st.r1, 8 * n) == cudaSuccess && cudaMalloc(&ctx->st.r2, 8 * n) == cudaSuccess &&
              cudaMalloc(&ctx->st.cf, 4 * n) == cudaSuccess && cudaMalloc(&ctx->st.p1, 4 * n) == cudaSuccess &&
              cudaMalloc(&ctx->st.p2, 4 * n) == cudaSuccess && cudaMalloc(&ctx->st.S, 16) == cudaSuccess &&
              cudaMalloc(&ctx->st.stats, 8 * kNStats) == cudaSuccess &&
              cudaMallocHost(&ctx->h_err, 128) == cudaSuccess &&
              cudaEventCreateWithFlags(&ctx->copy_done, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&ctx->produced, cudaEventDisableTiming) == cudaSuccess;
    if (ok) {
        ok = cudaMemsetAsync(ctx->st.S, 0, 16, ctx->stream) == cudaSuccess &&
             cudaMemsetAsync(ctx->st.stats, 0, 8 * kNStats, ctx->stream) == cudaSuccess;
        launch_init_state(ctx->st, ctx->stream);
        ok = ok && cudaGetLastError() == cudaSuccess;
    }
    if (ok && w_max_hint) ok = grow_index(ctx, w_max_hint) == TC_OK;
    if (ok) ok = cudaStreamSynchronize(ctx->stream) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        destroy_ctx(ctx);
        g_last_error = TC_ENOMEM;
        return nullptr;
    }
    return ctx;
}

tc_ctx *tc_create(uint64_t r, uint64_t seed) { return tc_create_shard(r, seed, 0, r, -1, 0); }


void tc_destroy(tc_ctx *ctx) { destroy_ctx(ctx); }

static int decode_err(uint32_t e) {
    if (e & kErrInternal) return TC_EINTERNAL;
    if (e & kErrInval) return TC_EINVAL;
    if (e & kErrLoop) return TC_ESELFLOOP;
    if (e & kErrDup) return TC_EDUP;
    if (e & kErrOvf) return TC_EOVERFLOW;
    return TC_OK;
}

static int recompute_S(tc_ctx *ctx);

// Wait for queued work and surface a pending asynchronous batch error (poisons the handle).
// Wait for stream s.  On a rank handle the wait polls the communicator too: an asynchronous NCCL error (or
// no progress for nccl_timeout_s) aborts the communicator and poisons the handle with TC_ENCCL, instead of
// blocking forever behind a collective whose peer is gone.
static int wait_stream(tc_ctx *ctx, cudaStream_t s) {
    if (!s) return TC_OK;
    if (!ctx->nccl || ctx->nccl_dead) return cudaStreamSynchronize(s) == cudaSuccess ? TC_OK : fail_cuda(ctx);
    const auto t0 = std::chrono::steady_clock::now();
    for (int spin = 0;; ++spin) {
        const cudaError_t q = cudaStreamQuery(s);
        if (q == cudaSuccess) return TC_OK;
        if (q != cudaErrorNotReady) return fail_cuda(ctx);
        ncclResult_t ae = ncclSuccess;
        const bool timed_out =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > ctx->nccl_timeout_s;
        if (nccl().CommGetAsyncError(ctx->nccl, &ae) != ncclSuccess || (ae != ncclSuccess && ae != ncclInProgress) ||
            timed_out) {
            nccl().CommAbort(ctx->nccl);
            ctx->nccl_dead = 1;
            ctx->poisoned = TC_ENCCL;
            return TC_ENCCL;
        }
        if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

#define WAIT(s)                                  \
    do {                                         \
        const int wrc_ = wait_stream(ctx, (s));  \
        if (wrc_ != TC_OK) return wrc_;          \
    } while (0)

static int settle(tc_ctx *ctx) {
    CK(cudaSetDevice(ctx->device));
    WAIT(ctx->comm);
    WAIT(ctx->stream);
    WAIT(ctx->side);
    WAIT(ctx->side2);
    if (ctx->async_errors && !ctx->poisoned && ctx->ix.ctr) {
        CK(cudaMemcpy(ctx->h_err, ctx->ix.ctr, 4 * kCtrWords, cudaMemcpyDeviceToHost));
        const int code = decode_err(ctx->h_err[kCtrErr]);
        if (code != TC_OK) {
            // the first batch whose estimator pass found the sticky error word set is the rejected one:
            // m and the batch count go back to what they were before it (all later batches were skipped)
            const uint32_t fb = ctx->h_err[kCtrFailB];
            if (fb >= ctx->async_b0 && fb - ctx->async_b0 < ctx->async_mprev.size()) {
                ctx->m = ctx->async_mprev[fb - ctx->async_b0];
                ctx->b = fb;
            }
            ctx->async_mprev.clear();
            ctx->async_b0 = ctx->b;
            ctx->poisoned = code;
            const int rs = recompute_S(ctx);  // later skipped batches reset the S slots
            return rs != TC_OK ? rs : code;
        }
        ctx->async_mprev.clear();
        ctx->async_b0 = ctx->b;
    }
    for (size_t i = 0; i < ctx->ev_used; ++i) {  // completed profiled pushes
        for (int p = 0; p < TC_NPHASES; ++p) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, ctx->ev_pool[i][2 * p], ctx->ev_pool[i][2 * p + 1]) == cudaSuccess)
                ctx->prof_ms[p] += ms;
        }
        for (int k = 0; k < K_NKERNELS; ++k) {
            if (!(ctx->ev_kused[i] >> k & 1u)) continue;
            float ms = 0.f;
            const cudaEvent_t *e = &ctx->ev_pool[i][2 * TC_NPHASES + 2 * k];
            if (cudaEventElapsedTime(&ms, e[0], e[1]) == cudaSuccess) {
                ctx->prof_kms[k] += ms;
                ctx->prof_klaunch[k] += 1;
            }
        }
    }
    cudaGetLastError();
    ctx->ev_used = 0;
    return poisoned_code(ctx);
}

// One push = prepare (checks, index capacity, the batch onto the device: staging upload and, on a rank handle,
// the broadcast from rank 0) + launch (the kernels, the strict-mode status, the counters).  A tc_create_ex
// group prepares all its peers inside one NCCL group, then launches them.
struct PushPrep {
    const uint2 *in = nullptr;  // the batch on this device
    int sb = -1;                // staging buffer used (host input), else -1
    int bslot = -1;             // broadcast receive buffer used (rank handles), else -1
    bool ovf = false;           // strict mode: the library's m limit is exceeded (reported by the kernels' word)
};

static int push_check(tc_ctx *ctx, const tc_edge *edges, uint64_t w) {
    if (!ctx) return TC_EINVAL;
    if (ctx->poisoned) return poisoned_code(ctx);
    if (w == 0) return TC_OK;
    if (w > kMaxBatch || (!edges && ctx->rank == 0)) return TC_EINVAL;
    return TC_OK;
}

static int push_prepare(tc_ctx *ctx, const tc_edge *edges, uint64_t w, PushPrep *pp) {
    CK(cudaSetDevice(ctx->device));
    pp->ovf = ctx->m + w > 0x7FFFFFFFull;  // the library's limit: 32-bit device positions (reading R13)
    if (pp->ovf && ctx->async_errors) return TC_EOVERFLOW;  // async mode: reported first, state untouched
    if (ctx->prof && ctx->ev_used == ctx->ev_pool.size()) {  // a new event set for this push
        std::array<cudaEvent_t, 2 * TC_NPHASES + 2 * K_NKERNELS> set{};
        for (auto &e : set)
            if (cudaEventCreate(&e) != cudaSuccess) return fail_cuda(ctx);
        ctx->ev_pool.push_back(set);
        ctx->ev_kused.push_back(0u);
    }
    int rc = grow_index(ctx, w);
    if (rc != TC_OK) return rc;
    IndexBufs &ix = ctx->ix;
    if (ctx->rank == 0) {
        // where are the edges?
        cudaPointerAttributes attr;
        if (cudaPointerGetAttributes(&attr, edges) != cudaSuccess) {
            cudaGetLastError();
            attr.type = cudaMemoryTypeUnregistered;
        }
        const bool on_device = (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged) &&
                               attr.device == ctx->device;
        if (attr.type == cudaMemoryTypeDevice && attr.device != ctx->device) return TC_EINVAL;
        if (on_device) {
            pp->in = reinterpret_cast<const uint2 *>(edges);
        } else {
            // upload on the copy stream into the staging buffer the push before last used (its kernels are done
            // with it: stage_free), so the copy overlaps the previous batch's kernels; the main stream waits
            pp->sb = ctx->stage_next;
            uint2 *dst = pp->sb ? ix.stage2 : ix.stage;
            CK(cudaStreamWaitEvent(ctx->copy, ctx->stage_free[pp->sb], 0));
            CK(cudaMemcpyAsync(dst, edges, 8 * w, cudaMemcpyHostToDevice, ctx->copy));
            CK(cudaEventRecord(ctx->copied[pp->sb], ctx->copy));
            CK(cudaStreamWaitEvent(ctx->stream, ctx->copied[pp->sb], 0));
            if (attr.type == cudaMemoryTypeHost) CK(cudaEventSynchronize(ctx->copied[pp->sb]));  // pinned: reusable
            pp->in = dst;
        }
    }
    if (ctx->nccl) {
        // the batch exchange: ncclBroadcast from rank 0 on the comm stream, into the receive
        // buffer the push before last used (its kernels are done with it: bc_free); rank 0 broadcasts in place
        // from its input.  The main stream waits for the broadcast before its kernels.
        pp->bslot = ctx->bc_next;
        uint2 *recv = ctx->rank == 0 ? const_cast<uint2 *>(pp->in) : ctx->bcast[pp->bslot];
        if (ctx->rank == 0) {
            CK(cudaEventRecord(ctx->inready, ctx->stream));  // the upload / the producer's work, as ordered so far
            CK(cudaStreamWaitEvent(ctx->comm, ctx->inready, 0));
        }
        CK(cudaStreamWaitEvent(ctx->comm, ctx->bc_free[pp->bslot], 0));
        if (nccl().Broadcast(recv, recv, 2 * w, ncclUint32, 0, ctx->nccl, ctx->comm) != ncclSuccess) {
            ctx->poisoned = TC_ENCCL;
            return TC_ENCCL;
        }
        CK(cudaEventRecord(ctx->bc_done, ctx->comm));
        CK(cudaStreamWaitEvent(ctx->stream, ctx->bc_done, 0));
        pp->in = recv;
    }
    return TC_OK;
}

// Event mode: can a vertex degree reach the limit in this batch (m + w > 2^30 - 1)?  Then the degrees are checked
// first and applied by a separate kernel once the batch is accepted.
static bool ed_post(const tc_ctx *ctx, uint64_t w) { return ctx->tune.event_checked || ctx->m + w > (uint64_t)kEdDegMax; }

// a4-a8: the bulk estimator pass (fused, or split per step), or the event mode's kernels
static uint32_t estimator_pass(tc_ctx *ctx, const BatchArgs &a, cudaStream_t s, const KRec &kr) {
    if (ctx->mode == TC_MODE_EVENT) return launch_ed_batch(ctx->ix, a, ctx->ed, ctx->st.stats, ed_post(ctx, a.g.w), s, kr);
    if (ctx->tune.split) return launch_update_split(ctx->ix, ctx->st, ctx->steps, a, s, kr);
    return launch_update(ctx->ix, ctx->st, a, s, kr);
}

// The kernels of one push (after k_desc), on the handle's streams; returns the number of launches.
static uint32_t enqueue_kernels(tc_ctx *ctx, const BatchArgs &a, const KRec &kr, bool *ok_out) {
    IndexBufs &ix = ctx->ix;
    bool ok = true;
    uint32_t launches = 0;
    // profiled pushes run every kernel on the main stream, so each kernel's events time it alone
    cudaStream_t ms = ctx->stream, ss = ctx->prof ? ms : ctx->side, s2 = ctx->prof ? ms : ctx->side2;
    auto rec = [&](int e, cudaStream_t st) {
        if (ctx->prof) ok = ok && cudaEventRecord(ctx->ev_pool[ctx->ev_used][e], st) == cudaSuccess;
    };
    if (a.g.small_index) {  // small batch: the whole index by one CTA, then the estimator pass
        rec(2 * TC_PHASE_PARTITION, ms);
        launches += launch_small_index(ix, a, ms, kr);
        rec(2 * TC_PHASE_PARTITION + 1, ms);
        rec(2 * TC_PHASE_UPDATE, ms);
        launches += estimator_pass(ctx, a, ms, kr);
        rec(2 * TC_PHASE_UPDATE + 1, ms);
        *ok_out = ok;
        return launches;
    }
    // a1: count, scans, scatter (k_count zeroes the counters and this batch's S)
    rec(2 * TC_PHASE_PARTITION, ms);
    launches += launch_partition(ix, a, ms, kr);
    rec(2 * TC_PHASE_PARTITION + 1, ms);
    // a3 (it reads only the raw batch) on the second stream, alongside the vertex phase
    ok = ok && cudaEventRecord(ctx->fork, ms) == cudaSuccess;
    ok = ok && cudaStreamWaitEvent(ss, ctx->fork, 0) == cudaSuccess;
    rec(2 * TC_PHASE_PAIRS, ss);
    launches += launch_pairs(ix, a, ss, kr);
    rec(2 * TC_PHASE_PAIRS + 1, ss);
    ok = ok && cudaEventRecord(ctx->join, ss) == cudaSuccess;
    ok = ok && cudaEventRecord(ctx->fork2, ms) == cudaSuccess;
    // a2: the large vertex buckets on the third stream, the common ones on the main stream
    ok = ok && cudaStreamWaitEvent(s2, ctx->fork2, 0) == cudaSuccess;
    launches += launch_vertices_big(ix, a, s2, kr);
    ok = ok && cudaEventRecord(ctx->join2, s2) == cudaSuccess;
    rec(2 * TC_PHASE_VERTICES, ms);
    launches += launch_vertices(ix, a, ms, kr);
    ok = ok && cudaStreamWaitEvent(ms, ctx->join2, 0) == cudaSuccess;
    rec(2 * TC_PHASE_VERTICES + 1, ms);
    ok = ok && cudaStreamWaitEvent(ms, ctx->join, 0) == cudaSuccess;
    rec(2 * TC_PHASE_UPDATE, ms);
    launches += estimator_pass(ctx, a, ms, kr);
    rec(2 * TC_PHASE_UPDATE + 1, ms);
    *ok_out = ok;
    return launches;
}

static uint32_t *ed_ctr(const tc_ctx *ctx) { return ctx->mode == TC_MODE_EVENT ? ctx->ed.ctr : nullptr; }

// The graph of a batch shape: found in the cache, or captured (k_desc + the kernels) and instantiated.
static int graph_for(tc_ctx *ctx, const BatchArgs &a, const BatchDesc &d, tc_ctx::GraphEntry **out) {
    const uint64_t key = (uint64_t)a.g.w | ((uint64_t)a.small << 32) | ((uint64_t)ctx->tune.split << 33) |
                         ((uint64_t)a.g.small_index << 34) | ((uint64_t)ctx->mode << 35) |
                         ((uint64_t)(ctx->mode == TC_MODE_EVENT && ed_post(ctx, a.g.w)) << 36);
    for (auto &g : ctx->graphs)
        if (g.key == key) {
            g.last_use = ++ctx->graph_clock;
            *out = &g;
            return TC_OK;
        }
    if (ctx->graphs.size() >= 4) {  // evict the least recently used shape
        auto lru = std::min_element(ctx->graphs.begin(), ctx->graphs.end(),
                                    [](const tc_ctx::GraphEntry &x, const tc_ctx::GraphEntry &y) { return x.last_use < y.last_use; });
        if (lru->exec) cudaGraphExecDestroy(lru->exec);
        if (lru->graph) cudaGraphDestroy(lru->graph);
        ctx->graphs.erase(lru);
    }
    tc_ctx::GraphEntry e;
    e.key = key;
    e.last_use = ++ctx->graph_clock;
    CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    launch_desc(ctx->ix, a, d, ed_ctr(ctx), ctx->stream);
    bool ok = true;
    e.launches = 1 + enqueue_kernels(ctx, a, KRec(), &ok);
    const bool cap = cudaStreamEndCapture(ctx->stream, &e.graph) == cudaSuccess && e.graph;
    if (!ok || !cap) {
        if (e.graph) cudaGraphDestroy(e.graph);
        return fail_cuda(ctx);
    }
    size_t n = 0;
    CK(cudaGraphGetNodes(e.graph, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    CK(cudaGraphGetNodes(e.graph, nodes.data(), &n));
    for (auto nd : nodes) {
        cudaGraphNodeType t;
        if (cudaGraphNodeGetType(nd, &t) != cudaSuccess || t != cudaGraphNodeTypeKernel) continue;
        cudaKernelNodeParams kp;
        if (cudaGraphKernelNodeGetParams(nd, &kp) == cudaSuccess && kp.func == desc_kernel()) e.desc_node = nd;
    }
    cudaGetLastError();
    if (!e.desc_node || cudaGraphInstantiate(&e.exec, e.graph, 0) != cudaSuccess) {
        cudaGraphDestroy(e.graph);
        return fail_cuda(ctx);
    }
    ++ctx->graph_captures;
    ctx->graphs.push_back(e);
    *out = &ctx->graphs.back();
    return TC_OK;
}

// Event mode: the persistent vertex table keeps load <= 1/2.  Its count is known exactly at the last settle; each
// edge adds at most 2 vertices, so only when that bound could pass half the capacity does the host settle, read
// the exact count and, if needed, rehash into a larger table (drops the captured graphs: they hold the table).
static int ed_reserve_vertices(tc_ctx *ctx, uint64_t w) {
    const uint64_t cap = (uint64_t)ctx->ed.pv_mask + 1;
    if (ctx->ed_pv_known + 2 * (ctx->m - ctx->ed_m_known) + 2 * w <= cap / 2) return TC_OK;
    int rc = settle(ctx);
    if (rc != TC_OK) return rc;
    uint32_t n = 0;
    CK(cudaMemcpy(&n, ctx->ed.ctr + kEdPVN, 4, cudaMemcpyDeviceToHost));
    ctx->ed_pv_known = n;
    ctx->ed_m_known = ctx->m;
    if (n + 2 * w <= cap / 2) return TC_OK;
    drop_graphs(ctx);
    if (ed_rehash_pv(ctx->ed, 8 * (n + 2 * w), ctx->stream) != 0) return TC_ENOMEM;
    return TC_OK;
}

static int push_launch(tc_ctx *ctx, uint64_t w, const PushPrep &pp) {
    IndexBufs &ix = ctx->ix;
    const int slot = (int)((ctx->b + 1) & 1u);
    BatchArgs a;
    a.first = ctx->first;
    a.seed = ctx->seed;
    a.S = ctx->st.S;
    a.g = make_geometry((uint32_t)w, ctx->tune);
    a.small = ctx->mode == TC_MODE_BULK && (ctx->tune.small == 2 || (ctx->tune.small == 0 && w <= kSmallBatchMax));
    a.pfilt = ctx->mode == TC_MODE_BULK && !ctx->tune.split && !a.g.small_index &&
              (ctx->tune.pair_filter == 2 || (ctx->tune.pair_filter == 0 && w >= kPairFilterMin));
    if (a.pfilt) {  // this batch fills filter `slot`, which must start zeroed; k_count zeroes the other one
        const uint32_t need = pf_words((uint32_t)w);
        if (ctx->pf_zeroed[slot] < need)
            CK(cudaMemsetAsync(ix.pf + (size_t)slot * pf_words((uint32_t)ix.wcap), 0, 4ull * need, ctx->stream));
        ctx->pf_zeroed[slot] = 0;
        ctx->pf_zeroed[slot ^ 1] = std::max(ctx->pf_zeroed[slot ^ 1], need);
    }
    if (++ctx->ptag == 255) {  // edge-pair slot tags 1..254: clear the table once per 254 pushes
        CK(cudaMemsetAsync(ix.pt, 0, 32ull * pair_groups_alloc((uint32_t)ix.wcap), ctx->stream));
        ctx->ptag = 1;
    }
    BatchDesc d;
    d.in = pp.in;
    d.m_prev = ctx->m;
    d.batch = ctx->b;
    d.ptag = ctx->ptag;
    d.slot = (uint32_t)slot;
    d.pad = 0;
    if (ctx->mode == TC_MODE_EVENT) {
        // S carries over; a full sweep early in the stream (m < 8 w), where most estimators change anyway
        const bool full = ctx->m < 8 * w;
        d.pad = 1u | (full ? 2u : 0u) | (ed_post(ctx, w) ? 0u : 4u);
        const int rc = ed_reserve_vertices(ctx, w);
        if (rc != TC_OK) return rc;
    }
    // the error word is sticky in asynchronous mode, and cleared (or set to the overflow error) here in strict
    // mode -- stream operations ahead of the kernels, outside any graph
    if (!ctx->async_errors) {
        CK(cudaMemsetAsync(ix.ctr + kCtrErr, 0, 4, ctx->stream));
        CK(cudaMemsetAsync(ix.ctr + kCtrFailB, 0xFF, 4, ctx->stream));
        if (pp.ovf) CK(cudaMemsetAsync(ix.ctr + kCtrErr, (int)kErrOvf, 1, ctx->stream));
    }
    const bool graph = ctx->use_graph != 0 && !ctx->prof;  // profiling events need plain launches
    uint32_t launches = 0;
    if (graph) {
        tc_ctx::GraphEntry *ge = nullptr;
        const int rc = graph_for(ctx, a, d, &ge);
        if (rc != TC_OK) return rc;
        BatchDesc *dst = ix.desc;
        uint32_t *ctr = ix.ctr;
        unsigned long long *S = a.S;
        uint32_t *filt = a.small ? ix.filt : nullptr;
        uint32_t *edctr = ed_ctr(ctx);
        void *args[] = {&d, &dst, &ctr, &S, &filt, &edctr};
        cudaKernelNodeParams kp{};
        kp.func = const_cast<void *>(desc_kernel());
        kp.gridDim = dim3(1);
        kp.blockDim = dim3(256);
        kp.kernelParams = args;
        CK(cudaGraphExecKernelNodeSetParams(ge->exec, ge->desc_node, &kp));
        CK(cudaGraphLaunch(ge->exec, ctx->stream));
        launches = ge->launches;
    } else {
        KRec kr;
        if (ctx->prof) {
            kr.ev = &ctx->ev_pool[ctx->ev_used][2 * TC_NPHASES];
            ctx->ev_kused[ctx->ev_used] = 0u;
            kr.used = &ctx->ev_kused[ctx->ev_used];
        }
        launch_desc(ix, a, d, ed_ctr(ctx), ctx->stream);
        bool ok = true;
        launches = 1 + enqueue_kernels(ctx, a, kr, &ok);
        if (ctx->prof)
            for (int p = 0; p < TC_NPHASES; ++p)
                ctx->prof_launch[p] += (p == TC_PHASE_PARTITION ? 4 + (a.g.bs ? 1 : 0) : p == TC_PHASE_VERTICES ? 3 : 1);
        if (!ok) return fail_cuda(ctx);
    }
    if (ctx->prof) ++ctx->ev_used;
    CK(cudaGetLastError());
    if (pp.sb >= 0) {
        CK(cudaEventRecord(ctx->stage_free[pp.sb], ctx->stream));
        ctx->stage_next = pp.sb ^ 1;
    }
    if (pp.bslot >= 0) {
        CK(cudaEventRecord(ctx->bc_free[pp.bslot], ctx->stream));
        ctx->bc_next = pp.bslot ^ 1;
    }
    if (!ctx->async_errors) {
        CK(cudaMemcpyAsync(ctx->h_err, ix.ctr + kCtrErr, 4, cudaMemcpyDeviceToHost, ctx->stream));
        WAIT(ctx->stream);
        const int code = decode_err(*ctx->h_err);
        if (code != TC_OK) return code;  // nothing was mutated: k_update bailed out
    }
    if (ctx->async_errors) {
        if (ctx->async_mprev.empty()) ctx->async_b0 = ctx->b;
        ctx->async_mprev.push_back(ctx->m);
    }
    ctx->m += w;
    ctx->b += 1;
    ctx->S_slot = slot;
    ctx->last_launches = launches;
    return TC_OK;
}

int tc_push_batch(tc_ctx *ctx, const tc_edge *edges, uint64_t w) {
    int rc = push_check(ctx, edges, w);
    if (rc != TC_OK || w == 0) return rc;
    if (!ctx->peers.empty()) {  // tc_create_ex group: peer 0 takes the edges, the others receive them
        for (tc_ctx *p : ctx->peers) {
            rc = push_check(p, p->rank == 0 ? edges : nullptr, w);
            if (rc != TC_OK) return rc;
        }
        std::vector<PushPrep> pp(ctx->peers.size());
        if (nccl().GroupStart() != ncclSuccess) return TC_ENCCL;
        int first_err = TC_OK;
        for (size_t g = 0; g < ctx->peers.size(); ++g) {
            tc_ctx *p = ctx->peers[g];
            rc = push_prepare(p, p->rank == 0 ? edges : nullptr, w, &pp[g]);
            if (rc != TC_OK && first_err == TC_OK) first_err = rc;
        }
        if (nccl().GroupEnd() != ncclSuccess && first_err == TC_OK) first_err = TC_ENCCL;
        if (first_err != TC_OK) return first_err;
        for (size_t g = 0; g < ctx->peers.size(); ++g) {
            rc = push_launch(ctx->peers[g], w, pp[g]);
            if (rc != TC_OK && first_err == TC_OK) first_err = rc;
        }
        if (first_err == TC_OK) {
            ctx->m = ctx->peers[0]->m;
            ctx->b = ctx->peers[0]->b;
        }
        return first_err;
    }
    PushPrep pp;
    rc = push_prepare(ctx, edges, w, &pp);
    if (rc != TC_OK) return rc;
    return push_launch(ctx, w, pp);
}

int tc_push_batch_after(tc_ctx *ctx, const tc_edge *edges, uint64_t w, void *producer_stream) {
    if (!ctx) return TC_EINVAL;
    if (producer_stream && w) {
        tc_ctx *c = ctx->peers.empty() ? ctx : ctx->peers[0];  // a group reads the edges on peer 0's device
        if (c->poisoned) return poisoned_code(c);
        if (cudaSetDevice(c->device) != cudaSuccess || cudaEventRecord(c->produced, (cudaStream_t)producer_stream) != cudaSuccess ||
            cudaStreamWaitEvent(c->stream, c->produced, 0) != cudaSuccess)
            return fail_cuda(c);
    }
    return tc_push_batch(ctx, edges, w);
}

// Run f on every peer of a tc_create_ex group (first error wins); f(ctx) itself on any other handle.
extern "C++" {
template <typename F>
static int each(tc_ctx *ctx, F f) {
    if (ctx->peers.empty()) return f(ctx);
    int first = TC_OK;
    for (tc_ctx *p : ctx->peers) {
        const int rc = f(p);
        if (rc != TC_OK && first == TC_OK) first = rc;
    }
    return first;
}
}

int tc_set_graphs(tc_ctx *ctx, int enable) {
    if (!ctx) return TC_EINVAL;
    return each(ctx, [&](tc_ctx *c) -> int {
        int rc = settle(c);
        if (rc != TC_OK) return rc;
        c->use_graph = enable ? 1 : 0;
        return TC_OK;
    });
}

int tc_tune(tc_ctx *ctx, int knob, uint64_t value) {
    if (!ctx) return TC_EINVAL;
    return each(ctx, [&](tc_ctx *c) -> int {
        int rc = settle(c);
        if (rc != TC_OK) return rc;
        drop_graphs(c);  // the geometry of a batch shape may change
        switch (knob) {
            case TC_TUNE_VBUCKET_ARCS:
                if (value < 1 || value > (1u << 30)) return TC_EINVAL;
                c->tune.vbucket_arcs = (uint32_t)value;
                return TC_OK;
            case TC_TUNE_VBUCKET_CAP:
                if (value < 1 || value > 2048) return TC_EINVAL;
                c->tune.vcap = (uint32_t)value;
                return TC_OK;
            case TC_TUNE_SMALL_BATCH:
                if (value > 2) return TC_EINVAL;
                c->tune.small = (uint32_t)value;
                return TC_OK;
            case TC_TUNE_VBUCKET_SORT_CAP:
                if (value < 1 || value > kVChunk) return TC_EINVAL;
                c->tune.sortcap = (uint32_t)value;
                return TC_OK;
            case TC_TUNE_SMALL_INDEX:
                if (value > 2) return TC_EINVAL;
                c->tune.small_index = (uint32_t)value;
                return TC_OK;
            case TC_TUNE_SMALL_INDEX_ARCS:
                if (value < 16 || value > 8192) return TC_EINVAL;
                c->tune.small_index_arcs = (uint32_t)value;
                return TC_OK;
            case TC_TUNE_EVENT_CHECKED:
                if (value > 1) return TC_EINVAL;
                c->tune.event_checked = (uint32_t)value;
                return TC_OK;
            case TC_TUNE_PAIR_FILTER:
                if (value > 2) return TC_EINVAL;
                c->tune.pair_filter = (uint32_t)value;
                return TC_OK;
            case TC_TUNE_SPLIT_KERNELS:
                if (value > 1) return TC_EINVAL;
                if (value && !c->steps.j) {
                    CK2(c, cudaSetDevice(c->device));
                    if (!alloc_steps(c->steps, c->count)) return TC_ENOMEM;
                }
                c->tune.split = (uint32_t)value;
                return TC_OK;
            default:
                return TC_EINVAL;
        }
    });
}

// settle() for calls that are allowed on a handle poisoned by a rejected asynchronous batch (its state is
// that of the last accepted batch): only a CUDA / NCCL failure is an error for them.
static int settle_allow_poisoned(tc_ctx *ctx) {
    const int rc = settle(ctx);
    if (rc == TC_OK || (ctx->poisoned && poisoned_code(ctx) == TC_ESTATE && rc != TC_ECUDA && rc != TC_ENCCL))
        return TC_OK;
    return rc;
}

int tc_reset(tc_ctx *ctx) {
    if (!ctx) return TC_EINVAL;
    const int rc0 = each(ctx, [&](tc_ctx *c) -> int {
        int rc = settle_allow_poisoned(c);
        if (rc != TC_OK) return rc;
        tc_ctx *ctx = c;  // for CK
        launch_init_state(ctx->st, ctx->stream);
        if (ctx->mode == TC_MODE_EVENT) launch_ed_init(ctx->ed, ctx->stream);
        ctx->ed_pv_known = ctx->ed_m_known = 0;
        CK(cudaGetLastError());
        CK(cudaMemsetAsync(ctx->st.S, 0, 16, ctx->stream));
        if (ctx->ix.ctr) {
            CK(cudaMemsetAsync(ctx->ix.ctr, 0, 4 * kCtrWords, ctx->stream));
            CK(cudaMemsetAsync(ctx->ix.ctr + kCtrFailB, 0xFF, 4, ctx->stream));
        }
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->m = 0;
        ctx->b = 0;
        ctx->S_slot = -1;
        ctx->poisoned = 0;
        ctx->async_mprev.clear();
        ctx->async_b0 = 0;
        return TC_OK;
    });
    if (rc0 == TC_OK) {
        ctx->m = 0;
        ctx->b = 0;
    }
    return rc0;
}

int tc_sync(tc_ctx *ctx) {
    if (!ctx) return TC_EINVAL;
    return each(ctx, [](tc_ctx *c) { return settle(c); });
}

// Device scratch for the all-reduces of a rank handle.
static int red_scratch(tc_ctx *ctx, uint64_t words) {
    if (ctx->d_red_words >= words) return TC_OK;
    cudaFree(ctx->d_red);
    ctx->d_red = nullptr;
    ctx->d_red_words = 0;
    if (cudaMalloc(&ctx->d_red, 8 * words) != cudaSuccess) {
        cudaGetLastError();
        return TC_ENOMEM;
    }
    ctx->d_red_words = words;
    return TC_OK;
}

// In-place sum over the ranks of n u64 words on the handle's stream (no-op unless a rank handle).
static int allreduce_u64(tc_ctx *ctx, unsigned long long *dev, uint64_t n) {
    if (!ctx->nccl) return TC_OK;
    if (ctx->nccl_dead) return TC_ENCCL;
    if (nccl().AllReduce(dev, dev, n, ncclUint64, ncclSum, ctx->nccl, ctx->stream) != ncclSuccess) {
        ctx->poisoned = TC_ENCCL;
        return TC_ENCCL;
    }
    return TC_OK;
}

// S of this handle's estimators; on a rank handle the sum over all ranks (a collective: every rank calls).
static int closed_sum_one(tc_ctx *ctx, uint64_t *S) {
    int rc = settle(ctx);
    if (rc != TC_OK) return rc;
    *S = 0;
    if (!ctx->nccl) {
        if (ctx->S_slot >= 0) {
            unsigned long long v = 0;
            CK(cudaMemcpy(&v, ctx->st.S + ctx->S_slot, 8, cudaMemcpyDeviceToHost));
            *S = v;
        }
        return TC_OK;
    }
    rc = red_scratch(ctx, 1);
    if (rc != TC_OK) return rc;
    if (ctx->S_slot >= 0) CK(cudaMemcpyAsync(ctx->d_red, ctx->st.S + ctx->S_slot, 8, cudaMemcpyDeviceToDevice, ctx->stream));
    else CK(cudaMemsetAsync(ctx->d_red, 0, 8, ctx->stream));
    rc = allreduce_u64(ctx, ctx->d_red, 1);
    if (rc != TC_OK) return rc;
    unsigned long long v = 0;
    CK(cudaMemcpyAsync(ctx->h_err + 16, ctx->d_red, 8, cudaMemcpyDeviceToHost, ctx->stream));
    WAIT(ctx->stream);
    std::memcpy(&v, ctx->h_err + 16, 8);
    *S = v;
    return TC_OK;
}

int tc_closed_sum(tc_ctx *ctx, uint64_t *S) {
    if (!ctx || !S) return TC_EINVAL;
    if (ctx->peers.empty()) return closed_sum_one(ctx, S);
    uint64_t tot = 0;
    for (tc_ctx *p : ctx->peers) {  // one process: the host adds the peers' exact sums
        uint64_t v = 0;
        const int rc = p->nccl ? settle(p) : TC_OK;
        if (rc != TC_OK) return rc;
        tc_ctx *ctx = p;  // for CK
        if (p->S_slot >= 0) {
            unsigned long long x = 0;
            CK(cudaMemcpy(&x, p->st.S + p->S_slot, 8, cudaMemcpyDeviceToHost));
            v = x;
        }
        tot += v;
    }
    *S = tot;
    return TC_OK;
}

int tc_estimate(tc_ctx *ctx, double *out) {
    if (!out) return TC_EINVAL;
    uint64_t S = 0;
    int rc = tc_closed_sum(ctx, &S);
    if (rc != TC_OK) return rc;
    *out = (double)ctx->m * (double)S / (double)ctx->r;  // reading R9: one fixed fp64 expression
    return TC_OK;
}

int tc_closed_sum_async(tc_ctx *ctx, uint64_t *S) {
    if (!ctx || !S || !ctx->peers.empty()) return TC_EINVAL;
    if (ctx->poisoned) return poisoned_code(ctx);
    CK(cudaSetDevice(ctx->device));
    if (!ctx->nccl) {
        if (ctx->S_slot < 0) {
            *S = 0;
            return TC_OK;
        }
        CK(cudaMemcpyAsync(S, ctx->st.S + ctx->S_slot, 8, cudaMemcpyDeviceToHost, ctx->stream));
        return TC_OK;
    }
    int rc = red_scratch(ctx, 1);  // rank handle: the all-reduced S, enqueued behind the last batch
    if (rc != TC_OK) return rc;
    if (ctx->S_slot >= 0) CK(cudaMemcpyAsync(ctx->d_red, ctx->st.S + ctx->S_slot, 8, cudaMemcpyDeviceToDevice, ctx->stream));
    else CK(cudaMemsetAsync(ctx->d_red, 0, 8, ctx->stream));
    rc = allreduce_u64(ctx, ctx->d_red, 1);
    if (rc != TC_OK) return rc;
    CK(cudaMemcpyAsync(S, ctx->d_red, 8, cudaMemcpyDeviceToHost, ctx->stream));
    return TC_OK;
}

// S_g over contiguous groups of the GLOBAL ids [floor(g r / G), floor((g+1) r / G)): this handle's part (a
// shard contributes only to the groups its ids fall in), summed over the ranks on a rank handle.
static int group_sums_one(tc_ctx *ctx, uint32_t groups, uint64_t *S_g) {
    int rc = settle(ctx);
    if (rc != TC_OK) return rc;
    unsigned long long *d = nullptr;
    if (ctx->mode == TC_MODE_EVENT) launch_ed_export(ctx->ed, ctx->st, ctx->stream);
    CK(cudaMalloc(&d, 8ull * groups));
    bool ok = cudaMemsetAsync(d, 0, 8ull * groups, ctx->stream) == cudaSuccess;
    if (ok) {
        launch_group_sums(ctx->st, ctx->first, ctx->r, groups, d, ctx->stream);
        ok = cudaGetLastError() == cudaSuccess;
    }
    if (ok) rc = allreduce_u64(ctx, d, groups);
    ok = ok && rc == TC_OK && cudaMemcpyAsync(S_g, d, 8ull * groups, cudaMemcpyDeviceToHost, ctx->stream) == cudaSuccess;
    const int wrc = ok ? wait_stream(ctx, ctx->stream) : TC_OK;
    cudaFree(d);
    if (rc != TC_OK) return rc;
    if (wrc != TC_OK) return wrc;
    return ok ? TC_OK : fail_cuda(ctx);
}

int tc_group_sums(tc_ctx *ctx, uint32_t groups, uint64_t *S_g) {
    if (!ctx || !S_g || groups == 0 || groups > ctx->r) return TC_EINVAL;
    if (ctx->peers.empty()) return group_sums_one(ctx, groups, S_g);
    std::vector<uint64_t> part(groups);
    std::fill(S_g, S_g + groups, 0ull);
    for (tc_ctx *p : ctx->peers) {
        ncclComm_t saved = p->nccl;  // no all-reduce inside one process: the host adds the peers' vectors
        p->nccl = nullptr;
        const int rc = group_sums_one(p, groups, part.data());
        p->nccl = saved;
        if (rc != TC_OK) return rc;
        for (uint32_t g = 0; g < groups; ++g) S_g[g] += part[g];
    }
    return TC_OK;
}

int tc_required_estimators(double eps, double delta, uint64_t m, uint64_t Delta, uint64_t tau, uint64_t *r) {
    if (!r || !(eps > 0.0) || !(delta > 0.0 && delta < 1.0) || tau == 0) return TC_EINVAL;
    if (Delta && m > UINT64_MAX / Delta) return TC_EINVAL;
    const double x = 96.0 / (eps * eps) * ((double)(m * Delta) / (double)tau) * std::log(1.0 / delta);
    const double c = std::ceil(x);
    if (!(c < 18446744073709551616.0)) return TC_EOVERFLOW;
    *r = (uint64_t)c;
    return TC_OK;
}

int tc_estimate_mom(tc_ctx *ctx, uint32_t groups, double *out) {
    if (!ctx || !out || groups == 0 || groups > ctx->r) return TC_EINVAL;
    // the groups cover all r estimators: a lone shard (tc_create_shard with count < r) has only its part
    if (ctx->peers.empty() && !ctx->nccl && ctx->count != ctx->r) return TC_EINVAL;
    std::vector<uint64_t> S(groups);
    int rc = tc_group_sums(ctx, groups, S.data());
    if (rc != TC_OK) return rc;
    std::vector<double> means(groups);
    const uint64_t n = ctx->r;
    for (uint32_t g = 0; g < groups; ++g) {
        const uint64_t lo = (uint64_t)g * n / groups, hi = (uint64_t)(g + 1) * n / groups;
        // group mean of X_i = chi_i * m: (double)m * (double)S_g / (double)|g|, the oracle's expression
        // (nbsi.median_of_means); no 64-bit product m * S_g, which could wrap
        means[g] = (double)ctx->m * (double)S[g] / (double)(hi - lo);
    }
    std::sort(means.begin(), means.end());
    *out = means[(groups - 1) / 2];
    return TC_OK;
}

int tc_get_state(tc_ctx *ctx, uint64_t first, uint64_t count, uint32_t *r1, uint64_t *p1, uint32_t *r2,
                 uint64_t *p2, uint32_t *c, uint8_t *closed) {
    if (ctx && !ctx->peers.empty()) {  // a group: [first, first + count) of the global ids, across the peers
        if (first > ctx->r || count > ctx->r - first) return TC_EINVAL;
        for (tc_ctx *p : ctx->peers) {
            const uint64_t lo = std::max(first, p->first), hi = std::min(first + count, p->first + p->count);
            if (lo >= hi) continue;
            const uint64_t o = lo - first;
            const int rc = tc_get_state(p, lo - p->first, hi - lo, r1 ? r1 + 2 * o : nullptr, p1 ? p1 + o : nullptr,
                                        r2 ? r2 + 2 * o : nullptr, p2 ? p2 + o : nullptr, c ? c + o : nullptr,
                                        closed ? closed + o : nullptr);
            if (rc != TC_OK) return rc;
        }
        return TC_OK;
    }
    if (!ctx || first > ctx->count || count > ctx->count - first) return TC_EINVAL;
    int rc = settle_allow_poisoned(ctx);
    if (rc != TC_OK) return rc;
    if (count == 0) return TC_OK;
    if (ctx->mode == TC_MODE_EVENT) {
        launch_ed_export(ctx->ed, ctx->st, ctx->stream);
        CK(cudaStreamSynchronize(ctx->stream));
    }
    if (r1) CK(cudaMemcpy(r1, ctx->st.r1 + first, 8 * count, cudaMemcpyDeviceToHost));
    if (r2) CK(cudaMemcpy(r2, ctx->st.r2 + first, 8 * count, cudaMemcpyDeviceToHost));
    if (p1 || p2) {  // stored as u32 (positions < 2^31, reading R13); 0xFFFFFFFF -> UINT64_MAX
        std::vector<uint32_t> q(count);
        for (int f = 0; f < 2; ++f) {
            uint64_t *dst = f ? p2 : p1;
            if (!dst) continue;
            CK(cudaMemcpy(q.data(), (f ? ctx->st.p2 : ctx->st.p1) + first, 4 * count, cudaMemcpyDeviceToHost));
            for (uint64_t i = 0; i < count; ++i) dst[i] = q[i] == 0xFFFFFFFFu ? ~0ull : (uint64_t)q[i];
        }
    }
    if (c || closed) {
        std::vector<uint32_t> cf(count);
        CK(cudaMemcpy(cf.data(), ctx->st.cf + first, 4 * count, cudaMemcpyDeviceToHost));
        for (uint64_t i = 0; i < count; ++i) {
            if (c) c[i] = cf[i] & kCMask;
            if (closed) closed[i] = (cf[i] & kClosedBit) ? 1 : 0;
        }
    }
    return TC_OK;
}

// S of the restored state, into the accumulator slot the next push does not overwrite
static int recompute_S(tc_ctx *ctx) {
    if (ctx->b == 0) {
        ctx->S_slot = -1;
        return TC_OK;
    }
    const int slot = (int)(ctx->b & 1u);
    if (ctx->mode == TC_MODE_EVENT) launch_ed_export(ctx->ed, ctx->st, ctx->stream);
    CK(cudaMemsetAsync(ctx->st.S + slot, 0, 8, ctx->stream));
    launch_group_sums(ctx->st, 0, 1, 1, ctx->st.S + slot, ctx->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->S_slot = slot;
    return TC_OK;
}

int tc_set_state(tc_ctx *ctx, uint64_t first, uint64_t count, const uint32_t *r1, const uint64_t *p1,
                 const uint32_t *r2, const uint64_t *p2, const uint32_t *c, const uint8_t *closed) {
    if (!ctx || !ctx->peers.empty() || first > ctx->count || count > ctx->count - first) return TC_EINVAL;
    if (count && (!r1 || !p1 || !r2 || !p2 || !c || !closed)) return TC_EINVAL;
    if (ctx->mode == TC_MODE_EVENT) return TC_EINVAL;  // the event mode's state has more than the NBSI fields
    int rc = settle(ctx);
    if (rc != TC_OK) return rc;
    std::vector<uint32_t> q1(count), q2(count), cf(count);
    for (uint64_t i = 0; i < count; ++i) {  // validate everything before touching the device
        for (int f = 0; f < 2; ++f) {
            const uint32_t lo = (f ? r2 : r1)[2 * i], hi = (f ? r2 : r1)[2 * i + 1];
            const uint64_t p = (f ? p2 : p1)[i];
            const bool empty = lo == 0xFFFFFFFFu && hi == 0xFFFFFFFFu;
            if (empty != (p == ~0ull)) return TC_EINVAL;
            if (!empty && (lo >= hi || p >= 0x7FFFFFFFull)) return TC_EINVAL;
            (f ? q2 : q1)[i] = empty ? 0xFFFFFFFFu : (uint32_t)p;
        }
        if (c[i] > kCMask || closed[i] > 1) return TC_EINVAL;
        // NBSI as the estimator pass relies on it: an empty f1 has nothing else;
        // chi == 0 <=> f2 empty; closed => f2 present; f2 after f1 and sharing exactly one endpoint
        const bool e1 = q1[i] == 0xFFFFFFFFu, e2 = q2[i] == 0xFFFFFFFFu;
        if (e1 && (!e2 || c[i] || closed[i])) return TC_EINVAL;
        if ((c[i] == 0) != e2 || (closed[i] && e2)) return TC_EINVAL;
        if (!e2) {
            const uint32_t a0 = r1[2 * i], a1 = r1[2 * i + 1], b0 = r2[2 * i], b1 = r2[2 * i + 1];
            const int shared = (a0 == b0) + (a0 == b1) + (a1 == b0) + (a1 == b1);
            if (shared != 1 || q2[i] <= q1[i]) return TC_EINVAL;
        }
        cf[i] = c[i] | (closed[i] ? kClosedBit : 0u);
    }
    if (count) {
        CK(cudaMemcpy(ctx->st.r1 + first, r1, 8 * count, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->st.r2 + first, r2, 8 * count, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->st.p1 + first, q1.data(), 4 * count, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->st.p2 + first, q2.data(), 4 * count, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->st.cf + first, cf.data(), 4 * count, cudaMemcpyHostToDevice));
    }
    return recompute_S(ctx);
}

int tc_set_counters(tc_ctx *ctx, uint64_t m, uint32_t batches) {
    if (!ctx || !ctx->peers.empty() || m > 0x7FFFFFFFull || (batches == 0) != (m == 0)) return TC_EINVAL;
    if (ctx->mode == TC_MODE_EVENT) return TC_EINVAL;
    int rc = settle(ctx);
    if (rc != TC_OK) return rc;
    ctx->m = m;
    ctx->b = batches;
    return recompute_S(ctx);
}

int tc_counters(tc_ctx *ctx, uint64_t *m, uint32_t *batches) {
    if (!ctx) return TC_EINVAL;
    if (!ctx->peers.empty()) return tc_counters(ctx->peers[0], m, batches);  // every peer saw every batch
    if (ctx->async_errors) {  // enqueued batches count only once they are known to be accepted
        const int rc = settle_allow_poisoned(ctx);
        if (rc != TC_OK) return rc;
    }
    if (m) *m = ctx->m;
    if (batches) *batches = ctx->b;
    return TC_OK;
}

int tc_set_async(tc_ctx *ctx, int async_errors) {
    if (!ctx) return TC_EINVAL;
    return each(ctx, [&](tc_ctx *c) -> int {
        int rc = settle(c);
        if (rc != TC_OK) return rc;
        c->async_errors = async_errors ? 1 : 0;
        return TC_OK;
    });
}

int tc_set_mode(tc_ctx *ctx, int mode) {
    if (!ctx || (mode != TC_MODE_BULK && mode != TC_MODE_EVENT)) return TC_EINVAL;
    return each(ctx, [&](tc_ctx *c) -> int {
        int rc = settle(c);
        if (rc != TC_OK) return rc;
        if (c->m != 0 || c->b != 0) return TC_EINVAL;
        if (mode == c->mode) return TC_OK;
        tc_ctx *ctx = c;  // for CK
        drop_graphs(c);
        ed_free(c->ed);
        c->mode = TC_MODE_BULK;
        if (mode == TC_MODE_EVENT) {
            const uint64_t pv_cap = 8 * std::max<uint64_t>(2 * c->ix.wcap, 2048);
            if (!ed_alloc(c->ed, c->count, c->first, c->seed, pv_cap) || (c->ix.wcap && !ed_alloc_seg(c->ed, c->ix.wcap))) {
                ed_free(c->ed);
                return TC_ENOMEM;
            }
            launch_ed_init(c->ed, c->stream);
            CK(cudaGetLastError());
            CK(cudaMemsetAsync(c->st.S, 0, 16, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            c->ed_pv_known = c->ed_m_known = 0;
            c->mode = TC_MODE_EVENT;
        }
        return TC_OK;
    });
}

int tc_get_event_state(tc_ctx *ctx, uint64_t first, uint64_t count, uint32_t *J, uint32_t *K, uint32_t *ev) {
    if (ctx && !ctx->peers.empty()) {
        if (first > ctx->r || count > ctx->r - first) return TC_EINVAL;
        for (tc_ctx *p : ctx->peers) {
            const uint64_t lo = std::max(first, p->first), hi = std::min(first + count, p->first + p->count);
            if (lo >= hi) continue;
            const uint64_t o = lo - first;
            const int rc = tc_get_event_state(p, lo - p->first, hi - lo, J ? J + o : nullptr, K ? K + o : nullptr,
                                              ev ? ev + o : nullptr);
            if (rc != TC_OK) return rc;
        }
        return TC_OK;
    }
    if (!ctx || ctx->mode != TC_MODE_EVENT || first > ctx->count || count > ctx->count - first) return TC_EINVAL;
    int rc = settle_allow_poisoned(ctx);
    if (rc != TC_OK) return rc;
    if (count == 0) return TC_OK;
    if (J) CK(cudaMemcpy(J, ctx->ed.J + first, 4 * count, cudaMemcpyDeviceToHost));
    if (K) CK(cudaMemcpy(K, ctx->ed.K + first, 4 * count, cudaMemcpyDeviceToHost));
    if (ev) CK(cudaMemcpy(ev, ctx->ed.ev + first, 4 * count, cudaMemcpyDeviceToHost));
    return TC_OK;
}

int tc_event_counters(tc_ctx *ctx, uint64_t *out, int n) {
    if (!ctx || !out || !ctx->peers.empty() || ctx->mode != TC_MODE_EVENT) return TC_EINVAL;
    int rc = settle_allow_poisoned(ctx);
    if (rc != TC_OK) return rc;
    uint32_t v[kEdWords];
    CK(cudaMemcpy(v, ctx->ed.ctr, 4 * kEdWords, cudaMemcpyDeviceToHost));
    const uint64_t vals[4] = {v[kEdVisited], v[kEdEvents], v[kEdSweeps], v[kEdPVN]};
    for (int i = 0; i < n && i < 4; ++i) out[i] = vals[i];
    return 4;
}

void *tc_stream(tc_ctx *ctx) {
    if (ctx && !ctx->peers.empty()) ctx = ctx->peers[0];
    return ctx ? (void *)ctx->stream : nullptr;
}

int tc_profile(tc_ctx *ctx, int enable) {
    if (!ctx || !ctx->peers.empty()) return TC_EINVAL;
    int rc = settle(ctx);
    if (rc != TC_OK) return rc;
    ctx->prof = enable ? 1 : 0;
    CK(cudaMemsetAsync(ctx->st.stats, 0, 8 * kNStats, ctx->stream));
    for (int p = 0; p < TC_NPHASES; ++p) {
        ctx->prof_ms[p] = 0;
        ctx->prof_launch[p] = 0;
    }
    for (int k = 0; k < K_NKERNELS; ++k) {
        ctx->prof_kms[k] = 0;
        ctx->prof_klaunch[k] = 0;
    }
    return TC_OK;
}

int tc_profile_kernels(tc_ctx *ctx, double *ms, uint64_t *launches, int n) {
    if (!ctx || !ctx->peers.empty()) return TC_EINVAL;
    int rc = settle(ctx);
    if (rc != TC_OK) return rc;
    for (int k = 0; k < n && k < K_NKERNELS; ++k) {
        if (ms) ms[k] = ctx->prof_kms[k];
        if (launches) launches[k] = ctx->prof_klaunch[k];
    }
    return K_NKERNELS;
}

const char *tc_kernel_name(int k) {
    static const char *names[K_NKERNELS] = {"k_count", "k_scan_cols", "k_scan_tot", "k_scatter", "k_split",
                                            "k_pairs", "k_vhub", "k_vbig", "k_vhash", "k_update",
                                            "k_u1_resample", "k_u2_count", "k_u3_select", "k_u4_close", "k_r_reduce",
                                            "k_small_index", "k_ed_pre", "k_ed_trigger", "k_ed_process",
                                            "k_ed_post", "k_ed_front"};
    return (k >= 0 && k < K_NKERNELS) ? names[k] : "";
}

int tc_profile_read(tc_ctx *ctx, double *ms, uint64_t *launches, int n) {
    if (!ctx || !ctx->peers.empty()) return TC_EINVAL;
    int rc = settle(ctx);
    if (rc != TC_OK) return rc;
    for (int p = 0; p < n && p < TC_NPHASES; ++p) {
        if (ms) ms[p] = ctx->prof_ms[p];
        if (launches) launches[p] = ctx->prof_launch[p];
    }
    return TC_NPHASES;
}

int tc_stats(tc_ctx *ctx, uint64_t *out, int n) {
    if (!ctx || !out || !ctx->peers.empty()) return TC_EINVAL;
    int rc = settle(ctx);
    if (rc != TC_OK) return rc;
    unsigned long long v[kNStats];
    CK(cudaMemcpy(v, ctx->st.stats, 8 * kNStats, cudaMemcpyDeviceToHost));
    for (int i = 0; i < n && i < kNStats; ++i) out[i] = v[i];
    return kNStats;
}

int tc_graph_captures(tc_ctx *ctx, uint64_t *captures) {
    if (!ctx || !captures) return TC_EINVAL;
    *captures = 0;
    if (!ctx->peers.empty())
        for (tc_ctx *p : ctx->peers) *captures += p->graph_captures;
    else
        *captures = ctx->graph_captures;
    return TC_OK;
}

int tc_last_launches(tc_ctx *ctx, uint32_t *launches) {
    if (!ctx || !launches) return TC_EINVAL;
    *launches = 0;
    if (!ctx->peers.empty())
        for (tc_ctx *p : ctx->peers) *launches += p->last_launches;
    else
        *launches = ctx->last_launches;
    return TC_OK;
}

int tc_get_steps(tc_ctx *ctx, uint64_t first, uint64_t count, uint32_t *j, uint32_t *chim, uint32_t *ld, uint32_t *rd,
                 uint64_t *d2, uint32_t *k2) {
    if (!ctx || !ctx->peers.empty() || !ctx->steps.j || first > ctx->count || count > ctx->count - first)
        return TC_EINVAL;
    int rc = settle_allow_poisoned(ctx);
    if (rc != TC_OK) return rc;
    if (count == 0) return TC_OK;
    const StepBufs &sb = ctx->steps;
    if (j) CK(cudaMemcpy(j, sb.j + first, 4 * count, cudaMemcpyDeviceToHost));
    if (chim) CK(cudaMemcpy(chim, sb.chim + first, 4 * count, cudaMemcpyDeviceToHost));
    if (ld) CK(cudaMemcpy(ld, sb.ld + first, 4 * count, cudaMemcpyDeviceToHost));
    if (rd) CK(cudaMemcpy(rd, sb.rd + first, 4 * count, cudaMemcpyDeviceToHost));
    if (d2) CK(cudaMemcpy(d2, sb.d2 + first, 8 * count, cudaMemcpyDeviceToHost));
    if (k2) CK(cudaMemcpy(k2, sb.k2 + first, 4 * count, cudaMemcpyDeviceToHost));
    return TC_OK;
}

// ------------------------------------------------------------------------------------------------
// Multi-GPU handles.

int tc_nccl_unique_id(void *id) {
    if (!id) return TC_EINVAL;
    if (!nccl().ok) return TC_ENCCL;
    ncclUniqueId u;
    if (nccl().GetUniqueId(&u) != ncclSuccess) return TC_ENCCL;
    std::memcpy(id, &u, sizeof(u));
    return TC_OK;
}

// Give a freshly created shard handle its communicator and the broadcast machinery.
static int attach_comm(tc_ctx *ctx, ncclComm_t comm, int rank, int world) {
    ctx->nccl = comm;
    ctx->rank = rank;
    ctx->world = world;
    if (const char *t = std::getenv("TC_NCCL_TIMEOUT_S")) ctx->nccl_timeout_s = std::atof(t);
    CK(cudaSetDevice(ctx->device));
    CK(cudaStreamCreateWithFlags(&ctx->comm, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->bc_done, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->inready, cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i) CK(cudaEventCreateWithFlags(&ctx->bc_free[i], cudaEventDisableTiming));
    if (ctx->ix.wcap) {  // the index was preallocated before the communicator existed: add the receive buffers
        for (int i = 0; i < 2; ++i)
            if (cudaMalloc(&ctx->bcast[i], 8 * ctx->ix.wcap) != cudaSuccess) {
                cudaGetLastError();
                return TC_ENOMEM;
            }
    }
    return TC_OK;
}

tc_ctx *tc_create_rank(uint64_t r, uint64_t seed, int rank, int world, const void *nccl_unique_id, int device,
                       uint64_t w_max_hint) {
    g_last_error = TC_OK;
    if (r == 0 || world < 1 || rank < 0 || rank >= world || !nccl_unique_id) {
        g_last_error = TC_EINVAL;
        return nullptr;
    }
    if (!nccl().ok) {
        g_last_error = TC_ENCCL;
        return nullptr;
    }
    const uint64_t first = (uint64_t)rank * r / (uint64_t)world;
    const uint64_t count = (uint64_t)(rank + 1) * r / (uint64_t)world - first;
    tc_ctx *ctx = tc_create_shard(r, seed, first, count, device, w_max_hint);
    if (!ctx) return nullptr;
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof(id));
    ncclComm_t comm = nullptr;
    cudaSetDevice(ctx->device);
    if (nccl().CommInitRank(&comm, world, id, rank) != ncclSuccess) {
        destroy_ctx(ctx);
        g_last_error = TC_ENCCL;
        return nullptr;
    }
    const int rc = attach_comm(ctx, comm, rank, world);
    if (rc != TC_OK) {
        destroy_ctx(ctx);
        g_last_error = rc;
        return nullptr;
    }
    return ctx;
}

tc_ctx *tc_create_ex(uint64_t r, uint64_t seed, const tc_config *cfg) {
    g_last_error = TC_OK;
    tc_config def{};
    if (!cfg) cfg = &def;
    const int G = cfg->ngpus < 1 ? 1 : cfg->ngpus;
    std::vector<int> devs(G);
    for (int g = 0; g < G; ++g) devs[g] = cfg->devices ? cfg->devices[g] : (G == 1 ? -1 : g);
    auto configure = [&](tc_ctx *c) -> int {
        return tc_set_async(c, cfg->strict_errors ? 0 : 1) == TC_OK && tc_set_graphs(c, cfg->graphs ? 1 : 0) == TC_OK;
    };
    if (G == 1) {  // one GPU: a plain handle
        tc_ctx *ctx = tc_create_shard(r, seed, 0, r, devs[0], cfg->w_max_hint);
        if (ctx && !configure(ctx)) {
            destroy_ctx(ctx);
            g_last_error = TC_ECUDA;
            return nullptr;
        }
        return ctx;
    }
    if (r == 0) {
        g_last_error = TC_EINVAL;
        return nullptr;
    }
    if (!nccl().ok) {
        g_last_error = TC_ENCCL;
        return nullptr;
    }
    std::vector<ncclComm_t> comms(G, nullptr);
    if (nccl().CommInitAll(comms.data(), G, devs.data()) != ncclSuccess) {
        g_last_error = TC_ENCCL;
        return nullptr;
    }
    tc_ctx *grp = new (std::nothrow) tc_ctx();
    if (!grp) {
        for (auto c : comms) nccl().CommDestroy(c);
        g_last_error = TC_ENOMEM;
        return nullptr;
    }
    grp->r = r;
    grp->seed = seed;
    grp->count = r;
    grp->device = devs[0];
    for (int g = 0; g < G; ++g) {
        const uint64_t first = (uint64_t)g * r / (uint64_t)G, count = (uint64_t)(g + 1) * r / (uint64_t)G - first;
        tc_ctx *p = tc_create_shard(r, seed, first, count, devs[g], cfg->w_max_hint);
        const int rc = p ? attach_comm(p, comms[g], g, G) : tc_last_error();
        if (p) grp->peers.push_back(p);
        else nccl().CommDestroy(comms[g]);
        if (rc != TC_OK || !configure(p)) {
            for (int h = g + 1; h < G; ++h) nccl().CommDestroy(comms[h]);
            destroy_ctx(grp);
            g_last_error = rc != TC_OK ? rc : TC_ECUDA;
            return nullptr;
        }
    }
    return grp;
}

int tc_rank_info(tc_ctx *ctx, int *rank, int *world, uint64_t *first, uint64_t *count) {
    if (!ctx) return TC_EINVAL;
    if (rank) *rank = ctx->rank;
    if (world) *world = ctx->peers.empty() ? ctx->world : (int)ctx->peers.size();
    if (first) *first = ctx->first;
    if (count) *count = ctx->count;
    return TC_OK;
}

// Test hooks: copy host arrays in, run the device function, copy the results out (own stream-less path on
// the current device; synchronous).
int tc_test_draws(const uint64_t *n, const uint64_t *x, const uint64_t *id, const uint32_t *b, const uint32_t *base,
                  uint64_t seed, uint64_t count, uint64_t *out) {
    if (!count) return TC_OK;
    if (!n || !x || !id || !b || !base || !out) return TC_EINVAL;
    for (uint64_t i = 0; i < count; ++i)
        if (n[i] == 0) return TC_EINVAL;
    uint64_t *d = nullptr;
    const size_t B8 = 8 * count, B4 = 4 * count;
    if (cudaMalloc(&d, 4 * B8 + 2 * B4) != cudaSuccess) {
        cudaGetLastError();
        return TC_ENOMEM;
    }
    uint64_t *dn = d, *dx = d + count, *did = d + 2 * count, *dout = d + 3 * count;
    uint32_t *db = reinterpret_cast<uint32_t *>(d + 4 * count), *dbase = db + count;
    bool ok = cudaMemcpy(dn, n, B8, cudaMemcpyHostToDevice) == cudaSuccess &&
              cudaMemcpy(dx, x, B8, cudaMemcpyHostToDevice) == cudaSuccess &&
              cudaMemcpy(did, id, B8, cudaMemcpyHostToDevice) == cudaSuccess &&
              cudaMemcpy(db, b, B4, cudaMemcpyHostToDevice) == cudaSuccess &&
              cudaMemcpy(dbase, base, B4, cudaMemcpyHostToDevice) == cudaSuccess;
    if (ok) {
        launch_test_draws(dn, dx, did, db, dbase, seed, count, dout, 0);
        ok = cudaGetLastError() == cudaSuccess && cudaMemcpy(out, dout, B8, cudaMemcpyDeviceToHost) == cudaSuccess;
    }
    cudaFree(d);
    if (!ok) cudaGetLastError();
    return ok ? TC_OK : TC_ECUDA;
}

int tc_test_philox(const uint32_t *ctr, const uint32_t *key, uint64_t count, uint32_t *out) {
    if (!count) return TC_OK;
    if (!ctr || !key || !out) return TC_EINVAL;
    uint32_t *d = nullptr;
    if (cudaMalloc(&d, 40 * count) != cudaSuccess) {
        cudaGetLastError();
        return TC_ENOMEM;
    }
    uint32_t *dc = d, *dk = d + 4 * count, *dout = d + 6 * count;
    bool ok = cudaMemcpy(dc, ctr, 16 * count, cudaMemcpyHostToDevice) == cudaSuccess &&
              cudaMemcpy(dk, key, 8 * count, cudaMemcpyHostToDevice) == cudaSuccess;
    if (ok) {
        launch_test_philox(dc, dk, count, dout, 0);
        ok = cudaGetLastError() == cudaSuccess && cudaMemcpy(out, dout, 16 * count, cudaMemcpyDeviceToHost) == cudaSuccess;
    }
    cudaFree(d);
    if (!ok) cudaGetLastError();
    return ok ? TC_OK : TC_ECUDA;
}

const char *tc_strerror(int code) {
    switch (code) {
        case TC_OK: return "ok";
        case TC_EINVAL: return "invalid argument or reserved vertex id 0xFFFFFFFF";
        case TC_ENOMEM: return "out of memory";
        case TC_ESELFLOOP: return "self-loop in batch";
        case TC_EDUP: return "duplicate edge in batch";
        case TC_EOVERFLOW: return "stream longer than 2^31-1 edges (chi field overflow)";
        case TC_ECUDA: return "CUDA error";
        case TC_ESTATE: return "handle poisoned by an earlier asynchronous error";
        case TC_ENCCL: return "NCCL error (communicator aborted)";
        case TC_EINTERNAL: return "internal bounds check failed (TC_CHECKED build)";
        case TC_EPARSE: return "malformed edge-list line";
        case TC_EIO: return "cannot open or read the edge-list file";
        default: return "unknown error";
    }
}

int tc_last_error(void) { return g_last_error; }

}  // extern "C"

// kernels.h -- launch wrappers of the per-batch pipeline (kernels.cu).  Host-side, internal.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "index.cuh"

namespace tcb {

struct IndexBufs {
    uint64_t wcap = 0;         // edges the buffers hold
    uint2 *E = nullptr;        // [wcap] normalized edges
    uint32_t *keyA = nullptr, *valA = nullptr;  // [2 wcap] radix ping-pong buffers: arc vertex / arc value
    uint32_t *keyB = nullptr, *valB = nullptr;
    uint32_t *hist = nullptr;  // [kPasses * kRadix] digit histograms of the arc keys
    uint32_t *cnt = nullptr;   // [kRadix * tiles] per-tile digit counts -> offsets (current pass)
    uint64_t tiles_cap = 0;
    uint4 *einfo = nullptr;    // [wcap] {slot_lo, end_lo, slot_hi, end_hi}
    VSlot *vt = nullptr;       // [vmask+1]
    uint32_t vmask = 0;
    PSlot *pt = nullptr;       // [pmask+1]
    uint32_t pmask = 0;
    uint32_t *ctr = nullptr;   // device counters (index.cuh kCtr*)
    uint2 *stage = nullptr;    // [wcap] H2D staging for host batches
};

struct StateBufs {
    uint64_t count = 0;
    uint2 *r1 = nullptr, *r2 = nullptr;
    uint32_t *cf = nullptr;  // chi in bits 0..30, closed flag in bit 31
    uint64_t *p1 = nullptr, *p2 = nullptr;
    unsigned long long *S = nullptr;  // [2] closed-sum accumulators (double-buffered by batch parity)
    unsigned long long *stats = nullptr;  // [4] fresh f1, replaced f2 of retained f1, sum of D, batches
};

struct BatchArgs {
    const uint2 *in;  // w raw edges (device)
    uint32_t w;
    uint64_t m_prev;
    uint32_t batch;  // index b of this (non-empty) batch
    uint32_t tag;    // table tag of this push (never reused while a table slot may carry it)
    uint64_t first;  // global id of local estimator 0
    uint64_t seed;
    int S_slot;
};

// Each returns the number of kernel launches issued.
int launch_stage(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s);
int launch_pairs(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s);
int launch_sort(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s);
int launch_segment(const IndexBufs &ix, const BatchArgs &a, cudaStream_t s);
int launch_update(const IndexBufs &ix, const StateBufs &st, const BatchArgs &a, cudaStream_t s);
int launch_init_tables(const IndexBufs &ix, cudaStream_t s);

int launch_init_state(const StateBufs &st, cudaStream_t s);
int launch_group_sums(const StateBufs &st, uint32_t groups, unsigned long long *out, cudaStream_t s);
int launch_unpack_state(const StateBufs &st, uint64_t first, uint64_t count, uint32_t *c, uint8_t *closed,
                        cudaStream_t s);

int sm_count();

}  // namespace tcb

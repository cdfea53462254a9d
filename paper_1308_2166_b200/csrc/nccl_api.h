// nccl_api.h -- NCCL entry points, resolved at run time with dlopen("libnccl.so.2").
//
// The library needs NCCL only for multi-GPU handles (tc_create_rank / tc_create_ex with ngpus > 1: the
// per-batch broadcast of the edges and the all-reduce of the exact partial sums).  Loading
// it lazily keeps single-GPU use free of the dependency, and in a process that already has NCCL loaded (e.g.
// by PyTorch) dlopen returns that same library, so every rank uses one NCCL.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

namespace tcb {

struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t *, int, const int *) = nullptr;
    ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
};

// The process-wide NCCL entry points (ok == false if libnccl.so.2 cannot be loaded).
inline const NcclApi &nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        bool all = true;
        auto sym = [&](auto &fn, const char *name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            all = all && fn != nullptr;
        };
        sym(a.GetUniqueId, "ncclGetUniqueId");
        sym(a.CommInitRank, "ncclCommInitRank");
        sym(a.CommInitAll, "ncclCommInitAll");
        sym(a.Broadcast, "ncclBroadcast");
        sym(a.AllReduce, "ncclAllReduce");
        sym(a.CommGetAsyncError, "ncclCommGetAsyncError");
        sym(a.CommAbort, "ncclCommAbort");
        sym(a.CommDestroy, "ncclCommDestroy");
        sym(a.GroupStart, "ncclGroupStart");
        sym(a.GroupEnd, "ncclGroupEnd");
        a.ok = all;
        return a;
    }();
    return api;
}

}  // namespace tcb

"""paper_1308_2166_b200 -- B200 (sm_100a) bulk neighborhood-sampling triangle estimator.

Thin Python binding of the C ABI in include/tc.h (``libtc_b200.so``).  The binding only marshals
arguments; the whole per-batch update (Steps 1-3 of bulkUpdateAll) runs in the
library's CUDA kernels.  PyTorch, when used, only supplies device memory and streams.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from ._lib import PHASES, TCError

__all__ = ["TriangleCounter", "TCError", "PHASES", "load_library", "required_estimators", "exact_triangles", "parse_edges",
           "test_draws", "test_philox", "nccl_unique_id"]


def load_library():
    return _lib.load()


def required_estimators(eps: float, delta: float, m: int, Delta: int, tau: int) -> int:
    """tc_required_estimators: r = ceil(96/eps^2 * m*Delta/tau * ln(1/delta))."""
    out = C.c_uint64()
    rc = _lib.load().tc_required_estimators(float(eps), float(delta), int(m), int(Delta), int(tau), C.byref(out))
    if rc != 0:
        raise TCError(rc, "tc_required_estimators")
    return int(out.value)


def exact_triangles(edges, timing: bool = False):
    """tc_exact_triangles: tau = |T(G)| of the simple graph with these edges, on the
    current CUDA device.  edges: (m, 2) uint32 numpy array or uint32/int32 torch tensor (host or cuda).
    Returns tau, or (tau, device_ms) with timing=True."""
    ptr, m, keep = _edges_ptr(edges)
    tau, ms = C.c_uint64(), C.c_double()
    rc = _lib.load().tc_exact_triangles(ptr, int(m), C.byref(tau), C.byref(ms))
    del keep
    if rc != 0:
        raise TCError(rc, "tc_exact_triangles")
    return (int(tau.value), float(ms.value)) if timing else int(tau.value)


def parse_edges(text: bytes, final: bool = True, skip_loops: bool = False, cap: int | None = None):
    """tc_parse_edges on a bytes chunk: returns (edges (n, 2) uint32, bytes consumed, lines consumed)."""
    buf = bytes(text)
    cap = len(buf) // 4 + 1 if cap is None else int(cap)  # an edge line takes >= 4 bytes ("1 2\n")
    out = np.empty((cap, 2), dtype=np.uint32)
    n, used, lines = C.c_uint64(), C.c_uint64(), C.c_uint64()
    rc = _lib.load().tc_parse_edges(buf, len(buf), int(final), _lib.TC_INGEST_SKIP_LOOPS if skip_loops else 0,
                                    out.ctypes.data_as(C.c_void_p), cap, C.byref(n), C.byref(used), C.byref(lines))
    if rc != 0:
        err = TCError(rc, f"tc_parse_edges (line {lines.value})")
        err.line = int(lines.value)
        raise err
    return out[:n.value].copy(), int(used.value), int(lines.value)


def test_draws(n, x, ids, b, base, seed):
    """tc_test_draws: the device bounded uniform on chosen inputs (uint64 arrays n, x, ids; uint32 b, base)."""
    P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    n, x, ids = (np.ascontiguousarray(v, dtype=np.uint64) for v in (n, x, ids))
    b, base = (np.ascontiguousarray(v, dtype=np.uint32) for v in (b, base))
    out = np.empty(len(n), np.uint64)
    rc = _lib.load().tc_test_draws(P(n), P(x), P(ids), P(b), P(base), int(seed), len(n), P(out))
    if rc != 0:
        raise TCError(rc, "tc_test_draws")
    return out


def test_philox(ctr, key):
    """tc_test_philox: device Philox4x32-10 blocks; ctr (k, 4) and key (k, 2) uint32 -> (k, 4) uint32."""
    P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    ctr = np.ascontiguousarray(ctr, dtype=np.uint32).reshape(-1, 4)
    key = np.ascontiguousarray(key, dtype=np.uint32).reshape(-1, 2)
    out = np.empty_like(ctr)
    rc = _lib.load().tc_test_philox(P(ctr), P(key), ctr.shape[0], P(out))
    if rc != 0:
        raise TCError(rc, "tc_test_philox")
    return out


def _producer_stream(edges):
    """cudaStream_t (int) of torch's current stream when edges is a CUDA tensor (the stream that produced
    it, by torch's convention), else None."""
    if type(edges).__module__.startswith("torch") and edges.is_cuda:
        import torch
        return torch.cuda.current_stream(edges.device).cuda_stream
    return None


def _edges_ptr(edges):
    """(pointer, w, keepalive) for a numpy (host) or torch (host / cuda) array of shape (w, 2) uint32."""
    mod = type(edges).__module__
    if mod.startswith("torch"):
        import torch
        t = edges
        if t.dtype not in (torch.int32, torch.uint32):
            raise TypeError("edges must be a uint32/int32 tensor of shape (w, 2)")
        if t.dim() != 2 or t.shape[1] != 2 or not t.is_contiguous():
            raise ValueError("edges must be contiguous with shape (w, 2)")
        return C.c_void_p(t.data_ptr()), t.shape[0], t
    a = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
    return a.ctypes.data_as(C.c_void_p), a.shape[0], a


def nccl_unique_id() -> bytes:
    """tc_nccl_unique_id: a fresh 128-byte ncclUniqueId (rank 0 creates it and shares it out of band)."""
    buf = C.create_string_buffer(128)
    rc = _lib.load().tc_nccl_unique_id(buf)
    if rc != 0:
        raise TCError(rc, "tc_nccl_unique_id")
    return buf.raw


class TriangleCounter:
    """r estimators (or the shard [first, first+count) of them) on one GPU.

    tc_create(r, seed) / tc_create_shard(...), tc_push_batch, tc_estimate, tc_destroy (include/tc.h).
    Multi-GPU: TriangleCounter.rank(...) (tc_create_rank: one process per GPU, NCCL inside the library) and
    TriangleCounter.multi(...) (tc_create_ex: one process, several GPUs).
    """

    def __init__(self, r: int, seed: int, first: int = 0, count: int | None = None, device: int = -1,
                 w_max_hint: int = 0, _handle=None):
        L = _lib.load()
        self.r, self.seed, self.first = int(r), int(seed), int(first)
        self.count = self.r - self.first if count is None else int(count)
        self.rank_id, self.world = 0, 1
        if _handle is not None:
            self._h = _handle
            return
        self._h = L.tc_create_shard(self.r, self.seed, self.first, self.count, int(device), int(w_max_hint))
        if not self._h:
            raise TCError(L.tc_last_error(), "tc_create_shard")

    @classmethod
    def rank(cls, r: int, seed: int, rank: int, world: int, unique_id: bytes, device: int = -1, w_max_hint: int = 0):
        """tc_create_rank: this rank's shard [floor(rank r / world), floor((rank+1) r / world)) with an NCCL
        communicator; push_batch / estimate / closed_sum / group_sums are then collective (every rank calls
        them; ranks other than 0 pass edges=None with the batch size w)."""
        L = _lib.load()
        uid = C.create_string_buffer(bytes(unique_id), 128)
        h = L.tc_create_rank(int(r), int(seed), int(rank), int(world), uid, int(device), int(w_max_hint))
        if not h:
            raise TCError(L.tc_last_error(), "tc_create_rank")
        return cls._wrap(h, r, seed)

    @classmethod
    def multi(cls, r: int, seed: int, devices, strict: bool = False, graphs: bool = True, w_max_hint: int = 0):
        """tc_create_ex: one handle over the GPUs `devices` of this process (ncclCommInitAll)."""
        L = _lib.load()
        devs = (C.c_int * len(devices))(*[int(d) for d in devices])
        cfg = _lib.TCConfig(len(devices), devs, 1 if strict else 0, 1 if graphs else 0, int(w_max_hint))
        h = L.tc_create_ex(int(r), int(seed), C.byref(cfg))
        if not h:
            raise TCError(L.tc_last_error(), "tc_create_ex")
        return cls._wrap(h, r, seed)

    @classmethod
    def _wrap(cls, h, r, seed):
        rk, wd, first, count = C.c_int(), C.c_int(), C.c_uint64(), C.c_uint64()
        _lib.load().tc_rank_info(h, C.byref(rk), C.byref(wd), C.byref(first), C.byref(count))
        obj = cls(r, seed, first=int(first.value), count=int(count.value), _handle=h)
        obj.rank_id, obj.world = int(rk.value), int(wd.value)
        return obj

    # -- lifecycle -------------------------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            _lib.load().tc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- the path ------------------------------------------------------------------------------
    def push_batch(self, edges, check: bool = True, w: int | None = None) -> int:
        """tc_push_batch; a CUDA tensor goes through tc_push_batch_after with torch's current stream as the
        producer, so the engine's stream waits for the kernels / copies that wrote it.  On a rank handle the
        ranks other than 0 pass edges=None and the batch size w."""
        if edges is None:
            rc = _lib.load().tc_push_batch(self._h, None, int(w))
            if check and rc != 0:
                raise TCError(rc, "tc_push_batch")
            return rc
        ptr, w, keep = _edges_ptr(edges)
        prod = _producer_stream(edges)
        if prod is not None:
            rc = _lib.load().tc_push_batch_after(self._h, ptr, int(w), C.c_void_p(prod))
        else:
            rc = _lib.load().tc_push_batch(self._h, ptr, int(w))
        del keep
        if check and rc != 0:
            raise TCError(rc, "tc_push_batch")
        return rc

    def push_batch_ptr(self, ptr: int, w: int) -> int:
        """Raw pointer form (device or host address of w tc_edge); returns the status code."""
        return _lib.load().tc_push_batch(self._h, C.c_void_p(ptr), int(w))

    def ingest_file(self, path: str, w: int, skip_loops: bool = False) -> dict:
        """tc_ingest_file: stream a SNAP-format edge list through push_batch in batches of w (a reader
        thread parses ahead into two pinned buffers).  Returns the tc_ingest_stats fields as a dict."""
        st = _lib.IngestStats()
        rc = _lib.load().tc_ingest_file(self._h, os.fsencode(path), int(w),
                                        _lib.TC_INGEST_SKIP_LOOPS if skip_loops else 0, C.byref(st))
        out = {f: getattr(st, f) for f, _ in st._fields_}
        if rc != 0:
            err = TCError(rc, "tc_ingest_file" + (f" (line {st.error_line})" if st.error_line else ""))
            err.stats = out
            raise err
        return out

    def estimate(self) -> float:
        out = C.c_double()
        self._ck(_lib.load().tc_estimate(self._h, C.byref(out)), "tc_estimate")
        return out.value

    def closed_sum(self) -> int:
        out = C.c_uint64()
        self._ck(_lib.load().tc_closed_sum(self._h, C.byref(out)), "tc_closed_sum")
        return int(out.value)

    def closed_sum_async(self, buf, index: int = 0):
        """tc_closed_sum_async: enqueue the copy of the last batch's S into buf[index] (a pinned host torch
        int64 tensor, or a numpy uint64/int64 array); valid after the next successful sync."""
        if type(buf).__module__.startswith("torch"):
            if buf.device.type != "cpu" or buf.element_size() != 8:
                raise TypeError("buf must be a host 8-byte tensor")
            ptr = buf.data_ptr() + 8 * int(index)
        else:
            if buf.dtype.itemsize != 8:
                raise TypeError("buf must hold 8-byte integers")
            ptr = buf.ctypes.data + 8 * int(index)
        self._ck(_lib.load().tc_closed_sum_async(self._h, C.c_void_p(ptr)), "tc_closed_sum_async")

    def estimate_mom(self, groups: int) -> float:
        out = C.c_double()
        self._ck(_lib.load().tc_estimate_mom(self._h, int(groups), C.byref(out)), "tc_estimate_mom")
        return out.value

    def group_sums(self, groups: int) -> np.ndarray:
        out = np.zeros(int(groups), np.uint64)
        self._ck(_lib.load().tc_group_sums(self._h, int(groups), out.ctypes.data_as(C.c_void_p)), "tc_group_sums")
        return out

    def state(self, first: int = 0, count: int | None = None) -> dict:
        n = self.count - first if count is None else count
        r1 = np.empty((n, 2), np.uint32)
        r2 = np.empty((n, 2), np.uint32)
        p1 = np.empty(n, np.uint64)
        p2 = np.empty(n, np.uint64)
        c = np.empty(n, np.uint32)
        closed = np.empty(n, np.uint8)
        P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        self._ck(_lib.load().tc_get_state(self._h, int(first), int(n), P(r1), P(p1), P(r2), P(p2), P(c), P(closed)),
                 "tc_get_state")
        return dict(r1=r1, p1=p1, r2=r2, p2=p2, c=c, closed=closed)

    def set_state(self, state: dict, first: int = 0):
        """tc_set_state: restore estimators [first, first + n) from a dict in state()'s layout."""
        a = {f: np.ascontiguousarray(state[f], dtype=t) for f, t in
             (("r1", np.uint32), ("p1", np.uint64), ("r2", np.uint32), ("p2", np.uint64), ("c", np.uint32),
              ("closed", np.uint8))}
        n = len(a["c"])
        P = lambda x: x.ctypes.data_as(C.c_void_p)  # noqa: E731
        self._ck(_lib.load().tc_set_state(self._h, int(first), n, P(a["r1"]), P(a["p1"]), P(a["r2"]), P(a["p2"]),
                                          P(a["c"]), P(a["closed"])), "tc_set_state")

    def set_counters(self, m: int, batches: int):
        """tc_set_counters: restore m and the number of accepted batches (resume a checkpointed stream)."""
        self._ck(_lib.load().tc_set_counters(self._h, int(m), int(batches)), "tc_set_counters")

    def counters(self):
        m, b = C.c_uint64(), C.c_uint32()
        self._ck(_lib.load().tc_counters(self._h, C.byref(m), C.byref(b)), "tc_counters")
        return int(m.value), int(b.value)

    def reset(self):
        """Back to the freshly created state (tc_reset); allocations are kept."""
        self._ck(_lib.load().tc_reset(self._h), "tc_reset")

    def set_async(self, on: bool = True):
        self._ck(_lib.load().tc_set_async(self._h, 1 if on else 0), "tc_set_async")

    def set_graphs(self, on: bool = True):
        self._ck(_lib.load().tc_set_graphs(self._h, 1 if on else 0), "tc_set_graphs")

    def graph_captures(self) -> int:
        out = C.c_uint64()
        self._ck(_lib.load().tc_graph_captures(self._h, C.byref(out)), "tc_graph_captures")
        return int(out.value)

    def set_mode(self, mode: str):
        """tc_set_mode: "bulk" (the paper's bulkUpdateAll, default) or "event" (skip-sampled neighborhood
        sampling that visits only the estimators a batch changes).  Fresh handles only."""
        code = {"bulk": 0, "event": 1}[mode]
        self._ck(_lib.load().tc_set_mode(self._h, code), "tc_set_mode")

    def event_state(self, first: int = 0, count: int | None = None) -> dict:
        """tc_get_event_state: J (next f1 replacement time, 1-based), K (adjacency count of the next f2
        replacement), ev (random words used); 0xFFFFFFFF = never."""
        n = self.count - first if count is None else count
        out = dict(J=np.empty(n, np.uint32), K=np.empty(n, np.uint32), ev=np.empty(n, np.uint32))
        P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        self._ck(_lib.load().tc_get_event_state(self._h, int(first), int(n), P(out["J"]), P(out["K"]), P(out["ev"])),
                 "tc_get_event_state")
        return out

    def event_counters(self) -> dict:
        v = np.zeros(4, np.uint64)
        rc = _lib.load().tc_event_counters(self._h, v.ctypes.data_as(C.c_void_p), 4)
        if rc < 0:
            self._ck(rc, "tc_event_counters")
        return dict(visited=int(v[0]), events=int(v[1]), sweeps=int(v[2]), vertices=int(v[3]))

    def tune(self, **knobs):
        """Index-geometry knobs (tc_tune): vbucket_arcs, vbucket_cap, vbucket_sort_cap."""
        for k, v in knobs.items():
            self._ck(_lib.load().tc_tune(self._h, _lib.TUNE[k], int(v)), f"tc_tune({k})")

    def steps(self, first: int = 0, count: int | None = None) -> dict:
        """tc_get_steps: the per-step values of the last batch (split estimator pass, tune(split_kernels=1))."""
        n = self.count - first if count is None else count
        out = dict(j=np.empty(n, np.uint32), chi_m=np.empty(n, np.uint32), ld=np.empty(n, np.uint32),
                   rd=np.empty(n, np.uint32), d2=np.empty(n, np.uint64), k2=np.empty(n, np.uint32))
        P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        self._ck(_lib.load().tc_get_steps(self._h, int(first), int(n), *[P(out[f]) for f in
                                                                         ("j", "chi_m", "ld", "rd", "d2", "k2")]),
                 "tc_get_steps")
        return out

    def sync(self) -> int:
        return _lib.load().tc_sync(self._h)

    @property
    def stream_ptr(self) -> int:
        return int(_lib.load().tc_stream(self._h) or 0)

    def profile(self, on: bool = True):
        self._ck(_lib.load().tc_profile(self._h, 1 if on else 0), "tc_profile")

    def profile_read(self):
        ms = np.zeros(_lib.TC_NPHASES, np.float64)
        n = np.zeros(_lib.TC_NPHASES, np.uint64)
        rc = _lib.load().tc_profile_read(self._h, ms.ctypes.data_as(C.c_void_p), n.ctypes.data_as(C.c_void_p),
                                         _lib.TC_NPHASES)
        if rc < 0:
            raise TCError(rc, "tc_profile_read")
        return {p: (float(ms[i]), int(n[i])) for i, p in enumerate(PHASES)}

    def profile_kernels(self):
        """tc_profile_kernels: {kernel name: (total ms, launches)} since the last profile() call."""
        L = _lib.load()
        n = L.tc_profile_kernels(self._h, None, None, 0)
        if n < 0:
            raise TCError(n, "tc_profile_kernels")
        ms = np.zeros(n, np.float64)
        cnt = np.zeros(n, np.uint64)
        L.tc_profile_kernels(self._h, ms.ctypes.data_as(C.c_void_p), cnt.ctypes.data_as(C.c_void_p), n)
        return {L.tc_kernel_name(k).decode(): (float(ms[k]), int(cnt[k])) for k in range(n)}

    def stats(self) -> dict:
        out = np.zeros(7, np.uint64)
        rc = _lib.load().tc_stats(self._h, out.ctypes.data_as(C.c_void_p), 7)
        if rc < 0:
            raise TCError(rc, "tc_stats")
        return {"fresh": int(out[0]), "r2_replaced_retained": int(out[1]), "vertices": int(out[2]),
                "batches": int(out[3]), "skipped": int(out[4]), "arcs_big": int(out[5]), "vertices_big": int(out[6])}

    def last_launches(self) -> int:
        out = C.c_uint32()
        self._ck(_lib.load().tc_last_launches(self._h, C.byref(out)), "tc_last_launches")
        return int(out.value)

    @staticmethod
    def _ck(rc, where):
        if rc != 0:
            raise TCError(rc, where)

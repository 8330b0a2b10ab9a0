"""Thin ctypes binding of include/mspipe.h (libmspipe.so).  Argument marshalling
only: every step of the stage runs in the library's sm_100a kernels.  There
is no CPU fallback — a missing library or a non-CUDA tensor raises.

Names mirror the C entry points without the ``mspipe_`` prefix.
"""
from __future__ import annotations

import ctypes as C
import gc
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MSPIPE_LIB") or os.path.join(_HERE, "libmspipe.so")  # override: debug builds only

OK, EINVAL, ERANGE, ESTALE, EORDER, EUNSUPPORTED, ECUDA, ENCCL = 0, -1, -2, -3, -4, -5, -6, -7
FP32_SIMT, FP32_3XTF32, BF16 = 0, 1, 2
ABI_VERSION = 2

P = C.c_void_p
i32, i64, f32, f64 = C.c_int32, C.c_int64, C.c_float, C.c_double

EXPORTS = ("mspipe_abi_version", "mspipe_last_error", "mspipe_check", "mspipe_sample_recent",
           "mspipe_sample_batch", "mspipe_memory_create", "mspipe_memory_destroy",
           "mspipe_memory_committed", "mspipe_memory_reset", "mspipe_memory_fetch",
           "mspipe_memory_dedup", "mspipe_gru_create", "mspipe_gru_destroy", "mspipe_memory_update",
           "mspipe_memory_writeback", "mspipe_memory_prep", "mspipe_gru_workspace_size",
           "mspipe_message_build", "mspipe_gru_apply", "mspipe_gru_apply_commit", "mspipe_util_event_record",
           "mspipe_memory_local_rows", "mspipe_nccl_unique_id", "mspipe_memory_writeback_keyed",
           "mspipe_shard_fetch_plan", "mspipe_shard_fetch_serve", "mspipe_shard_fetch_finish",
           "mspipe_shard_commit_pack", "mspipe_shard_commit_merge", "mspipe_shard_exchange", "mspipe_shard_loopback",
           "mspipe_util_graph_begin", "mspipe_util_graph_end", "mspipe_util_graph_launch", "mspipe_util_graph_destroy",
           "mspipe_memory_double_buffer", "mspipe_memory_tables", "mspipe_memory_set_committed",
           "mspipe_plan_timeline", "mspipe_plan_min_staleness", "mspipe_stale_histogram",
           "mspipe_feature_fetch", "mspipe_updater_create",
           "mspipe_message_build_deferred", "mspipe_memory_mail_deferred",
           "mspipe_util_rows_to_host",
           "mspipe_gru_apply_commit_out", "mspipe_plan_stale_fractions", "mspipe_staleness_error",
           "mspipe_shard_window_handle", "mspipe_shard_connect", "mspipe_shard_connect_local",
           "mspipe_shard_sent_bytes", "mspipe_util_record_to_device", "mspipe_shard_mitigation_candidates",
           "mspipe_shard_fetch_finish_table", "mspipe_shard_mitigate", "mspipe_train_layout", "mspipe_train_create",
           "mspipe_train_destroy", "mspipe_gru_save_gates", "mspipe_train_step", "mspipe_train_sgd",
           "mspipe_apan_create", "mspipe_apan_destroy", "mspipe_message_build_apan", "mspipe_apan_deliver",
           "mspipe_util_kernel_events", "mspipe_apan_refresh_keys")
XCHG_FETCH_IDS, XCHG_FETCH_ROWS, XCHG_COMMIT = 0, 1, 2


class MspipeError(RuntimeError):
    def __init__(self, status, where, text):
        super().__init__(f"{where}: status {status}: {text}")
        self.status = status


class Tcsr(C.Structure):
    _fields_ = [("num_nodes", i64), ("nnz", i64), ("indptr", P), ("nbr", P), ("eid", P), ("ts", P)]


class Mitigation(C.Structure):
    _fields_ = [("lam", f32), ("gamma", f64), ("n_sim", i32), ("fanout", i32), ("g", C.POINTER(Tcsr)),
                ("src", P), ("dst", P), ("ts", P), ("num_events", i64), ("out_h", P), ("out_omega", P),
                ("out_elig", P)]


_lib = None


def lib():
    """Load libmspipe.so (built by paper_2402_15113_b200.build.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                               "(nvcc, sm_100a). There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        L.mspipe_abi_version.restype = i32
        L.mspipe_last_error.restype = C.c_char_p
        L.mspipe_check.argtypes = [P]
        L.mspipe_sample_recent.argtypes = [C.POINTER(Tcsr), P, P, i64, i32, P, P, P, P, P, P, P]
        L.mspipe_sample_batch.argtypes = [C.POINTER(Tcsr), P, P, P, P, i64, i32, P, P, P, P, P, P, P]
        L.mspipe_memory_create.argtypes = [C.POINTER(P), i64, i32, i32, i32, P, P, P, P, i64, i32, i32, P]
        L.mspipe_memory_destroy.argtypes = [P]
        L.mspipe_memory_committed.argtypes = [P]
        L.mspipe_memory_committed.restype = i64
        L.mspipe_memory_reset.argtypes = [P, i32, P]
        L.mspipe_memory_fetch.argtypes = [P, i64, P, i64, P, P, P, P, C.POINTER(Mitigation),
                                          C.POINTER(i64), P]
        L.mspipe_gru_create.argtypes = [C.POINTER(P), i32, i32, i32, i32, i64, P, P, P, P, P, P, P]
        L.mspipe_gru_destroy.argtypes = [P]
        L.mspipe_memory_dedup.argtypes = [P, P, P, i64, P, P, P, P]
        L.mspipe_memory_update.argtypes = [P, P, P, P, P, i64, P, P, P, i64, P, P, P, P, P, P, P]
        L.mspipe_memory_writeback.argtypes = [P, i64, P, P, i64, P, P, P, P]
        L.mspipe_util_event_record.argtypes = [P, P]
        L.mspipe_memory_double_buffer.argtypes = [P, P, P, P, P]
        L.mspipe_memory_set_committed.argtypes = [P, i64]
        L.mspipe_plan_timeline.argtypes = [P, i64, P, P, P]
        L.mspipe_plan_min_staleness.argtypes = [P, i64, i32, P, C.POINTER(i64)]
        L.mspipe_stale_histogram.argtypes = [C.POINTER(Tcsr), P, P, i64, i64, i32, P, P]
        L.mspipe_plan_stale_fractions.argtypes = [P, i32, P, i32, P]
        L.mspipe_staleness_error.argtypes = [P, P, i64, P, i64, P, i64, i32, P, P]
        L.mspipe_memory_tables.argtypes = [P, i64, C.POINTER(P), C.POINTER(P), C.POINTER(P), C.POINTER(P)]
        L.mspipe_util_rows_to_host.argtypes = [P, P, P, P, i64, P, P, i64, i64, P]
        L.mspipe_util_graph_begin.argtypes = [P]
        L.mspipe_util_graph_end.argtypes = [P, C.POINTER(P)]
        L.mspipe_util_graph_launch.argtypes = [P, P]
        L.mspipe_util_graph_destroy.argtypes = [P]
        L.mspipe_memory_prep.argtypes = [P, C.POINTER(Tcsr), i64, P, P, P, P, i64, i32, P, P, P, P, P, P, P, P, P, P,
                                         P, P, P, C.POINTER(Mitigation), C.POINTER(i64), P]
        L.mspipe_updater_create.argtypes = [C.POINTER(P), i32, i32, i32, i32, i32, i32, i64, P, P, P, P, P, P, P]
        L.mspipe_message_build_deferred.argtypes = [P, P, i64, P, P, P, i64, i64, P, P, P, P, C.c_size_t, P]
        L.mspipe_memory_mail_deferred.argtypes = [P, i64, P, P, P, P, i64, P, P, P, P]
        L.mspipe_feature_fetch.argtypes = [P, P, i64, i32, P, i64, i32, P, i64, i32, P, P, P]
        L.mspipe_gru_workspace_size.argtypes = [P, i64]
        L.mspipe_gru_workspace_size.restype = C.c_size_t
        L.mspipe_message_build.argtypes = [P, P, i64, P, P, P, i64, P, P, P, P, P, i64, P, C.c_size_t, P]
        L.mspipe_gru_apply.argtypes = [P, i64, P, i64, P, P, P, P, P, C.c_size_t, P]
        L.mspipe_gru_apply_commit.argtypes = [P, P, i64, i64, P, i64, P, P, P, P, P, P, P, P, C.c_size_t, P]
        L.mspipe_gru_apply_commit_out.argtypes = [P, P, i64, i64, P, i64, P, P, P, P, P, P, P, P, P, P,
                                                  C.c_size_t, P]
        L.mspipe_memory_local_rows.argtypes = [P]
        L.mspipe_memory_local_rows.restype = i64
        L.mspipe_nccl_unique_id.argtypes = [P, i32]
        L.mspipe_memory_writeback_keyed.argtypes = [P, i64, P, P, P, i64, i64, P, P, P, P]
        L.mspipe_shard_fetch_plan.argtypes = [P, i64, P, i64, i32, P]
        L.mspipe_shard_fetch_serve.argtypes = [P, P]
        L.mspipe_shard_fetch_finish.argtypes = [P, P, i64, P, P, P, P, C.POINTER(i64), P]
        L.mspipe_shard_commit_pack.argtypes = [P, i64, P, P, P, i64, i64, P, P, P, P]
        L.mspipe_shard_commit_merge.argtypes = [P, i64, P]
        L.mspipe_shard_exchange.argtypes = [P, i32, P]
        L.mspipe_shard_loopback.argtypes = [P, i32, i32, P]
        L.mspipe_shard_window_handle.argtypes = [P, P, i32]
        L.mspipe_shard_connect.argtypes = [P, P, i32]
        L.mspipe_shard_connect_local.argtypes = [P, i32]
        L.mspipe_shard_sent_bytes.argtypes = [P, P]
        L.mspipe_util_record_to_device.argtypes = [P, P, i64, P]
        L.mspipe_shard_mitigation_candidates.argtypes = [P, C.POINTER(Mitigation), P, i64, P, P]
        L.mspipe_shard_fetch_finish_table.argtypes = [P, P, i64, P, P, P]
        L.mspipe_shard_mitigate.argtypes = [P, C.POINTER(Mitigation), P, P, P]
        L.mspipe_train_layout.argtypes = [i32, i32, i32, i32, P]
        L.mspipe_train_layout.restype = i64
        L.mspipe_train_create.argtypes = [C.POINTER(P), P, i64, i32, i32, i64, P, P, P]
        L.mspipe_train_destroy.argtypes = [P]
        L.mspipe_gru_save_gates.argtypes = [P, P]
        L.mspipe_train_step.argtypes = [P, P, i64, P, P, P, P, P, P, P, P, C.c_size_t, P, P, P, P]
        L.mspipe_train_sgd.argtypes = [P, P, f32, P]
        L.mspipe_util_kernel_events.argtypes = [P, P]
        L.mspipe_apan_create.argtypes = [C.POINTER(P), i64, i32, i32, i32, i64, P, P, P, P, P, P, P]
        L.mspipe_apan_destroy.argtypes = [P]
        L.mspipe_apan_refresh_keys.argtypes = [P, P]
        L.mspipe_message_build_apan.argtypes = [P, P, P, i64, P, P, i64, P, P, P, P, P, C.c_size_t, P]
        L.mspipe_apan_deliver.argtypes = [P, P, i64, P, P, P, P, i64, P, P, P, P, P, i32, P]
        if L.mspipe_abi_version() != ABI_VERSION:
            raise RuntimeError(f"libmspipe ABI {L.mspipe_abi_version()} != binding {ABI_VERSION}")
        _lib = L
    return _lib


def _ck(status, where):
    if status != OK:
        raise MspipeError(status, where, lib().mspipe_last_error().decode(errors="replace"))


def ptr(t):
    """Device pointer of a CUDA tensor (None -> NULL).  Refuses host tensors."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("libmspipe takes CUDA tensors (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError("libmspipe takes contiguous tensors")
    return C.c_void_p(t.data_ptr())


def stream_ptr(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def check(stream=None):
    _ck(lib().mspipe_check(stream_ptr(stream)), "mspipe_check")


def last_error() -> str:
    return lib().mspipe_last_error().decode(errors="replace")


def kernel_events(begin, end):
    """The next gru_apply_commit of this thread brackets its GEMM kernel with (begin, end)."""
    _ck(lib().mspipe_util_kernel_events(C.c_void_p(begin.cuda_event) if begin is not None else None,
                                        C.c_void_p(end.cuda_event) if end is not None else None),
        "kernel_events")


def event_record(event: torch.cuda.Event, stream=None):
    """Record a timing event so that it is also captured as a graph node."""
    _ck(lib().mspipe_util_event_record(C.c_void_p(event.cuda_event), stream_ptr(stream)), "event_record")


def _host_ptr(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def plan_timeline(tau, num_iters, k=None):
    """Eq. 3-4 on the host (mspipe_plan_timeline): (b, e) arrays [num_iters, 5]."""
    import numpy as np
    t = np.ascontiguousarray(tau, dtype=np.float64)
    assert t.shape == (5,)
    kk = None if k is None else np.ascontiguousarray(k, dtype=np.int32)
    b = np.zeros((num_iters, 5))
    e = np.zeros((num_iters, 5))
    _ck(lib().mspipe_plan_timeline(_host_ptr(t), int(num_iters), _host_ptr(kk), _host_ptr(b), _host_ptr(e)),
        "mspipe_plan_timeline")
    return b, e


def plan_min_staleness(tau, num_iters, k_max):
    """Minimal k_i under C1-C3 (mspipe_plan_min_staleness): (k array, first infeasible iteration or 0)."""
    import numpy as np
    t = np.ascontiguousarray(tau, dtype=np.float64)
    assert t.shape == (5,)
    k = np.zeros(num_iters, np.int32)
    bad = i64(0)
    _ck(lib().mspipe_plan_min_staleness(_host_ptr(t), int(num_iters), int(k_max), _host_ptr(k), C.byref(bad)),
        "mspipe_plan_min_staleness")
    return k, int(bad.value)


def plan_stale_fractions(hist, k_values):
    """Stale share per paper staleness k (mspipe_plan_stale_fractions, host)."""
    import numpy as np
    h = np.ascontiguousarray(hist.cpu().numpy() if isinstance(hist, torch.Tensor) else hist, dtype=np.int64)
    k = np.ascontiguousarray(k_values, dtype=np.int32)
    out = np.zeros(len(k), np.float64)
    _ck(lib().mspipe_plan_stale_fractions(_host_ptr(h), len(h), _host_ptr(k), len(k), _host_ptr(out)),
        "mspipe_plan_stale_fractions")
    return out


def staleness_error(winner, num_unique, num_events, rows_a, stride_a, rows_b, stride_b, mem_dim, out, stream=None):
    """‖x − s‖_F of one batch's update targets into the device f64 scalar `out`."""
    _ck(lib().mspipe_staleness_error(ptr(winner), ptr(num_unique), int(num_events), ptr(rows_a), int(stride_a),
                                     ptr(rows_b), int(stride_b), int(mem_dim), ptr(out), stream_ptr(stream)),
        "mspipe_staleness_error")


def stale_histogram(g: "TcsrHandle", src, dst, batch, max_d=64, stream=None):
    """C3 statistic on the GPU (mspipe_stale_histogram): int64 device tensor [max_d + 2]."""
    out = torch.empty(max_d + 2, dtype=torch.int64, device=src.device)
    _ck(lib().mspipe_stale_histogram(C.byref(g.c), ptr(src), ptr(dst), src.numel(), int(batch), int(max_d),
                                     ptr(out), stream_ptr(stream)), "mspipe_stale_histogram")
    return out


def record_to_device(dst, host_src, stream=None):
    """H2D of a pinned host record into a device buffer (mspipe_util_record_to_device)."""
    n = host_src.numel() * host_src.element_size()
    _ck(lib().mspipe_util_record_to_device(ptr(dst), C.c_void_p(host_src.data_ptr()), n, stream_ptr(stream)),
        "mspipe_util_record_to_device")


def rows_to_host(num, host_num, a, host_a, b, host_b, max_rows, stream=None):
    """Zero-copy read-back of the first *num rows of a and b into pinned host tensors."""
    def hp(t):
        return C.c_void_p(t.data_ptr())
    _ck(lib().mspipe_util_rows_to_host(ptr(num), hp(host_num), ptr(a), hp(host_a), a[0].numel() * a.element_size(),
                                       ptr(b), hp(host_b), b[0].numel() * b.element_size(), int(max_rows),
                                       stream_ptr(stream)), "mspipe_util_rows_to_host")


_capture_seq = 0  # bumped at every capture start: events of another capture must not be waited on


def capture_seq():
    return _capture_seq


class StepGraph:
    """One captured step (mspipe_util_graph_*).  Capture must not allocate: the
    stage's buffers are preallocated, and an allocation during capture raises."""

    def __init__(self):
        self.exec = C.c_void_p()

    def capture(self, fn, stream):
        global _capture_seq
        _capture_seq += 1
        # a handle freed by the cyclic GC mid-capture would cudaFree inside it
        # and invalidate the capture: collect first, and keep the GC off meanwhile
        gc.collect()
        was_enabled = gc.isenabled()
        gc.disable()
        before = torch.cuda.memory_stats(stream.device).get("allocation.all.allocated", 0)
        try:
            with torch.cuda.stream(stream):
                _ck(lib().mspipe_util_graph_begin(stream_ptr(stream)), "util_graph_begin")
                try:
                    fn()
                finally:
                    _ck(lib().mspipe_util_graph_end(stream_ptr(stream), C.byref(self.exec)), "util_graph_end")
        finally:
            _capture_seq += 1  # events recorded inside this capture stay inside it
            if was_enabled:
                gc.enable()
        after = torch.cuda.memory_stats(stream.device).get("allocation.all.allocated", 0)
        if after != before:
            raise RuntimeError(f"StepGraph: {after - before} torch allocations during capture")
        return self

    def replay(self, stream=None):
        _ck(lib().mspipe_util_graph_launch(self.exec, stream_ptr(stream)), "util_graph_launch")

    def __del__(self):
        if getattr(self, "exec", None) and self.exec.value and _lib is not None:
            _lib.mspipe_util_graph_destroy(self.exec)
            self.exec = C.c_void_p()


def sample_recent(g: "TcsrHandle", roots, query_ts, fanout, out, stream=None):
    _ck(lib().mspipe_sample_recent(C.byref(g.c), ptr(roots), ptr(query_ts), roots.numel(), fanout,
                                   ptr(out["nbr"]), ptr(out["eid"]), ptr(out["ts"]), ptr(out["dt"]),
                                   ptr(out["cnt"]), ptr(out.get("sub")), stream_ptr(stream)), "mspipe_sample_recent")
    return out


def sample_batch(g: "TcsrHandle", src, dst, neg, ts, fanout, out, stream=None):
    _ck(lib().mspipe_sample_batch(C.byref(g.c), ptr(src), ptr(dst), ptr(neg), ptr(ts), src.numel(), fanout,
                                  ptr(out["nbr"]), ptr(out["eid"]), ptr(out["ts"]), ptr(out["dt"]),
                                  ptr(out["cnt"]), ptr(out.get("sub")), stream_ptr(stream)), "mspipe_sample_batch")
    return out


def alloc_sample(num_roots, fanout, device, sub=True):
    d = dict(nbr=torch.empty((num_roots, fanout), dtype=torch.int32, device=device),
             eid=torch.empty((num_roots, fanout), dtype=torch.int32, device=device),
             ts=torch.empty((num_roots, fanout), dtype=torch.float64, device=device),
             dt=torch.empty((num_roots, fanout), dtype=torch.float32, device=device),
             cnt=torch.empty((num_roots,), dtype=torch.int32, device=device))
    if sub:
        d["sub"] = torch.empty((num_roots, fanout + 1), dtype=torch.int32, device=device)
    return d


class TcsrHandle:
    """Device-resident T-CSR (caller-owned tensors + the C struct pointing at them)."""

    def __init__(self, num_nodes, indptr, nbr, eid, ts):
        self.indptr, self.nbr, self.eid, self.ts = indptr, nbr, eid, ts
        self.c = Tcsr(int(num_nodes), int(nbr.numel()), ptr(indptr), ptr(nbr), ptr(eid), ptr(ts))


CELL_GRU, CELL_RNN = 0, 1
MAILBOX_IMMEDIATE, MAILBOX_DEFERRED = 0, 1


class GruHandle:
    """Memory updater (mspipe_updater_create): GRU (default) or RNN cell (row F3),
    immediate or deferred mailbox (row F3)."""

    def __init__(self, mem_dim, edge_dim, time_dim, params: dict, device, precision=FP32_3XTF32, max_events=600,
                 stream=None, cell=CELL_GRU, mailbox=MAILBOX_IMMEDIATE):
        self.dims = (mem_dim, edge_dim, time_dim)
        self.cell, self.mailbox = cell, mailbox
        self.w = {k: torch.as_tensor(v, dtype=torch.float32).contiguous().to(device) for k, v in params.items()}
        h = C.c_void_p()
        _ck(lib().mspipe_updater_create(C.byref(h), mem_dim, edge_dim, time_dim, precision, int(cell), int(mailbox),
                                        int(max_events), ptr(self.w["w_ih"]),
                                        ptr(self.w["w_hh"]), ptr(self.w["b_ih"]), ptr(self.w["b_hh"]),
                                        ptr(self.w["time_w"]), ptr(self.w["time_b"]), stream_ptr(stream)),
            "mspipe_updater_create")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.mspipe_gru_destroy(self.h)
            self.h = None


def mail_stride_for(mem_dim, edge_dim):
    Dm = 2 * mem_dim + edge_dim
    return (Dm + 3) // 4 * 4


class MemoryHandle:
    """mspipe_memory over caller-owned (here: this object's) state tables."""

    def __init__(self, num_nodes, mem_dim, edge_dim, staleness_k, device, rank=0, world=1, nccl_id=None,
                 double_buffer=False):
        """world > 1: the tables hold this rank's shard (rows v with v % world == rank);
        nccl_id (bytes) selects the NCCL transport, None the in-process loopback.
        double_buffer: a second table set (mspipe_memory_double_buffer); mem / mem_ts /
        mail / mail_ts always name the set holding the committed version."""
        self.num_nodes, self.mem_dim, self.edge_dim, self.k = num_nodes, mem_dim, edge_dim, staleness_k
        self.rank, self.world = rank, world
        self.mail_stride = mail_stride_for(mem_dim, edge_dim)
        rows = (num_nodes - rank + world - 1) // world

        def tables():
            return dict(mem=torch.zeros((rows, mem_dim), dtype=torch.float32, device=device),
                        mem_ts=torch.zeros((rows,), dtype=torch.float64, device=device),
                        mail=torch.zeros((rows, self.mail_stride), dtype=torch.float32, device=device),
                        mail_ts=torch.zeros((rows,), dtype=torch.float64, device=device))

        self._sets = [tables()]
        t0 = self._sets[0]
        h = C.c_void_p()
        self._nccl_id = None if nccl_id is None else C.create_string_buffer(bytes(nccl_id), len(nccl_id))
        _ck(lib().mspipe_memory_create(C.byref(h), num_nodes, mem_dim, edge_dim, staleness_k, ptr(t0["mem"]),
                                       ptr(t0["mem_ts"]), ptr(t0["mail"]), ptr(t0["mail_ts"]), self.mail_stride,
                                       rank, world, self._nccl_id), "mspipe_memory_create")
        self.h = h
        assert lib().mspipe_memory_local_rows(h) == rows
        self.double_buffer = bool(double_buffer)
        if double_buffer:
            t1 = tables()
            _ck(lib().mspipe_memory_double_buffer(h, ptr(t1["mem"]), ptr(t1["mem_ts"]), ptr(t1["mail"]),
                                                  ptr(t1["mail_ts"])), "mspipe_memory_double_buffer")
            self._sets.append(t1)

    def tables(self, version=None):
        """The table set holding `version` (default: the committed one)."""
        if not self.double_buffer:
            return self._sets[0]
        v = self.committed if version is None else version
        out = C.c_void_p()
        _ck(lib().mspipe_memory_tables(self.h, v, C.byref(out), None, None, None), "mspipe_memory_tables")
        return self._sets[0] if out.value == self._sets[0]["mem"].data_ptr() else self._sets[1]

    mem = property(lambda self: self.tables()["mem"])
    mem_ts = property(lambda self: self.tables()["mem_ts"])
    mail = property(lambda self: self.tables()["mail"])
    mail_ts = property(lambda self: self.tables()["mail_ts"])

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.mspipe_memory_destroy(self.h)
            self.h = None

    @property
    def committed(self):
        return int(lib().mspipe_memory_committed(self.h))

    def set_committed(self, version):
        """After replaying captured steps from a reset (see mspipe_memory_set_committed)."""
        _ck(lib().mspipe_memory_set_committed(self.h, int(version)), "mspipe_memory_set_committed")

    def reset(self, zero_tables=True, stream=None):
        """New epoch: committed := 0; tables back to S_0 = 0 (G17).  The library
        zeroes and mirrors on `stream` (default: the current torch stream), so
        the reset is ordered after the caller's earlier work on it."""
        _ck(lib().mspipe_memory_reset(self.h, 1 if zero_tables else 0, stream_ptr(stream)), "mspipe_memory_reset")


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _ck(lib().mspipe_nccl_unique_id(buf, 128), "mspipe_nccl_unique_id")
    return buf.raw


def memory_writeback_keyed(st: MemoryHandle, commit_version, upd, key_base, stream=None):
    _ck(lib().mspipe_memory_writeback_keyed(st.h, int(commit_version), ptr(upd["nodes"]), ptr(upd["winner"]),
                                            ptr(upd["num"]), upd["nodes"].numel(), int(key_base), ptr(upd["mem"]),
                                            ptr(upd["ts"]), ptr(upd["mail"]), stream_ptr(stream)),
        "mspipe_memory_writeback_keyed")


def shard_fetch_plan(st, iteration, ids, with_mail=False, stream=None):
    _ck(lib().mspipe_shard_fetch_plan(st.h, int(iteration), ptr(ids), ids.numel(), 1 if with_mail else 0,
                                      stream_ptr(stream)), "mspipe_shard_fetch_plan")


def shard_fetch_serve(st, stream=None):
    _ck(lib().mspipe_shard_fetch_serve(st.h, stream_ptr(stream)), "mspipe_shard_fetch_serve")


def shard_fetch_finish(st, ids, out_mem, out_mem_ts, out_mail=None, out_mail_ts=None, stream=None) -> int:
    v = i64(-1)
    _ck(lib().mspipe_shard_fetch_finish(st.h, ptr(ids), ids.numel(), ptr(out_mem), ptr(out_mem_ts), ptr(out_mail),
                                        ptr(out_mail_ts), C.byref(v), stream_ptr(stream)), "mspipe_shard_fetch_finish")
    return int(v.value)


def shard_commit_pack(st, commit_version, upd, key_base, stream=None):
    _ck(lib().mspipe_shard_commit_pack(st.h, int(commit_version), ptr(upd["nodes"]), ptr(upd["winner"]),
                                       ptr(upd["num"]), upd["nodes"].numel(), int(key_base), ptr(upd["mem"]),
                                       ptr(upd["ts"]), ptr(upd["mail"]), stream_ptr(stream)),
        "mspipe_shard_commit_pack")


def shard_commit_merge(st, commit_version, stream=None):
    _ck(lib().mspipe_shard_commit_merge(st.h, int(commit_version), stream_ptr(stream)), "mspipe_shard_commit_merge")


def shard_exchange(st, kind, stream=None):
    _ck(lib().mspipe_shard_exchange(st.h, int(kind), stream_ptr(stream)), "mspipe_shard_exchange")


IPC_HANDLE_BYTES = 64


def shard_window_handle(st) -> bytes:
    """This rank's receive window as a CUDA IPC handle (row E transport)."""
    buf = C.create_string_buffer(IPC_HANDLE_BYTES)
    _ck(lib().mspipe_shard_window_handle(st.h, buf, IPC_HANDLE_BYTES), "mspipe_shard_window_handle")
    return buf.raw


def shard_connect(st, handles):
    """Open every peer's window (handles: one IPC handle per rank, rank order)."""
    blob = b"".join(handles)
    _ck(lib().mspipe_shard_connect(st.h, blob, IPC_HANDLE_BYTES), "mspipe_shard_connect")


def shard_connect_local(handles):
    """Connect in-process ranks (one device): their windows are shared directly."""
    arr = (C.c_void_p * len(handles))(*[h.h.value for h in handles])
    _ck(lib().mspipe_shard_connect_local(arr, len(handles)), "mspipe_shard_connect_local")


def shard_sent_bytes(st):
    """Bytes this rank stored into windows: (fetch ids, reply rows, commit records)."""
    out = (C.c_int64 * 3)()
    _ck(lib().mspipe_shard_sent_bytes(st.h, out), "mspipe_shard_sent_bytes")
    return tuple(int(x) for x in out)


def shard_mitigation_candidates(st, mit, root_mem_ts, root_step, out_ids, stream=None):
    """MSPipe-S at world > 1: the ids whose rows the eligible targets' mitigation reads."""
    _ck(lib().mspipe_shard_mitigation_candidates(st.h, C.byref(mit), ptr(root_mem_ts), int(root_step), ptr(out_ids),
                                                 stream_ptr(stream)), "mspipe_shard_mitigation_candidates")


def shard_fetch_finish_table(st, ids, table_mem, table_mem_ts, stream=None):
    _ck(lib().mspipe_shard_fetch_finish_table(st.h, ptr(ids), ids.numel(), ptr(table_mem), ptr(table_mem_ts),
                                              stream_ptr(stream)), "mspipe_shard_fetch_finish_table")


def shard_mitigate(st, mit, table_mem, table_mem_ts, stream=None):
    _ck(lib().mspipe_shard_mitigate(st.h, C.byref(mit), ptr(table_mem), ptr(table_mem_ts), stream_ptr(stream)),
        "mspipe_shard_mitigate")


def shard_loopback(handles, kind, stream=None):
    arr = (C.c_void_p * len(handles))(*[h.h.value for h in handles])
    _ck(lib().mspipe_shard_loopback(arr, len(handles), int(kind), stream_ptr(stream)), "mspipe_shard_loopback")


def memory_fetch(st: MemoryHandle, iteration, ids, out_mem, out_mem_ts, out_mail=None, out_mail_ts=None,
                 mitigation: Mitigation | None = None, stream=None) -> int:
    v = i64(-1)
    _ck(lib().mspipe_memory_fetch(st.h, int(iteration), ptr(ids), ids.numel(), ptr(out_mem), ptr(out_mem_ts),
                                  ptr(out_mail), ptr(out_mail_ts),
                                  C.byref(mitigation) if mitigation is not None else None, C.byref(v),
                                  stream_ptr(stream)), "mspipe_memory_fetch")
    return int(v.value)


def make_mitigation(g: TcsrHandle, lam, gamma, n_sim, fanout, src, dst, ts, out_h, out_omega=None, out_elig=None):
    m = Mitigation(float(lam), float(gamma), int(n_sim), int(fanout), C.pointer(g.c), ptr(src), ptr(dst), ptr(ts),
                   src.numel(), ptr(out_h), ptr(out_omega), ptr(out_elig))
    m._keep = (g, src, dst, ts, out_h, out_omega, out_elig)
    return m


def memory_dedup(st: MemoryHandle, src, dst, out, stream=None):
    """A2: fills out["nodes"], out["winner"], out["num"] (device U)."""
    _ck(lib().mspipe_memory_dedup(st.h, ptr(src), ptr(dst), src.numel(), ptr(out["nodes"]), ptr(out["winner"]),
                                  ptr(out["num"]), stream_ptr(stream)), "mspipe_memory_dedup")
    return out






def memory_update(st: MemoryHandle, gru: GruHandle, src, dst, ts, edge_feat, snap_mem, snap_mem_ts, snap_step,
                  out, snap_h=None, stream=None):
    """A5+A6: reads out["winner"], out["num"] (from memory_dedup); fills out["mem"], out["ts"], out["mail"]."""
    _ck(lib().mspipe_memory_update(st.h, gru.h, ptr(src), ptr(dst), ptr(ts), src.numel(), ptr(edge_feat),
                                   ptr(snap_mem), ptr(snap_mem_ts), int(snap_step), ptr(snap_h),
                                   ptr(out["winner"]), ptr(out["num"]), ptr(out["mem"]), ptr(out["ts"]),
                                   ptr(out["mail"]), stream_ptr(stream)), "mspipe_memory_update")
    return out


def memory_prep(st: MemoryHandle, g: TcsrHandle, iteration, src, dst, neg, ts, fanout, samp, dd, out_mem, out_mem_ts,
                out_mail=None, out_mail_ts=None, mitigation: Mitigation | None = None, stream=None) -> int:
    """A1+A2+A3(+A4) fused: fills samp (alloc_sample), dd (alloc_dedup) and the fetched rows."""
    v = i64(-1)
    dd = dd if dd is not None else {}  # None: no dedup (A1 + A3 only)
    _ck(lib().mspipe_memory_prep(st.h, C.byref(g.c), int(iteration), ptr(src), ptr(dst), ptr(neg), ptr(ts),
                                 src.numel(), fanout, ptr(samp["nbr"]), ptr(samp["eid"]), ptr(samp["ts"]),
                                 ptr(samp["dt"]), ptr(samp["cnt"]), ptr(samp["sub"]), ptr(dd.get("nodes")),
                                 ptr(dd.get("winner")), ptr(dd.get("num")), ptr(out_mem), ptr(out_mem_ts), ptr(out_mail),
                                 ptr(out_mail_ts), C.byref(mitigation) if mitigation is not None else None,
                                 C.byref(v), stream_ptr(stream)), "mspipe_memory_prep")
    return int(v.value)




def feature_fetch(sub_ids, sampled_eids, fanout, node_feat=None, edge_feat=None, out_node=None, out_edge=None,
                  stream=None):
    """F2: node-feature rows of the subgraph nodes, edge-feature rows of the sampled links."""
    R = (sub_ids if sub_ids is not None else sampled_eids).shape[0]
    _ck(lib().mspipe_feature_fetch(ptr(sub_ids), ptr(sampled_eids), int(R), int(fanout), ptr(node_feat),
                                   node_feat.shape[0] if node_feat is not None else 0,
                                   node_feat.shape[1] if node_feat is not None else 0, ptr(edge_feat),
                                   edge_feat.shape[0] if edge_feat is not None else 0,
                                   edge_feat.shape[1] if edge_feat is not None else 0, ptr(out_node), ptr(out_edge),
                                   stream_ptr(stream)), "mspipe_feature_fetch")


def message_build_deferred(gru: GruHandle, ts, snap_mem, snap_mem_ts, snap_mail, snap_step, winner, num, out_ts,
                           workspace, stream=None):
    """Row F3 A5 (deferred mailbox): operand images from the snapshot mail rows."""
    _ck(lib().mspipe_message_build_deferred(gru.h, ptr(ts), ts.numel(), ptr(snap_mem), ptr(snap_mem_ts),
                                            ptr(snap_mail), snap_mail.shape[1], int(snap_step), ptr(winner), ptr(num),
                                            ptr(out_ts), ptr(workspace), workspace.numel() * workspace.element_size(),
                                            stream_ptr(stream)), "mspipe_message_build_deferred")


def memory_mail_deferred(st: MemoryHandle, commit_version, src, dst, ts, edge_feat, nodes, winner, num, stream=None):
    """Row F3: after a deferred-mailbox commit, mail = [mem[w] | mem[o] | e] from the committed memories."""
    _ck(lib().mspipe_memory_mail_deferred(st.h, int(commit_version), ptr(src), ptr(dst), ptr(ts), ptr(edge_feat),
                                          src.numel(), ptr(nodes), ptr(winner), ptr(num), stream_ptr(stream)),
        "mspipe_memory_mail_deferred")


def gru_workspace_size(gru: GruHandle, num_events) -> int:
    return int(lib().mspipe_gru_workspace_size(gru.h, int(num_events)))


def message_build(gru: GruHandle, ts, edge_feat, snap_mem, snap_mem_ts, snap_step, winner, num, out_ts, out_mail,
                  workspace, snap_h=None, stream=None):
    """A5: message + time encoding -> tensor-core operand images (workspace), mail rows, commit ts."""
    _ck(lib().mspipe_message_build(gru.h, ptr(ts), ts.numel(), ptr(edge_feat), ptr(snap_mem), ptr(snap_mem_ts),
                                   int(snap_step), ptr(snap_h), ptr(winner), ptr(num), ptr(out_ts), ptr(out_mail),
                                   out_mail.shape[1], ptr(workspace), workspace.numel() * workspace.element_size(),
                                   stream_ptr(stream)), "mspipe_message_build")


def gru_apply(gru: GruHandle, num_events, snap_mem, snap_step, winner, num, out_mem, workspace, snap_h=None,
              stream=None):
    """A6: the GRU contraction + gates from the operand images of message_build."""
    _ck(lib().mspipe_gru_apply(gru.h, int(num_events), ptr(snap_mem), int(snap_step), ptr(snap_h), ptr(winner),
                               ptr(num), ptr(out_mem), ptr(workspace), workspace.numel() * workspace.element_size(),
                               stream_ptr(stream)), "mspipe_gru_apply")


def gru_apply_commit(gru: GruHandle, st: MemoryHandle, commit_version, num_events, snap_mem, snap_step, upd,
                     workspace, snap_h=None, stream=None, out_nodes=None, out_num=None):
    """A6+A7 in one launch: reads upd[nodes, winner, num, ts, mail] (dedup + message_build), writes the
    state rows of version commit_version and upd["mem"] (h' in winner order); with out_nodes / out_num
    (mspipe_gru_apply_commit_out) also the result record's winner ids and U."""
    if out_nodes is not None or out_num is not None:
        _ck(lib().mspipe_gru_apply_commit_out(gru.h, st.h, int(commit_version), int(num_events), ptr(snap_mem),
                                              int(snap_step), ptr(snap_h), ptr(upd["nodes"]), ptr(upd["winner"]),
                                              ptr(upd["num"]), ptr(upd["ts"]), ptr(upd.get("mail")),
                                              ptr(upd.get("mem")), ptr(out_nodes), ptr(out_num), ptr(workspace),
                                              workspace.numel() * workspace.element_size(), stream_ptr(stream)),
            "mspipe_gru_apply_commit_out")
        return
    _ck(lib().mspipe_gru_apply_commit(gru.h, st.h, int(commit_version), int(num_events), ptr(snap_mem),
                                      int(snap_step), ptr(snap_h), ptr(upd["nodes"]), ptr(upd["winner"]),
                                      ptr(upd["num"]), ptr(upd["ts"]), ptr(upd.get("mail")), ptr(upd.get("mem")),
                                      ptr(workspace), workspace.numel() * workspace.element_size(),
                                      stream_ptr(stream)), "mspipe_gru_apply_commit")




def alloc_dedup(num_events, device):
    n = 2 * num_events
    return dict(nodes=torch.empty((n,), dtype=torch.int32, device=device),
                winner=torch.empty((n,), dtype=torch.int32, device=device),
                num=torch.zeros((1,), dtype=torch.int32, device=device))


def alloc_update(num_events, mem_dim, mail_stride, device):
    """Dedup outputs + GRU outputs in one dict (the layout memory_writeback reads)."""
    n = 2 * num_events
    return dict(**alloc_dedup(num_events, device),
                mem=torch.empty((n, mem_dim), dtype=torch.float32, device=device),
                ts=torch.empty((n,), dtype=torch.float64, device=device),
                mail=torch.empty((n, mail_stride), dtype=torch.float32, device=device))


def memory_writeback(st: MemoryHandle, commit_version, upd, stream=None):
    _ck(lib().mspipe_memory_writeback(st.h, int(commit_version), ptr(upd["nodes"]), ptr(upd["num"]),
                                      upd["nodes"].numel(), ptr(upd["mem"]), ptr(upd["ts"]), ptr(upd["mail"]),
                                      stream_ptr(stream)), "mspipe_memory_writeback")


# ---------------------------------------------------------------- row F4
TRAIN_TENSORS = ("w_q", "w_k", "w_v", "w_o", "b_o", "w_1", "b_1", "w_2", "b_2", "w_ih", "w_hh", "b_ih", "b_hh")


def train_layout(mem_dim, edge_dim, time_dim, emb_dim):
    """(total floats, {tensor: offset}) of the flat parameter / gradient buffer."""
    off = (i64 * 13)()
    n = lib().mspipe_train_layout(int(mem_dim), int(edge_dim), int(time_dim), int(emb_dim), off)
    if n < 0:
        raise MspipeError(EINVAL, "mspipe_train_layout", "bad dimensions")
    return int(n), dict(zip(TRAIN_TENSORS, (int(o) for o in off)))


class TrainHandle:
    """mspipe_train over caller-owned (here: this object's) flat params / grads."""

    def __init__(self, gru: GruHandle, num_nodes, emb_dim, fanout, max_events, params: torch.Tensor,
                 grads: torch.Tensor, stream=None):
        if not (params.is_cuda and grads.is_cuda and params.dtype == torch.float32 and grads.dtype == torch.float32):
            raise ValueError("params / grads: CUDA float32 tensors")
        self.params, self.grads = params, grads
        h = C.c_void_p()
        _ck(lib().mspipe_train_create(C.byref(h), gru.h, int(num_nodes), int(emb_dim), int(fanout), int(max_events),
                                      ptr(params), ptr(grads), stream_ptr(stream)), "mspipe_train_create")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.mspipe_train_destroy(self.h)
            self.h = None


def gru_save_gates(gru: GruHandle, gates):
    _ck(lib().mspipe_gru_save_gates(gru.h, ptr(gates)), "mspipe_gru_save_gates")


def train_step(tr: TrainHandle, gru: GruHandle, num_events, samp, snap_mem, nodes, num, new_mem, workspace, gates,
               out_loss, out_logits=None, stream=None):
    _ck(lib().mspipe_train_step(tr.h, gru.h, int(num_events), ptr(samp["sub"]), ptr(samp["dt"]), ptr(samp["cnt"]),
                                ptr(snap_mem), ptr(nodes), ptr(num), ptr(new_mem), ptr(workspace),
                                workspace.numel() * workspace.element_size(), ptr(gates), ptr(out_loss),
                                ptr(out_logits), stream_ptr(stream)), "mspipe_train_step")


def train_sgd(tr: TrainHandle, gru: GruHandle, lr, stream=None):
    _ck(lib().mspipe_train_sgd(tr.h, gru.h, float(lr), stream_ptr(stream)), "mspipe_train_sgd")


# ---------------------------------------------------------------- row F3, APAN
class ApanHandle:
    """mspipe_apan over this object's mailbox tables (ring of `slots` mails per node)."""

    def __init__(self, num_nodes, mem_dim, edge_dim, slots, max_events, w_q, w_k, device, stream=None):
        Dm = 2 * mem_dim + edge_dim
        self.slots = slots
        self.mb = torch.zeros((num_nodes, slots, Dm), dtype=torch.float32, device=device)
        self.mb_ts = torch.zeros((num_nodes, slots), dtype=torch.float64, device=device)
        self.mb_pos = torch.zeros((num_nodes,), dtype=torch.int32, device=device)
        self.mb_cnt = torch.zeros((num_nodes,), dtype=torch.int32, device=device)
        wq = torch.as_tensor(w_q, dtype=torch.float32).contiguous().to(device)
        wk = torch.as_tensor(w_k, dtype=torch.float32).contiguous().to(device)
        h = C.c_void_p()
        _ck(lib().mspipe_apan_create(C.byref(h), int(num_nodes), int(mem_dim), int(edge_dim), int(slots),
                                     int(max_events), ptr(wq), ptr(wk), ptr(self.mb), ptr(self.mb_ts),
                                     ptr(self.mb_pos), ptr(self.mb_cnt), stream_ptr(stream)), "mspipe_apan_create")
        self.h = h

    def reset(self):
        for t in (self.mb, self.mb_ts, self.mb_pos, self.mb_cnt):
            t.zero_()
        self.refresh_keys()

    def refresh_keys(self, stream=None):
        """Recompute the cached keys after writing the mailbox tables directly."""
        _ck(lib().mspipe_apan_refresh_keys(self.h, stream_ptr(stream)), "mspipe_apan_refresh_keys")

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.mspipe_apan_destroy(self.h)
            self.h = None


def message_build_apan(ap: ApanHandle, gru: GruHandle, ts, snap_mem, snap_mem_ts, snap_step, nodes, winner, num,
                       out_ts, workspace, stream=None):
    _ck(lib().mspipe_message_build_apan(ap.h, gru.h, ptr(ts), ts.numel(), ptr(snap_mem), ptr(snap_mem_ts),
                                        int(snap_step), ptr(nodes), ptr(winner), ptr(num), ptr(out_ts),
                                        ptr(workspace), workspace.numel() * workspace.element_size(),
                                        stream_ptr(stream)), "mspipe_message_build_apan")


def apan_deliver(ap: ApanHandle, st: MemoryHandle, commit_version, src, dst, ts, ef, nodes, winner, num, nbr, cnt,
                 fanout, stream=None):
    _ck(lib().mspipe_apan_deliver(ap.h, st.h, int(commit_version), ptr(src), ptr(dst), ptr(ts), ptr(ef), src.numel(),
                                  ptr(nodes), ptr(winner), ptr(num), ptr(nbr), ptr(cnt), int(fanout),
                                  stream_ptr(stream)), "mspipe_apan_deliver")

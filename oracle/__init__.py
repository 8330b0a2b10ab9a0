"""ctypes wrapper of the plain CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package
paper_2402_15113_b200/.  Shares no code with the CUDA path.

Every function cites the passage it follows (see oracle.c for the full text).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P = C.c_void_p
        i32, i64, f32, f64 = C.c_int32, C.c_int64, C.c_float, C.c_double
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_get_threads.restype = C.c_int
        L.orc_sample_brute.argtypes = [i64, P, P, P, i64, P, P, i32, P, P, P, P, P]
        L.orc_graph_create.argtypes = [i64, i64, P, P, P]
        L.orc_graph_create.restype = P
        L.orc_graph_free.argtypes = [P]
        L.orc_sample.argtypes = [P, i64, P, P, i32, P, P, P, P, P]
        L.orc_dedup.argtypes = [i64, i64, P, P, P, P]
        L.orc_dedup.restype = i64
        L.orc_mitigate.argtypes = [P, i64, P, P, P, P, i32, f32, f64, i32, i32, P, P, P]
        L.orc_memory_update.argtypes = [i64, i64, P, P, P, P, i32, i32, i32, P, P, P, P, P, P,
                                        P, P, i32, P, f32, f64, i32, i32, P, P, P, P, P, P, P, P, P, i32]
        L.orc_memory_update.restype = i64
        L.orc_snapshot_version.argtypes = [i64, i32, i32]
        L.orc_snapshot_version.restype = i64
        L.orc_run_stream.argtypes = [i64, i64, P, P, P, P, i32, i32, i32, P, P, P, P, P, P, i64,
                                     i32, i32, i32, f32, f64, i32, i32, P, P, P, P, i64, P, P, i32, P, i32]
        L.orc_run_stream.restype = i64
        L.orc_run_stream_ex.argtypes = L.orc_run_stream.argtypes + [P]
        L.orc_run_stream_ex.restype = i64
        L.orc_staleness_error_series.argtypes = [i64, i64, P, P, P, P, i32, i32, i32, P, P, P, P, P, P, i64,
                                                 i32, i32, i32, f32, f64, i32, i32, i64, P]
        L.orc_staleness_error_series.restype = i64
        L.orc_delta_t_population.argtypes = [i64, i64, P, P, P, P]
        L.orc_delta_t_population.restype = i64
        L.orc_quantile_nearest_rank.argtypes = [i64, P, f64]
        L.orc_quantile_nearest_rank.restype = f64
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def get_threads() -> int:
    return int(lib().orc_get_threads())


def _alloc_sample(n, fanout):
    return (np.empty((n, fanout), np.int32), np.empty((n, fanout), np.int32),
            np.empty((n, fanout), np.float64), np.empty((n, fanout), np.float32),
            np.empty(n, np.int32))


def sample_brute(src, dst, ts, roots, qts, fanout):
    """A1 definition: backward scan of the whole log."""
    src, dst, ts = _c(src, np.int32), _c(dst, np.int32), _c(ts, np.float64)
    roots, qts = _c(roots, np.int32), _c(qts, np.float64)
    out = _alloc_sample(len(roots), fanout)
    rc = lib().orc_sample_brute(len(src), _p(src), _p(dst), _p(ts), len(roots), _p(roots),
                                _p(qts), fanout, *map(_p, out))
    if rc != 0:
        raise ValueError(f"orc_sample_brute rc={rc}")
    return dict(zip(("nbr", "eid", "ts", "dt", "cnt"), out))


class Graph:
    """The oracle's own per-node incident-event lists (stream order)."""

    def __init__(self, num_nodes, src, dst, ts):
        self.src, self.dst, self.ts = _c(src, np.int32), _c(dst, np.int32), _c(ts, np.float64)
        self.num_nodes = int(num_nodes)
        self.h = lib().orc_graph_create(self.num_nodes, len(self.src), _p(self.src),
                                        _p(self.dst), _p(self.ts))

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_graph_free(self.h)
            self.h = None

    def sample(self, roots, qts, fanout):
        roots, qts = _c(roots, np.int32), _c(qts, np.float64)
        out = _alloc_sample(len(roots), fanout)
        rc = lib().orc_sample(self.h, len(roots), _p(roots), _p(qts), fanout, *map(_p, out))
        if rc != 0:
            raise ValueError(f"orc_sample rc={rc}")
        return dict(zip(("nbr", "eid", "ts", "dt", "cnt"), out))

    def mitigate(self, ids, tstar, mem, mem_ts, lam, gamma, n_sim, fanout):
        """A4 for explicit targets against snapshot tables."""
        ids, tstar = _c(ids, np.int32), _c(tstar, np.float64)
        mem, mem_ts = _c(mem, np.float32), _c(mem_ts, np.float64)
        n, M = len(ids), mem.shape[1]
        h = np.empty((n, M), np.float32)
        om = np.empty((n, n_sim), np.int32)
        el = np.empty(n, np.uint8)
        rc = lib().orc_mitigate(self.h, n, _p(ids), _p(tstar), _p(mem), _p(mem_ts), M, lam,
                                gamma, n_sim, fanout, _p(h), _p(om), _p(el))
        if rc != 0:
            raise ValueError(f"orc_mitigate rc={rc}")
        return dict(h=h, omega=om, elig=el.astype(bool))


def dedup(num_nodes, src, dst):
    """A2: winners = last pair index per node."""
    src, dst = _c(src, np.int32), _c(dst, np.int32)
    nodes = np.empty(2 * len(src), np.int32)
    win = np.empty(2 * len(src), np.int32)
    U = lib().orc_dedup(num_nodes, len(src), _p(src), _p(dst), _p(nodes), _p(win))
    return nodes[:U].copy(), win[:U].copy()


def memory_update(num_nodes, src, dst, ts, ef, params, mem, mem_ts, mitigation=None,
                  graph: Graph | None = None, fanout=10, mail=None, mailbox="immediate", cell="gru"):
    """Teacher-forced A2+A4+A5+A6 for one batch against snapshot tables.  Row F3:
    mailbox="deferred" reads the snapshot `mail` [N, Dm]; cell="rnn" takes
    RNNCell weights (w_ih [M, Dx], w_hh [M, M], b_ih / b_hh [M])."""
    src, dst, ts = _c(src, np.int32), _c(dst, np.int32), _c(ts, np.float64)
    ef = _c(ef, np.float32)
    mem, mem_ts = _c(mem, np.float32), _c(mem_ts, np.float64)
    B, He = len(src), ef.shape[1]
    M = mem.shape[1]
    Dt = len(params["time_w"])
    Dm = 2 * M + He
    pr = {k: _c(v, np.float32) for k, v in params.items()}
    n_sim = mitigation["n_sim"] if mitigation else 5
    nodes = np.empty(2 * B, np.int32)
    win = np.empty(2 * B, np.int32)
    omem = np.empty((2 * B, M), np.float32)
    ots = np.empty(2 * B, np.float64)
    omail = np.empty((2 * B, Dm), np.float32)
    oh = np.empty((2 * B, M), np.float32)
    oom = np.empty((2 * B, n_sim), np.int32)
    oel = np.empty(2 * B, np.uint8)
    if mitigation and graph is None:
        raise ValueError("mitigation needs the graph")
    U = lib().orc_memory_update(
        num_nodes, B, _p(src), _p(dst), _p(ts), _p(ef), M, He, Dt, _p(pr["w_ih"]), _p(pr["w_hh"]),
        _p(pr["b_ih"]), _p(pr["b_hh"]), _p(pr["time_w"]), _p(pr["time_b"]), _p(mem), _p(mem_ts),
        1 if mitigation else 0, graph.h if graph is not None else None,
        float(mitigation["lam"]) if mitigation else 1.0,
        float(mitigation["gamma"]) if mitigation else 0.0, n_sim, fanout, _p(nodes), _p(win),
        _p(omem), _p(ots), _p(omail), _p(oh), _p(oom), _p(oel),
        _p(_c(mail, np.float32)) if mail is not None else None, _variant(mailbox, cell))
    if U < 0:
        raise ValueError(f"orc_memory_update rc={U}")
    return dict(nodes=nodes[:U], winner=win[:U], mem=omem[:U], ts=ots[:U], mail=omail[:U],
                h=oh[:U], omega=oom[:U], elig=oel[:U].astype(bool))


def _variant(mailbox, cell):
    """Row F3 updater variants: bit 0 deferred mailbox (TGL TGN), bit 1 RNN cell (JODIE)."""
    if mailbox not in ("immediate", "deferred") or cell not in ("gru", "rnn"):
        raise ValueError(f"mailbox={mailbox} cell={cell}")
    return (1 if mailbox == "deferred" else 0) | (2 if cell == "rnn" else 0)


def snapshot_version(i, k, schedule="exact"):
    """A3 (G8): exact v=max(0,i-1-k); grouped v=(k+1)floor((i-1)/(k+1))."""
    return int(lib().orc_snapshot_version(int(i), int(k), 1 if schedule == "grouped" else 0))


def new_state(num_nodes, mem_dim, edge_dim):
    """S_0: zeros (C.1; G17)."""
    Dm = 2 * mem_dim + edge_dim
    return dict(mem=np.zeros((num_nodes, mem_dim), np.float32), mem_ts=np.zeros(num_nodes),
                mail=np.zeros((num_nodes, Dm), np.float32), mail_ts=np.zeros(num_nodes))


class _Dump(C.Structure):
    _fields_ = [("n", C.c_int64), ("batches", C.c_void_p), ("sub_ids", C.c_void_p), ("mem", C.c_void_p),
                ("mem_ts", C.c_void_p)]


def run_stream(num_nodes, src, dst, ts, ef, params, batch, k, schedule="exact", mitigation=None,
               fanout=10, state=None, max_batches=-1, neg=None, plan=None, mailbox="immediate", cell="gru",
               dump_batches=None):
    """C.2 O1-O8 over the stream; returns (final state, per-batch versions).
    With `neg`, every batch also runs A1 on its 3B roots and gathers the
    snapshot rows of the subgraph (the whole per-batch path, for timing).
    plan (row F1): per-iteration paper staleness k_i (v(i) = max(0, i - k_i));
    k must then be >= max_i (i - v(i)) - 1 (copies kept).
    dump_batches (needs neg): 1-based iterations whose A3s output (subgraph ids
    [3B, fanout+1], rows of S_{v(i)} and their mem_ts) is returned as a third
    value {"batches", "sub_ids", "mem", "mem_ts"}."""
    planc = None if plan is None else _c(plan, np.int32)
    negc = None if neg is None else _c(neg, np.int32)
    src, dst, ts = _c(src, np.int32), _c(dst, np.int32), _c(ts, np.float64)
    ef = _c(ef, np.float32)
    He = ef.shape[1]
    pr = {kk: _c(v, np.float32) for kk, v in params.items()}
    M = pr["w_hh"].shape[1]
    Dt = len(pr["time_w"])
    st = new_state(num_nodes, M, He) if state is None else {kk: v.copy() for kk, v in state.items()}
    E = len(src)
    nb = -(-E // batch)
    if max_batches >= 0:
        nb = min(nb, max_batches)
    vers = np.zeros(max(nb, 1), np.int64)
    mit = mitigation
    dump, dres = None, None
    if dump_batches is not None:
        if negc is None:
            raise ValueError("dump_batches needs neg (the subgraph roots)")
        db = np.ascontiguousarray(np.sort(np.asarray(dump_batches, np.int64)))
        slots = 3 * batch * (fanout + 1)
        dres = dict(batches=db, sub_ids=np.full((len(db), slots), -2, np.int32),
                    mem=np.zeros((len(db), slots, M), np.float32), mem_ts=np.zeros((len(db), slots)))
        dump = _Dump(len(db), db.ctypes.data, dres["sub_ids"].ctypes.data, dres["mem"].ctypes.data,
                     dres["mem_ts"].ctypes.data)
    r = lib().orc_run_stream_ex(
        num_nodes, E, _p(src), _p(dst), _p(ts), _p(ef), M, He, Dt, _p(pr["w_ih"]),
        _p(pr["w_hh"]), _p(pr["b_ih"]), _p(pr["b_hh"]), _p(pr["time_w"]), _p(pr["time_b"]), batch,
        k, 1 if schedule == "grouped" else 0, 1 if mit else 0, float(mit["lam"]) if mit else 1.0,
        float(mit["gamma"]) if mit else 0.0, int(mit["n_sim"]) if mit else 5, fanout,
        _p(st["mem"]), _p(st["mem_ts"]), _p(st["mail"]), _p(st["mail_ts"]), max_batches, _p(vers),
        _p(negc), 0 if negc is None else 1, _p(planc), _variant(mailbox, cell),
        C.byref(dump) if dump is not None else None)
    if r < 0:
        raise ValueError(f"orc_run_stream rc={r}")
    if dres is not None:
        return st, vers[:r], dres
    return st, vers[:r]


def staleness_error_series(num_nodes, src, dst, ts, ef, params, batch, k, schedule="exact", mitigation=None,
                           fanout=10, max_batches=-1):
    """Row F1 analytics: per iteration, ‖x − s‖_F over
    the batch's update targets, x = the stale run's GRU hidden input (stale read,
    or MSPipe-S's mitigated row), s = a k = 0 run's S_{i-1} (reading F7)."""
    src, dst, ts = _c(src, np.int32), _c(dst, np.int32), _c(ts, np.float64)
    ef = _c(ef, np.float32)
    pr = {kk: _c(v, np.float32) for kk, v in params.items()}
    M, He, Dt = pr["w_hh"].shape[1], ef.shape[1], len(pr["time_w"])
    nb = -(-len(src) // batch)
    if max_batches >= 0:
        nb = min(nb, max_batches)
    out = np.zeros(max(nb, 1), np.float64)
    mit = mitigation
    r = lib().orc_staleness_error_series(
        num_nodes, len(src), _p(src), _p(dst), _p(ts), _p(ef), M, He, Dt, _p(pr["w_ih"]), _p(pr["w_hh"]),
        _p(pr["b_ih"]), _p(pr["b_hh"]), _p(pr["time_w"]), _p(pr["time_b"]), batch, k,
        1 if schedule == "grouped" else 0, 1 if mit else 0, float(mit["lam"]) if mit else 1.0,
        float(mit["gamma"]) if mit else 0.0, int(mit["n_sim"]) if mit else 5, fanout, max_batches, _p(out))
    if r < 0:
        raise ValueError(f"orc_staleness_error_series rc={r}")
    return out[:r]


def delta_t_population(num_nodes, src, dst, ts):
    """G16: gaps to each endpoint's previous event (first appearances excluded)."""
    src, dst, ts = _c(src, np.int32), _c(dst, np.int32), _c(ts, np.float64)
    out = np.empty(2 * len(src), np.float64)
    n = lib().orc_delta_t_population(num_nodes, len(src), _p(src), _p(dst), _p(ts), _p(out))
    return out[:n].copy()


def quantile_nearest_rank(values, p):
    """Nearest-rank quantile."""
    v = _c(values, np.float64)
    return float(lib().orc_quantile_nearest_rank(len(v), _p(v), float(p)))


def gamma(num_nodes, src, dst, ts, p=0.99):
    """γ = p-quantile of the Δt population (G16)."""
    return quantile_nearest_rank(delta_t_population(num_nodes, src, dst, ts), p)


def memory_overhead_bound(K, B, fanout, Hn, He, M):
    """Extra GPU memory of K prefetched subgraphs, bytes:
    12 K B (𝒩+1) (H_n + 2/3 H_e + M + 5/3)."""
    return 12.0 * K * B * (fanout + 1) * (Hn + 2.0 / 3.0 * He + M + 5.0 / 3.0)

"""Seeded synthetic event streams shaped like the paper's datasets.

Shapes pinned by the paper: |V|, |E|, edge-feature dim d_e (Table
``tab:datasets``), mean inter-event gaps (PAPER.md L876:
LastFM 106, Reddit 4, Wiki 17, MOOC 3.6, GDELT 0.1), and a power-law Δt
(Fig. ``fig:wiki``).  The user/item splits, Zipf
exponents and repeat probabilities are our proposals and
are flagged as such in DESIGN.md.

Nothing here implements any step of the method: this module only draws
inputs.  Random numbers are drawn from ``numpy.random.default_rng`` keyed by
(seed, stream-id), or — for edge features, which must also be reproducible on
the device for the GDELT-sized stream — from a counter-based splitmix64 hash
keyed by (seed, eid, column) that gives bit-identical f32 values anywhere.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass(frozen=True)
class WorkloadConfig:
    name: str
    num_nodes: int
    num_users: int          # 0 => unipartite
    num_events: int
    edge_dim: int           # d_e / He
    batch: int              # local batch size B
    staleness_k: int        # build k = paper k - 1
    mitigation: bool
    mean_gap: float
    ts_mode: str            # "exp_floor" | "gdelt"
    zipf_src: float
    zipf_dst: float
    repeat: float
    mem_dim: int = 100      # PAPER.md L412 "memory dimensions of 100"
    node_dim: int = 0       # |d_v| (Table `tab:datasets`): 413 for GDELT, else 0
    time_dim: int = 100     # reading G3
    fanout: int = 10        # PAPER.md L412 "10 most recent 1-hop neighbors"
    lam: float = 0.95       # PAPER.md L410 "lambda set to 0.95"
    quantile_p: float = 0.99  # PAPER.md L317 "99% quantile"
    n_sim: int = 5          # reading G10

    @property
    def mail_dim(self) -> int:
        return 2 * self.mem_dim + self.edge_dim

    @property
    def gru_in_dim(self) -> int:
        return self.mail_dim + self.time_dim


# Table tab:datasets + mean gaps; splits /
# Zipf / repeat are our proposals.
CONFIGS = {
    "tiny": WorkloadConfig("tiny", 1000, 0, 10_000, 172, 200, 0, False, 1.0, "exp_floor", 0.0, 0.0, 0.0),
    "wiki": WorkloadConfig("wiki", 9227, 8227, 157_474, 172, 600, 1, False, 17.0, "exp_floor", 1.1, 1.0, 0.7),
    "reddit": WorkloadConfig("reddit", 10_984, 10_000, 672_447, 172, 600, 2, True, 4.0, "exp_floor", 1.0, 1.1, 0.6),
    "lastfm": WorkloadConfig("lastfm", 1980, 980, 1_293_103, 128, 600, 2, False, 106.0, "exp_floor", 0.6, 1.1, 0.5),
    "mooc": WorkloadConfig("mooc", 7144, 7047, 411_749, 128, 600, 2, False, 3.6, "exp_floor", 0.9, 1.2, 0.5),
    "gdelt": WorkloadConfig("gdelt", 16_682, 0, 191_290_882, 186, 4000, 3, False, 0.1, "gdelt", 1.2, 1.2, 0.3,
                            node_dim=413),
}


def _rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.default_rng([int(seed), int(stream)])


def _zipf_ids(rng: np.random.Generator, n: int, s: float, size: int) -> np.ndarray:
    """Draw `size` ids in [0, n) with P(rank r) ∝ (r+1)^-s, ranks randomly permuted."""
    if s == 0.0:
        return rng.integers(0, n, size=size, dtype=np.int64)
    w = np.arange(1, n + 1, dtype=np.float64) ** (-s)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    perm = rng.permutation(n)
    r = np.searchsorted(cdf, rng.random(size), side="right")
    np.minimum(r, n - 1, out=r)
    return perm[r]


def _repeat_fill(key: np.ndarray, fresh: np.ndarray, repeat_mask: np.ndarray) -> np.ndarray:
    """Within each group of equal `key` (in stream order), a position whose
    repeat_mask is set copies the value of the previous position of that
    group; the first position of a group is always fresh."""
    # the stable order is unique; a 16-bit key takes numpy's radix sort (GDELT: ~5x faster)
    small = key.size and 0 <= key.min() and key.max() < 32768
    order = np.argsort(key.astype(np.int16) if small else key, kind="stable")
    k_sorted = key[order]
    first = np.ones(len(order), dtype=bool)
    first[1:] = k_sorted[1:] != k_sorted[:-1]
    take_fresh = first | ~repeat_mask[order]
    pos = np.where(take_fresh, np.arange(len(order)), -1)
    np.maximum.accumulate(pos, out=pos)
    out = np.empty_like(fresh)
    out[order] = fresh[order][pos]
    return out


def make_events(cfg: WorkloadConfig, seed: int = 0, num_events: int | None = None):
    """Return src, dst (int32), ts (float64, non-decreasing), neg (int32).

    `num_events` takes a prefix-sized stream of the same shape (used by tests
    and by the bounded CPU-baseline sample)."""
    E = cfg.num_events if num_events is None else int(num_events)
    N = cfg.num_nodes
    rs = _rng(seed, 1)
    if cfg.num_users > 0:
        nu, ni = cfg.num_users, N - cfg.num_users
        u = _zipf_ids(rs, nu, cfg.zipf_src, E)
        fresh_i = _zipf_ids(_rng(seed, 2), ni, cfg.zipf_dst, E) + nu
        rep = _rng(seed, 3).random(E) < cfg.repeat
        it = _repeat_fill(u, fresh_i, rep) if cfg.repeat > 0 else fresh_i
        src, dst = u, it
    else:
        src = _zipf_ids(rs, N, cfg.zipf_src, E)
        fresh_d = _zipf_ids(_rng(seed, 2), N, cfg.zipf_dst, E)
        if cfg.repeat > 0:
            rep = _rng(seed, 3).random(E) < cfg.repeat
            dst = _repeat_fill(src, fresh_d, rep)
        else:
            dst = fresh_d
    if cfg.ts_mode == "gdelt":
        # "records global events ... every 15 minutes": 15-unit
        # ticks with 150-way ties, mean gap 0.1.
        ts = 15.0 * np.floor(np.arange(E, dtype=np.float64) / 150.0)
    else:
        gaps = _rng(seed, 4).exponential(cfg.mean_gap, size=E)
        ts = np.floor(np.cumsum(gaps))
    neg = _rng(seed, 5).integers(0, N, size=E, dtype=np.int64)
    return (src.astype(np.int32), dst.astype(np.int32), ts.astype(np.float64), neg.astype(np.int32))


_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64, copy=True)
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return z


def edge_features(seed: int, eid0: int, n: int, edge_dim: int) -> np.ndarray:
    """f32 [n, edge_dim] edge features for eids eid0..eid0+n-1.

    Counter-based: value(eid, c) = (top24(splitmix64(seed*φ + eid*He + c + 1)) - 2^23) / 2^23,
    uniform on [-1, 1) and exactly representable in f32, so a device-side
    generator following the same integer recipe yields identical bytes."""
    with np.errstate(over="ignore"):
        base = np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15)
        ctr = (np.arange(eid0, eid0 + n, dtype=np.uint64)[:, None] * np.uint64(edge_dim)
               + np.arange(edge_dim, dtype=np.uint64)[None, :] + np.uint64(1) + base)
    z = _splitmix64(ctr)
    top = (z >> np.uint64(40)).astype(np.int64) - (1 << 23)
    return (top.astype(np.float32) * np.float32(2.0 ** -23)).astype(np.float32)


def node_features(seed: int, num_nodes: int, node_dim: int) -> np.ndarray:
    """f32 [num_nodes, node_dim] node features, the edge-feature recipe on a
    separate counter stream (key seed ^ 0x5EED, so node and edge values differ)."""
    if node_dim == 0:
        return np.zeros((num_nodes, 0), np.float32)
    return edge_features(seed ^ 0x5EED, 0, num_nodes, node_dim)


def rnn_params(mem_dim: int, mail_dim: int, time_dim: int, seed: int = 1234):
    """RNNCell-shaped weights (row F3, JODIE's updater), U(-1/sqrt(M), 1/sqrt(M)) like
    torch.nn.RNNCell; the same time encoder as gru_params.  All f32."""
    rng = _rng(seed, 8)
    Dx = mail_dim + time_dim
    a = 1.0 / math.sqrt(mem_dim)
    p = dict(w_ih=rng.uniform(-a, a, size=(mem_dim, Dx)).astype(np.float32),
             w_hh=rng.uniform(-a, a, size=(mem_dim, mem_dim)).astype(np.float32),
             b_ih=rng.uniform(-a, a, size=(mem_dim,)).astype(np.float32),
             b_hh=rng.uniform(-a, a, size=(mem_dim,)).astype(np.float32))
    g = gru_params(mem_dim, mail_dim, time_dim, seed)
    p.update(time_w=g["time_w"], time_b=g["time_b"])
    return p


def gru_params(mem_dim: int, mail_dim: int, time_dim: int, seed: int = 1234):
    """GRUCell-shaped weights, U(-1/sqrt(M), 1/sqrt(M)) like torch.nn.GRUCell's
    default init, gate order (r, z, n); time encoder ω_q = 10^(-9q/(d_t-1)), φ = 0
    (reading G2).  All f32."""
    rng = _rng(seed, 7)
    Dx = mail_dim + time_dim
    a = 1.0 / math.sqrt(mem_dim)
    w_ih = rng.uniform(-a, a, size=(3 * mem_dim, Dx)).astype(np.float32)
    w_hh = rng.uniform(-a, a, size=(3 * mem_dim, mem_dim)).astype(np.float32)
    b_ih = rng.uniform(-a, a, size=(3 * mem_dim,)).astype(np.float32)
    b_hh = rng.uniform(-a, a, size=(3 * mem_dim,)).astype(np.float32)
    q = np.arange(time_dim, dtype=np.float64)
    time_w = (10.0 ** (-9.0 * q / max(time_dim - 1, 1))).astype(np.float32)
    time_b = np.zeros(time_dim, dtype=np.float32)
    return dict(w_ih=w_ih, w_hh=w_hh, b_ih=b_ih, b_hh=b_hh, time_w=time_w, time_b=time_b)


def train_params(mem_dim: int, time_dim: int, emb_dim: int = 100, seed: int = 4321):
    """Row F4 weights (embedding attention + link decoder), U(-1/sqrt(fan_in),
    1/sqrt(fan_in)) like torch.nn.Linear's default init.  Shapes (reading T3/T4
    in DESIGN.md): w_q [H, M], w_k / w_v [H, M + d_t], w_o [H, H + M], b_o [H],
    w_1 [H, 2H], b_1 [H], w_2 [H], b_2 [1].  All f32."""
    rng = _rng(seed, 9)
    H, M, Dt = emb_dim, mem_dim, time_dim

    def u(shape, fan_in):
        a = 1.0 / math.sqrt(fan_in)
        return rng.uniform(-a, a, size=shape).astype(np.float32)

    return dict(w_q=u((H, M), M), w_k=u((H, M + Dt), M + Dt), w_v=u((H, M + Dt), M + Dt),
                w_o=u((H, H + M), H + M), b_o=u((H,), H + M), w_1=u((H, 2 * H), 2 * H), b_1=u((H,), 2 * H),
                w_2=u((H,), H), b_2=u((1,), H))


def make_workload(name: str, seed: int = 0, num_events: int | None = None, with_features: bool = True,
                  tcsr_events: int | None = None):
    """The first `num_events` events of the config's stream (default: all) with
    their edge features and the GRU weights.  tcsr_events > num_events (None:
    the whole stream) also returns that longer stream's (src, dst, ts) as
    "tcsr": the sampler's T-CSR is then built over it, so rows have their
    full-stream lengths (GDELT: 22,934 entries on average) while the batches
    run over the prefix.  The stream is prefix-consistent (every draw is
    sequential), so the prefix is the first events of the longer stream, and
    the sampler's strict ts < t_q never sees an event past the prefix."""
    cfg = CONFIGS[name]
    E = cfg.num_events if num_events is None else int(num_events)
    Et = E if tcsr_events is None else min(int(tcsr_events), cfg.num_events)
    if Et > E:
        fsrc, fdst, fts, fneg = make_events(cfg, seed, Et)
        src, dst, ts, neg = fsrc[:E].copy(), fdst[:E].copy(), fts[:E].copy(), fneg[:E].copy()
        del fneg
    else:
        src, dst, ts, neg = make_events(cfg, seed, E)
    out = dict(cfg=cfg, src=src, dst=dst, ts=ts, neg=neg, seed=seed)
    if Et > E:
        out["tcsr"] = (fsrc, fdst, fts)
    if with_features:
        out["ef"] = edge_features(seed, 0, len(src), cfg.edge_dim)
    out["params"] = gru_params(cfg.mem_dim, cfg.mail_dim, cfg.time_dim)
    return out

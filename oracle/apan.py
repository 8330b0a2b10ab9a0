"""Row F3 oracle, APAN updater — plain numpy f64, one iteration at a time.

TEST INFRASTRUCTURE ONLY (tests/ import it; the product package never does).
Shares no code with the CUDA path; A1 / A2 come from this oracle's C routines.

The paper names APAN among the MTGNNs it trains ("modified from TGL",
P:L405) and describes it as using "RNN as the memory update function while
incorporating an attention mechanism ... APAN further optimizes inference
speed by using asynchronous propagation".  Readings (DESIGN.md §3,
F3-4..F3-8):
  F3-4  mailbox: S_mb = 10 slots per node (ring): mail rows [N, S_mb, Dm],
        their times [N, S_mb], the next slot and the filled-slot count per node.
  F3-5  message of winner w (event a, t* = ts_a) from the snapshot S:
          q = W_q S.mem[w],  k_s = W_k S.mb[w, s]  (filled slots s),
          α = softmax_s(q·k_s / √M),  m = Σ_s α_s S.mb[w, s]  (0: empty box),
          x = [m ‖ cos(ω (t* - S.mem_ts[w]) + ϕ)]  (G2, G4);
        h' = GRUCell(x, S.mem[w]) — "RNN as the memory update function"
        (the GRU weights have the TGN shapes, Dx = Dm + d_t).
  F3-6  commit: mem[w] = h', mem_ts[w] = t* (A7).
  F3-7  the mail of winner w: [h'_w ‖ h'_o ‖ e_a] from the committed memories
        (o = the other endpoint, itself a winner), time t_a (as F3-2).
  F3-8  asynchronous propagation: w's mail is delivered to w and to the
        sampled neighbours of w's root row (A1 at t_a, the 𝒩 most recent);
        a node reached by several mails in one batch keeps the one with the
        largest key p (F + 1) + s (p = the sender's winning pair, s = 0 for
        itself, 1 + j for neighbour slot j) — the latest event's mail — and
        writes it into its next ring slot.
"""
from __future__ import annotations

import numpy as np

from . import Graph, dedup
from .train import gru_forward, time_encode

SLOTS = 10


def new_mailbox(num_nodes, mem_dim, edge_dim, slots=SLOTS):
    Dm = 2 * mem_dim + edge_dim
    return dict(mb=np.zeros((num_nodes, slots, Dm), np.float32), mb_ts=np.zeros((num_nodes, slots)),
                mb_pos=np.zeros(num_nodes, np.int32), mb_cnt=np.zeros(num_nodes, np.int32))


def attention_message(mem_w, mb_w, cnt_w, w_q, w_k):
    """F3-5 for U winners: mem_w [U, M], mb_w [U, S, Dm], cnt_w [U] filled slots
    (slots 0..cnt-1 hold mails once the ring is full or partially filled from 0)."""
    M = mem_w.shape[1]
    q = np.asarray(mem_w, np.float64) @ np.asarray(w_q, np.float64).T           # [U, M]
    k = np.asarray(mb_w, np.float64) @ np.asarray(w_k, np.float64).T            # [U, S, M]
    S = mb_w.shape[1]
    valid = np.arange(S)[None, :] < np.asarray(cnt_w)[:, None]
    e = np.einsum("um,usm->us", q, k) / np.sqrt(M)
    e = np.where(valid, e, -np.inf)
    mx = np.max(np.where(valid, e, -1e300), axis=1, keepdims=True)
    p = np.where(valid, np.exp(e - mx), 0.0)
    den = p.sum(1, keepdims=True)
    a = np.divide(p, den, out=np.zeros_like(p), where=den > 0)
    return np.einsum("us,usd->ud", a, np.asarray(mb_w, np.float64)), a


def step(num_nodes, src, dst, ts, ef, state, box, graph: Graph, gru, apan, fanout=10, latest=None, latest_box=None):
    """One APAN iteration: the message and the GRU read the snapshot (state, box)
    = version v(i) (Eq. 2); the commit and the deliveries apply to
    the latest version (latest, latest_box; default: the snapshot, k = 0).
    Returns the new (state, box) and the winners' h'."""
    src, dst = np.asarray(src, np.int32), np.asarray(dst, np.int32)
    ts = np.asarray(ts, np.float64)
    B = len(src)
    M = state["mem"].shape[1]
    nodes, winner = dedup(num_nodes, src, dst)                                # A2
    ev, role = winner >> 1, winner & 1
    mem, mem_ts = state["mem"], state["mem_ts"]
    msg, _ = attention_message(mem[nodes], box["mb"][nodes], box["mb_cnt"][nodes], apan["w_q"], apan["w_k"])
    dt = (ts[ev] - mem_ts[nodes]).astype(np.float32)
    x = np.concatenate([msg, time_encode(dt, gru["time_w"], gru["time_b"])], 1)
    hn, _ = gru_forward(x, np.asarray(mem[nodes], np.float64), gru)          # F3-5
    new = {k: v.copy() for k, v in (state if latest is None else latest).items()}
    new["mem"][nodes] = hn.astype(np.float32)                                 # F3-6
    new["mem_ts"][nodes] = ts[ev]
    other = np.where(role == 1, src[ev], dst[ev])
    mails = np.concatenate([new["mem"][nodes], new["mem"][other], np.asarray(ef, np.float32)[ev]], 1)  # F3-7
    # F3-8: candidates (target, key, mail row index)
    roots = np.where(role == 1, dst[ev], src[ev])
    smp = graph.sample(roots, ts[ev], fanout)
    best = {}
    for u in range(len(nodes)):
        cands = [(int(nodes[u]), 0)] + [(int(smp["nbr"][u, j]), 1 + j) for j in range(int(smp["cnt"][u]))]
        for v, s in cands:
            key = int(winner[u]) * (fanout + 1) + s
            if v not in best or key > best[v][0]:
                best[v] = (key, u)
    nb = {k: v.copy() for k, v in (box if latest_box is None else latest_box).items()}
    S = box["mb"].shape[1]
    for v, (key, u) in best.items():
        pos = nb["mb_pos"][v]
        nb["mb"][v, pos] = mails[u]
        nb["mb_ts"][v, pos] = ts[ev[u]]
        nb["mb_pos"][v] = (pos + 1) % S
        nb["mb_cnt"][v] = min(nb["mb_cnt"][v] + 1, S)
    return new, nb, dict(nodes=nodes, winner=winner, h_new=hn, mails=mails, targets=best)


def run_stream(num_nodes, src, dst, ts, ef, gru, apan, batch, fanout=10, max_batches=-1, slots=SLOTS, k=0):
    """Over the stream (the T-CSR of the whole stream; A1's strict ts < t) under
    the exact staleness schedule: batch i reads version v(i) = max(0, i-1-k)."""
    import oracle
    src, dst, ts = np.asarray(src, np.int32), np.asarray(dst, np.int32), np.asarray(ts, np.float64)
    M = np.asarray(gru["w_hh"]).shape[1]
    He = np.asarray(ef).shape[1]
    state = oracle.new_state(num_nodes, M, He)
    box = new_mailbox(num_nodes, M, He, slots)
    graph = Graph(num_nodes, src, dst, ts)
    nb = -(-len(src) // batch)
    if max_batches >= 0:
        nb = min(nb, max_batches)
    hist = [(state, box)]  # version v = after batch v
    for i in range(1, nb + 1):
        b = slice((i - 1) * batch, min(i * batch, len(src)))
        snap_s, snap_b = hist[max(0, i - 1 - k)]
        state, box, _ = step(num_nodes, src[b], dst[b], ts[b], ef[b], snap_s, snap_b, graph, gru, apan, fanout,
                             latest=hist[-1][0], latest_box=hist[-1][1])
        hist.append((state, box))
    return state, box

"""Row F4 oracle — the MTGNN training stage of one iteration, plain numpy fp64.

TEST INFRASTRUCTURE ONLY: imported by tests/ (and nothing in the product
package).  Shares no code with the CUDA path; the A1 sampler and A2 dedup it
needs come from this oracle's own C routines (oracle/oracle.c via
oracle/__init__.py).

What it computes (Eq. 1, Eq. 2):
  m^(i)_v = msg(s~_v, s~_u, y_uv(t), Δt)          message of the winner event (A5, G1-G4)
  s~^(i)_v = mem(s~^(i-k)_v, m^(i)_v)             GRUCell (A6, G5)
  h^(i)_v  = emb(s~^(i)_v, s~^(i)_u | u ∈ N(v))   "a single layer GAT"
then the link decoder, the loss, "the loss and backward steps" and
the SGD update of every learnable module ("msg ..., mem ..., emb ... are all
learnable"; η, §5.1).  Readings (T1-T7):
  T1  s~^(i)_v for a subgraph node v = the GRU output h'_v of this batch if v
      is one of its winners, else the fetched (stale) row s^(v(i))_v — Eq. 2
      writes s~^(i) for every node, and nodes without an event at iteration i
      keep their memory.
  T2  the stored memory is not a parameter: gradients reach the GRU weights
      through h'_v and stop at the snapshot rows (TGN/TGL detach memory).
  T3  emb: single-head temporal attention over the node's sampled neighbours
      (A1 output, up to 𝒩 = 10), H = 100:
        q = W_q s~_v,  k_u = W_k [s~_u ‖ φ(Δt_u)],  v_u = W_v [s~_u ‖ φ(Δt_u)],
        α = softmax_u(q·k_u / √H) over the cnt valid neighbours,
        a = Σ_u α_u v_u  (0 when cnt = 0),   h_v = W_o [a ‖ s~_v] + b_o,
      φ = the message's fixed time encoder cos(ω Δt + ϕ) (G2), Δt_u = t_q - t_e
      as the sampler returns it (f32).
  T4  decoder (a link MLP; the paper names none): logit(a, b) =
      w_2·tanh(W_1 [h_a ‖ h_b] + b_1) + b_2 — smooth, so no f32-vs-f64 kink
      decision (TGN's ReLU) separates the GPU from this oracle.
  T5  loss: mean binary cross-entropy on logits over the B positive (src, dst)
      and B negative (src, neg) pairs ("equal number of positive and
      negative").
  T6  SGD θ <- θ - η g on every learnable tensor (the time encoder is fixed,
      S:L277-L279); parameters are stored in f32 (rounded after each step).
  T7  data parallel: every rank computes the gradient of its
      local batch's mean loss; the all-reduce averages them.
"""
from __future__ import annotations

import numpy as np

from . import Graph, dedup

TRAIN_KEYS = ("w_q", "w_k", "w_v", "w_o", "b_o", "w_1", "b_1", "w_2", "b_2")
GRU_KEYS = ("w_ih", "w_hh", "b_ih", "b_hh")


def _f64(a):
    return np.asarray(a, dtype=np.float64)


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def softplus(x):
    """log(1 + e^x), evaluated without overflow."""
    return np.maximum(x, 0.0) + np.log1p(np.exp(-np.abs(x)))


def time_encode(dt, time_w, time_b):
    """φ(Δt)_q = cos(ω_q Δt + ϕ_q) (G2): the argument rounded to f32 as the
    message's fmaf does (oracle.c orc_build_x), the cosine in f64."""
    dt = np.asarray(dt, np.float32)[..., None].astype(np.float64)
    arg = (dt * _f64(time_w) + _f64(time_b)).astype(np.float32)
    return np.cos(arg.astype(np.float64))


# ---------------------------------------------------------------- A6 (GRUCell)
def gru_forward(x, h, g):
    """torch.nn.GRUCell, gates (r, z, n) (G5):
      r = σ(W_ir x + b_ir + W_hr h + b_hr), z = σ(W_iz x + b_iz + W_hz h + b_hz),
      n = tanh(W_in x + b_in + r ⊙ (W_hn h + b_hn)),  h' = (1 - z) ⊙ n + z ⊙ h."""
    M = h.shape[1]
    gi = x @ _f64(g["w_ih"]).T + _f64(g["b_ih"])
    gh = h @ _f64(g["w_hh"]).T + _f64(g["b_hh"])
    r = sigmoid(gi[:, :M] + gh[:, :M])
    z = sigmoid(gi[:, M:2 * M] + gh[:, M:2 * M])
    n = np.tanh(gi[:, 2 * M:] + r * gh[:, 2 * M:])
    hn = (1.0 - z) * n + z * h
    return hn, dict(r=r, z=z, n=n, ghn=gh[:, 2 * M:])


def gru_backward(dhn, x, h, c):
    """Chain rule of gru_forward: gradients of w_ih, w_hh, b_ih, b_hh."""
    r, z, n, ghn = c["r"], c["z"], c["n"], c["ghn"]
    dn = dhn * (1.0 - z)
    dz = dhn * (h - n)
    dan = dn * (1.0 - n * n)          # d(pre-activation of n)
    dghn = dan * r                    # d(W_hn h + b_hn)
    dr = dan * ghn
    dar = dr * r * (1.0 - r)
    daz = dz * z * (1.0 - z)
    dgi = np.concatenate([dar, daz, dan], axis=1)   # d(W_ih x + b_ih)
    dgh = np.concatenate([dar, daz, dghn], axis=1)  # d(W_hh h + b_hh)
    return dict(w_ih=dgi.T @ x, w_hh=dgh.T @ h, b_ih=dgi.sum(0), b_hh=dgh.sum(0))


# ---------------------------------------------------------------- T3 (emb)
def attention_forward(s_root, s_nbr, phi, cnt, p):
    """T3 for R roots: s_root [R, M], s_nbr [R, F, M], phi [R, F, Dt], cnt [R]."""
    R, F, _ = s_nbr.shape
    H = p["w_q"].shape[0]
    zn = np.concatenate([s_nbr, phi], axis=2)                 # [R, F, M + Dt]
    q = s_root @ _f64(p["w_q"]).T                             # [R, H]
    k = zn @ _f64(p["w_k"]).T                                 # [R, F, H]
    v = zn @ _f64(p["w_v"]).T
    valid = np.arange(F)[None, :] < np.asarray(cnt)[:, None]  # [R, F]
    score = np.einsum("rh,rfh->rf", q, k) / np.sqrt(H)
    score = np.where(valid, score, -np.inf)
    mx = np.max(np.where(valid, score, -1e300), axis=1, keepdims=True)
    e = np.where(valid, np.exp(score - mx), 0.0)
    den = e.sum(1, keepdims=True)
    alpha = np.divide(e, den, out=np.zeros_like(e), where=den > 0)
    a = np.einsum("rf,rfh->rh", alpha, v)
    zo = np.concatenate([a, s_root], axis=1)                  # [R, H + M]
    emb = zo @ _f64(p["w_o"]).T + _f64(p["b_o"])
    return emb, dict(zn=zn, q=q, k=k, v=v, alpha=alpha, zo=zo, valid=valid)


def attention_backward(demb, s_root, c, p):
    """Chain rule of attention_forward: parameter gradients and the gradients
    of s_root [R, M] and of the neighbour memories s_nbr [R, F, M]."""
    H = p["w_q"].shape[0]
    M = s_root.shape[1]
    g = dict(w_o=demb.T @ c["zo"], b_o=demb.sum(0))
    dzo = demb @ _f64(p["w_o"])
    da, ds_root = dzo[:, :H], dzo[:, H:].copy()
    alpha, k, v, q = c["alpha"], c["k"], c["v"], c["q"]
    dalpha = np.einsum("rh,rfh->rf", da, v)
    dv = alpha[:, :, None] * da[:, None, :]
    dscore = alpha * (dalpha - np.sum(alpha * dalpha, axis=1, keepdims=True))
    dq = np.einsum("rf,rfh->rh", dscore, k) / np.sqrt(H)
    dk = dscore[:, :, None] * q[:, None, :] / np.sqrt(H)
    zn = c["zn"]
    g["w_q"] = dq.T @ s_root
    g["w_k"] = np.einsum("rfh,rfc->hc", dk, zn)
    g["w_v"] = np.einsum("rfh,rfc->hc", dv, zn)
    ds_root += dq @ _f64(p["w_q"])
    dzn = dk @ _f64(p["w_k"]) + dv @ _f64(p["w_v"])
    return g, ds_root, dzn[:, :, :M]


# ---------------------------------------------------------------- T4 + T5
def decode_loss(emb, B, p):
    """Roots are [src | dst | neg] (3B rows of emb): pair j = (src_j, dst_j)
    label 1, pair B + j = (src_j, neg_j) label 0."""
    za = np.concatenate([np.concatenate([emb[:B], emb[B:2 * B]], 1),
                         np.concatenate([emb[:B], emb[2 * B:3 * B]], 1)], 0)   # [2B, 2H]
    pre = za @ _f64(p["w_1"]).T + _f64(p["b_1"])
    y = np.tanh(pre)
    logit = y @ _f64(p["w_2"]) + _f64(p["b_2"])[0]
    lab = np.concatenate([np.ones(B), np.zeros(B)])
    loss = np.mean(softplus(-logit) * lab + softplus(logit) * (1.0 - lab))
    return loss, logit, dict(za=za, pre=pre, y=y, lab=lab)


def decode_backward(logit, B, c, p):
    H = p["w_2"].shape[0]
    dlogit = (sigmoid(logit) - c["lab"]) / (2.0 * B)
    g = dict(w_2=c["y"].T @ dlogit, b_2=np.array([dlogit.sum()]))
    dpre = dlogit[:, None] * _f64(p["w_2"])[None, :] * (1.0 - c["y"] ** 2)
    g["w_1"] = dpre.T @ c["za"]
    g["b_1"] = dpre.sum(0)
    dza = dpre @ _f64(p["w_1"])
    demb = np.zeros((3 * B, H))
    demb[:B] = dza[:B, :H] + dza[B:, :H]
    demb[B:2 * B] = dza[:B, H:]
    demb[2 * B:] = dza[B:, H:]
    return g, demb


# ---------------------------------------------------------------- one iteration
def build_message(src, dst, ts, ef, mem, mem_ts, winner, gru):
    """A5 for the winners (G1-G4): x = [s_w ‖ s_o ‖ e ‖ φ(t* - S.mem_ts[w])], h = s_w."""
    ev = winner >> 1
    role = winner & 1
    w = np.where(role == 1, dst[ev], src[ev])
    o = np.where(role == 1, src[ev], dst[ev])
    dt = (ts[ev] - mem_ts[w]).astype(np.float32)
    x = np.concatenate([_f64(mem[w]), _f64(mem[o]), _f64(ef[ev]), time_encode(dt, gru["time_w"], gru["time_b"])], 1)
    return x, _f64(mem[w])


def train_step(num_nodes, src, dst, neg, ts, ef, mem, mem_ts, graph: Graph, gru: dict, prm: dict, fanout=10,
               mitigation=None):
    """Forward and backward of one iteration on the snapshot tables (mem,
    mem_ts) = S_{v(i)}.  Returns loss, logits, emb, every gradient (fp64),
    and the winners' (nodes, h') that the stage commits.  mitigation
    (dict(lam, gamma, n_sim)): the GRU's hidden input is MSPipe-S's blended
    row (A4, G13), taken from this oracle's own A4."""
    src, dst, neg = (np.asarray(a, np.int32) for a in (src, dst, neg))
    ts = np.asarray(ts, np.float64)
    B = len(src)
    nodes, winner = dedup(num_nodes, src, dst)                   # A2
    x, h = build_message(src, dst, ts, ef, mem, mem_ts, winner, gru)
    if mitigation is not None:                                   # A4: h = ŝ of each winner
        from . import memory_update
        mu = memory_update(num_nodes, src, dst, ts, ef, gru, mem, mem_ts, mitigation=mitigation, graph=graph,
                           fanout=fanout)
        assert np.array_equal(mu["nodes"], nodes)
        h = np.asarray(mu["h"], np.float64)
    hn, gc = gru_forward(x, h, gru)                              # A6: s~^(i) of the winners
    roots = np.concatenate([src, dst, neg])
    qts = np.concatenate([ts, ts, ts])
    smp = graph.sample(roots, qts, fanout)                       # A1 on the 3B roots
    cnt, nbr, dtn = smp["cnt"], smp["nbr"], smp["dt"]
    wrow = np.full(num_nodes, -1, np.int64)
    wrow[nodes] = np.arange(len(nodes))

    def s_tilde(ids):  # T1
        ids = np.asarray(ids)
        out = np.zeros(ids.shape + (mem.shape[1],))
        ok = ids >= 0
        out[ok] = _f64(mem[ids[ok]])
        u = np.where(ok, wrow[np.where(ok, ids, 0)], -1)
        hit = u >= 0
        out[hit] = hn[u[hit]]
        return out, u

    s_root, u_root = s_tilde(roots)
    s_nbr, u_nbr = s_tilde(nbr)
    phi = time_encode(dtn, gru["time_w"], gru["time_b"])
    emb, ac = attention_forward(s_root, s_nbr, phi, cnt, prm)
    loss, logit, dc = decode_loss(emb, B, prm)
    # backward ("the loss and backward steps")
    g, demb = decode_backward(logit, B, dc, prm)
    ga, ds_root, ds_nbr = attention_backward(demb, s_root, ac, prm)
    g.update(ga)
    ds_nbr = np.where((np.arange(fanout)[None, :] < cnt[:, None])[:, :, None], ds_nbr, 0.0)
    dhn = np.zeros_like(hn)                                      # T2: only through h'
    np.add.at(dhn, u_root[u_root >= 0], ds_root[u_root >= 0])
    np.add.at(dhn, u_nbr[u_nbr >= 0], ds_nbr[u_nbr >= 0])
    g.update(gru_backward(dhn, x, h, gc))
    return dict(loss=loss, logit=logit, emb=emb, grads=g, nodes=nodes, winner=winner, h_new=hn,
                dh_new=dhn, alpha=ac["alpha"], cnt=cnt)


def sgd(params: dict, grads: dict, lr: float) -> dict:
    """T6: θ <- θ - η g, stored in f32."""
    return {k: (np.asarray(v, np.float32) if k not in grads else
                (_f64(v) - lr * grads[k]).astype(np.float32)) for k, v in params.items()}


def allreduce_mean(grad_list):
    """T7: the data-parallel all-reduce of per-rank gradients (mean over ranks)."""
    return {k: sum(g[k] for g in grad_list) / len(grad_list) for k in grad_list[0]}

"""Pins of the row F4 training-stage oracle (oracle/train.py) against things
other than itself: central finite differences of its own loss (every
learnable tensor, f64), library routines (torch.nn.GRUCell,
scaled_dot_product_attention, binary_cross_entropy_with_logits, all f64),
closed forms (zero decoder -> ln 2; no history -> a = 0; one neighbour ->
α = 1), invariants (neighbour permutation), and the descent property of the
SGD step.  No expected value here comes from the CUDA path."""
import math

import numpy as np
import pytest
import torch

import oracle
from oracle import train as ot
from synth import gru_params, train_params


def _instance(seed=0, N=9, M=4, He=3, Dt=2, H=3, B=4, hist=24, F=3):
    """A tiny stream: `hist` past events (the T-CSR) then one batch of B."""
    rng = np.random.default_rng(seed)
    E = hist + B
    src = rng.integers(0, N, E).astype(np.int32)
    dst = (src + 1 + rng.integers(0, N - 1, E)).astype(np.int32) % N
    ts = np.cumsum(rng.uniform(0.5, 2.0, E))
    ef = rng.uniform(-1, 1, (E, He)).astype(np.float32)
    neg = rng.integers(0, N, B).astype(np.int32)
    mem = rng.uniform(-1, 1, (N, M)).astype(np.float32)
    mem_ts = np.minimum(rng.uniform(0, ts[hist - 1], N), ts[hist]) * (rng.uniform(size=N) < 0.8)
    g = gru_params(M, 2 * M + He, Dt, seed=seed + 11)
    g["time_b"] = rng.uniform(-1, 1, Dt).astype(np.float32)
    p = train_params(M, Dt, H, seed=seed + 13)
    graph = oracle.Graph(N, src, dst, ts)
    b = slice(hist, E)
    return dict(N=N, src=src[b], dst=dst[b], neg=neg, ts=ts[b], ef=ef[b], mem=mem, mem_ts=mem_ts,
                graph=graph, gru=g, prm=p, F=F)


def _run(I, gru=None, prm=None):
    return ot.train_step(I["N"], I["src"], I["dst"], I["neg"], I["ts"], I["ef"], I["mem"], I["mem_ts"],
                         I["graph"], I["gru"] if gru is None else gru, I["prm"] if prm is None else prm,
                         fanout=I["F"])


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_gradients_match_central_differences(seed):
    """Every learnable tensor (emb, decoder, GRU): analytic vs central
    differences of the f64 loss, relative error < 1e-6."""
    I = _instance(seed)
    I["gru"] = {k: np.asarray(v, np.float64) for k, v in I["gru"].items()}
    I["prm"] = {k: np.asarray(v, np.float64) for k, v in I["prm"].items()}
    out = _run(I)
    assert len(out["nodes"]) > 0 and out["cnt"].max() > 1
    eps = 1e-6
    for group, keys in (("prm", ot.TRAIN_KEYS), ("gru", ot.GRU_KEYS)):
        for k in keys:
            base = I[group][k]
            fd = np.zeros(base.shape)
            for idx in np.ndindex(base.shape):
                lo, hi = base.copy(), base.copy()
                lo[idx] -= eps
                hi[idx] += eps
                Ll = _run(I, **{group: {**I[group], k: lo}})["loss"]
                Lh = _run(I, **{group: {**I[group], k: hi}})["loss"]
                fd[idx] = (Lh - Ll) / (2 * eps)
            an = out["grads"][k]
            scale = max(np.abs(fd).max(), 1e-12)
            assert np.abs(an - fd).max() <= 1e-6 * scale + 1e-10, (k, np.abs(an - fd).max(), scale)
            assert np.abs(fd).max() > 0, k  # the tensor is really on the path


def test_gru_matches_torch_grucell():
    rng = np.random.default_rng(3)
    M, Dx, U = 5, 7, 6
    g = dict(w_ih=rng.normal(size=(3 * M, Dx)), w_hh=rng.normal(size=(3 * M, M)), b_ih=rng.normal(size=3 * M),
             b_hh=rng.normal(size=3 * M))
    x, h = rng.normal(size=(U, Dx)), rng.normal(size=(U, M))
    cell = torch.nn.GRUCell(Dx, M).double()
    with torch.no_grad():
        for k in ("w_ih", "w_hh", "b_ih", "b_hh"):
            getattr(cell, k.replace("w_", "weight_").replace("b_", "bias_")).copy_(torch.from_numpy(g[k]))
    xt = torch.from_numpy(x).requires_grad_()
    ht = torch.from_numpy(h)
    ref = cell(xt, ht)
    got, c = ot.gru_forward(x, h, g)
    assert np.allclose(got, ref.detach().numpy(), rtol=1e-13, atol=1e-13)
    dh = rng.normal(size=(U, M))
    ref.backward(torch.from_numpy(dh))
    gg = ot.gru_backward(dh, x, h, c)
    assert np.allclose(gg["w_ih"], cell.weight_ih.grad.numpy(), rtol=1e-12, atol=1e-12)
    assert np.allclose(gg["w_hh"], cell.weight_hh.grad.numpy(), rtol=1e-12, atol=1e-12)
    assert np.allclose(gg["b_ih"], cell.bias_ih.grad.numpy(), rtol=1e-12, atol=1e-12)
    assert np.allclose(gg["b_hh"], cell.bias_hh.grad.numpy(), rtol=1e-12, atol=1e-12)


def test_attention_matches_sdpa():
    """T3's softmax attention = torch's scaled_dot_product_attention (one head,
    boolean mask of the valid neighbours) for rows with cnt >= 1."""
    rng = np.random.default_rng(4)
    R, F, M, Dt, H = 7, 5, 4, 3, 6
    p = dict(w_q=rng.normal(size=(H, M)), w_k=rng.normal(size=(H, M + Dt)), w_v=rng.normal(size=(H, M + Dt)),
             w_o=rng.normal(size=(H, H + M)), b_o=rng.normal(size=H))
    s_root, s_nbr = rng.normal(size=(R, M)), rng.normal(size=(R, F, M))
    phi = rng.normal(size=(R, F, Dt))
    cnt = np.array([1, 2, 5, 3, 4, 5, 1])
    emb, c = ot.attention_forward(s_root, s_nbr, phi, cnt, p)
    zn = torch.from_numpy(np.concatenate([s_nbr, phi], 2))
    q = torch.from_numpy(s_root) @ torch.from_numpy(p["w_q"]).T
    k = zn @ torch.from_numpy(p["w_k"]).T
    v = zn @ torch.from_numpy(p["w_v"]).T
    mask = torch.arange(F)[None, :] < torch.from_numpy(cnt)[:, None]
    a = torch.nn.functional.scaled_dot_product_attention(q[:, None, None, :], k[:, None], v[:, None],
                                                         attn_mask=mask[:, None, None, :])[:, 0, 0]
    ref = torch.cat([a, torch.from_numpy(s_root)], 1) @ torch.from_numpy(p["w_o"]).T + torch.from_numpy(p["b_o"])
    assert np.allclose(emb, ref.numpy(), rtol=1e-12, atol=1e-12)


def test_attention_closed_forms_and_permutation():
    rng = np.random.default_rng(5)
    R, F, M, Dt, H = 4, 4, 3, 2, 5
    p = dict(w_q=rng.normal(size=(H, M)), w_k=rng.normal(size=(H, M + Dt)), w_v=rng.normal(size=(H, M + Dt)),
             w_o=rng.normal(size=(H, H + M)), b_o=rng.normal(size=H))
    s_root, s_nbr, phi = rng.normal(size=(R, M)), rng.normal(size=(R, F, M)), rng.normal(size=(R, F, Dt))
    # no history: a = 0, h = W_o[:, H:] s + b_o
    emb, _ = ot.attention_forward(s_root, s_nbr, phi, np.zeros(R, int), p)
    assert np.allclose(emb, s_root @ p["w_o"][:, H:].T + p["b_o"], rtol=1e-14, atol=1e-14)
    # one neighbour: α = 1, a = v_0
    emb1, c1 = ot.attention_forward(s_root, s_nbr, phi, np.ones(R, int), p)
    v0 = np.concatenate([s_nbr[:, 0], phi[:, 0]], 1) @ p["w_v"].T
    assert np.allclose(c1["alpha"][:, 0], 1.0)
    assert np.allclose(emb1, np.concatenate([v0, s_root], 1) @ p["w_o"].T + p["b_o"], rtol=1e-13, atol=1e-13)
    # permutation of the valid neighbours leaves h unchanged
    perm = np.array([2, 0, 3, 1])
    e_a, _ = ot.attention_forward(s_root, s_nbr, phi, np.full(R, F), p)
    e_b, _ = ot.attention_forward(s_root, s_nbr[:, perm], phi[:, perm], np.full(R, F), p)
    assert np.allclose(e_a, e_b, rtol=1e-13, atol=1e-13)


def test_loss_matches_torch_bce_and_zero_decoder():
    rng = np.random.default_rng(6)
    B, H = 5, 4
    p = dict(w_1=rng.normal(size=(H, 2 * H)), b_1=rng.normal(size=H), w_2=rng.normal(size=H), b_2=rng.normal(size=1))
    emb = rng.normal(size=(3 * B, H))
    loss, logit, _ = ot.decode_loss(emb, B, p)
    lab = torch.cat([torch.ones(B), torch.zeros(B)]).double()
    ref = torch.nn.functional.binary_cross_entropy_with_logits(torch.from_numpy(logit), lab)
    assert abs(loss - ref.item()) < 1e-14
    # logits forced to 0 -> p = 1/2, loss = ln 2
    z = dict(p, w_2=np.zeros(H), b_2=np.zeros(1))
    assert abs(ot.decode_loss(emb, B, z)[0] - math.log(2.0)) < 1e-15


def test_winner_rows_reach_the_embedding():
    """T1: a root whose node is a winner sees h' (the GRU output), others the
    snapshot row: zeroing every GRU weight and bias gives h' = s/2 (r = z = 1/2,
    n = 0), which must change exactly the winners' root rows."""
    I = _instance(7)
    g0 = {k: (np.zeros_like(v) if k in ot.GRU_KEYS else v) for k, v in I["gru"].items()}
    out = _run(I, gru=g0)
    assert np.allclose(out["h_new"], 0.5 * I["mem"][out["nodes"]].astype(np.float64), rtol=0, atol=1e-15)


def test_sgd_step_descends():
    """A small step along -g lowers the same batch's loss (first-order descent)."""
    I = _instance(8)
    out = _run(I)
    lr = 1e-3
    prm = ot.sgd(I["prm"], out["grads"], lr)
    gru = ot.sgd(I["gru"], {k: out["grads"][k] for k in ot.GRU_KEYS}, lr)
    after = _run(I, gru=gru, prm=prm)["loss"]
    gn2 = sum(float(np.sum(out["grads"][k] ** 2)) for k in ot.TRAIN_KEYS + ot.GRU_KEYS)
    assert after < out["loss"]
    assert abs((out["loss"] - after) - lr * gn2) <= 0.05 * lr * gn2 + 1e-7  # ≈ η‖g‖² (f32 storage)


def test_allreduce_mean():
    a = dict(w=np.array([1.0, 2.0]))
    b = dict(w=np.array([3.0, 6.0]))
    assert np.array_equal(ot.allreduce_mean([a, b])["w"], np.array([2.0, 4.0]))

"""Pins of the APAN oracle (oracle/apan.py, row F3 readings F3-4..F3-8)
against things other than itself: torch's scaled_dot_product_attention (f64)
for the mailbox attention, closed forms (one mail -> that mail, empty box ->
0, W_q = 0 -> the plain mean of the filled slots), a hand-worked delivery
example (targets, winning keys, ring slots), and ring invariants."""
import numpy as np
import torch

import oracle
from oracle import apan
from synth import gru_params


def _w(M, Dm, seed):
    rng = np.random.default_rng(seed)
    return dict(w_q=rng.normal(size=(M, M)) / np.sqrt(M), w_k=rng.normal(size=(M, Dm)) / np.sqrt(Dm))


def test_attention_matches_sdpa():
    rng = np.random.default_rng(1)
    U, S, M, Dm = 6, 10, 4, 7
    w = _w(M, Dm, 2)
    mem, mb = rng.normal(size=(U, M)), rng.normal(size=(U, S, Dm))
    cnt = np.array([1, 3, 10, 7, 2, 10])
    got, _ = apan.attention_message(mem, mb, cnt, w["w_q"], w["w_k"])
    q = torch.from_numpy(mem @ w["w_q"].T)
    k = torch.from_numpy(mb @ w["w_k"].T)
    mask = torch.arange(S)[None, :] < torch.from_numpy(cnt)[:, None]
    ref = torch.nn.functional.scaled_dot_product_attention(q[:, None, None], k[:, None], torch.from_numpy(mb)[:, None],
                                                           attn_mask=mask[:, None, None])[:, 0, 0]
    assert np.allclose(got, ref.numpy(), rtol=1e-12, atol=1e-12)


def test_attention_closed_forms():
    rng = np.random.default_rng(3)
    U, S, M, Dm = 4, 10, 5, 6
    w = _w(M, Dm, 4)
    mem, mb = rng.normal(size=(U, M)), rng.normal(size=(U, S, Dm))
    one, a1 = apan.attention_message(mem, mb, np.ones(U, int), w["w_q"], w["w_k"])
    assert np.allclose(one, mb[:, 0]) and np.allclose(a1[:, 0], 1.0)
    zero, _ = apan.attention_message(mem, mb, np.zeros(U, int), w["w_q"], w["w_k"])
    assert np.array_equal(zero, np.zeros((U, Dm)))
    cnt = np.array([2, 5, 10, 3])
    mean, _ = apan.attention_message(mem, mb, cnt, np.zeros((M, M)), w["w_k"])
    for u in range(U):
        assert np.allclose(mean[u], mb[u, :cnt[u]].mean(0), rtol=1e-14, atol=1e-14)


def test_delivery_worked_example():
    """Nodes 0..5.  History (ts 1..4): (0,1) (0,2) (3,1) (4,5).  Batch (ts 10, 11):
    (0,3) then (1,0); fanout 2.  Winners (A2, last pair wins): node 0 <- pair 3
    (event 1, dst), node 3 <- pair 1, node 1 <- pair 2.  Sampled neighbours at
    the winner's event time (newest first): node 0 at t=11: events (0,3)@10,
    (0,2)@2 -> [3, 2]; node 3 at t=10: (3,1)@3 -> [1]; node 1 at t=11:
    (0,3)? no — node 1's events: (3,1)@3, (0,1)@1 -> [3, 0].
    Candidates (key = p*3 + s): node 0: self 9; node 3: from 0 (s=1) 10,
    self 3, ... node 2: from 0 (s=2) 11; node 1: from 3 (s=1) 4, self 6;
    node 3 also from 1 (s=1) 7; node 0 from 1 (s=2) 8.
    Winners per target: 0 <- 9 (self), 3 <- 10 (node 0's mail), 2 <- 11 (0's),
    1 <- 6 (self)."""
    src = np.array([0, 0, 3, 4, 0, 1], np.int32)
    dst = np.array([1, 2, 1, 5, 3, 0], np.int32)
    ts = np.array([1.0, 2.0, 3.0, 4.0, 10.0, 11.0])
    N, M, He, Dt = 6, 4, 2, 3
    g = gru_params(M, 2 * M + He, Dt, seed=5)
    w = _w(M, 2 * M + He, 6)
    graph = oracle.Graph(N, src, dst, ts)
    state = oracle.new_state(N, M, He)
    box = apan.new_mailbox(N, M, He, slots=3)
    ef = np.arange(2 * He, dtype=np.float32).reshape(2, He)
    new, nb, info = apan.step(N, src[4:], dst[4:], ts[4:], ef, state, box, graph, g, w, fanout=2)
    assert list(info["nodes"]) == [3, 1, 0] or sorted(info["nodes"]) == [0, 1, 3]
    keys = {v: k for v, (k, _) in info["targets"].items()}
    assert keys == {0: 9, 3: 10, 2: 11, 1: 6}
    u_of = {int(n): u for u, n in enumerate(info["nodes"])}
    for v, sender in ((0, 0), (3, 0), (2, 0), (1, 1)):
        assert np.array_equal(nb["mb"][v, 0], info["mails"][u_of[sender]].astype(np.float32))
        assert nb["mb_cnt"][v] == 1 and nb["mb_pos"][v] == 1
    assert nb["mb_ts"][3, 0] == 11.0 and nb["mb_ts"][1, 0] == 11.0 and nb["mb_ts"][2, 0] == 11.0
    assert nb["mb_cnt"][4] == 0 and nb["mb_cnt"][5] == 0
    # the mail of winner w is [h'_w | h'_o | e]
    m0 = info["mails"][u_of[0]]
    assert np.array_equal(m0[:M], new["mem"][0]) and np.array_equal(m0[M:2 * M], new["mem"][1])
    assert np.array_equal(m0[2 * M:], ef[1])


def test_ring_keeps_the_last_slots_mails():
    """A node that receives S + 3 mails (one per batch) holds the last S of them,
    slot = arrival index mod S, and its count saturates at S."""
    N, M, He, Dt, S = 3, 4, 1, 2, 4
    g = gru_params(M, 2 * M + He, Dt, seed=7)
    w = _w(M, 2 * M + He, 8)
    n_b = S + 3
    src = np.zeros(n_b, np.int32)
    dst = np.ones(n_b, np.int32)
    ts = np.arange(1, n_b + 1, dtype=np.float64)
    ef = np.arange(n_b, dtype=np.float32)[:, None]
    graph = oracle.Graph(N, src, dst, ts)
    state, box = oracle.new_state(N, M, He), apan.new_mailbox(N, M, He, slots=S)
    for i in range(n_b):
        state, box, _ = apan.step(N, src[i:i + 1], dst[i:i + 1], ts[i:i + 1], ef[i:i + 1], state, box, graph, g, w,
                                  fanout=2)
    assert box["mb_cnt"][0] == S and box["mb_pos"][0] == n_b % S
    for j in range(n_b - S, n_b):
        assert box["mb_ts"][0, j % S] == ts[j]
        assert box["mb"][0, j % S, -1] == ef[j, 0]


def test_staleness_zero_equals_sequential_and_k_reads_old_versions():
    """run_stream(k=0) = stepping the latest version; with k = 2 the third batch's
    message reads version 0 (zeros: empty boxes, zero memory), so its h' equals
    the GRU of [0 | cos(w t + p)] with h = 0."""
    rng = np.random.default_rng(9)
    N, M, He, Dt, B = 12, 4, 2, 3, 5
    E = 4 * B
    src = rng.integers(0, N, E).astype(np.int32)
    dst = ((src + 1 + rng.integers(0, N - 1, E)) % N).astype(np.int32)
    ts = np.cumsum(rng.uniform(0.5, 1.5, E))
    ef = rng.uniform(-1, 1, (E, He)).astype(np.float32)
    g = gru_params(M, 2 * M + He, Dt, seed=3)
    w = _w(M, 2 * M + He, 4)
    s0, b0 = apan.run_stream(N, src, dst, ts, ef, g, w, B, fanout=3, k=0)
    graph = oracle.Graph(N, src, dst, ts)
    st, bx = oracle.new_state(N, M, He), apan.new_mailbox(N, M, He)
    for i in range(4):
        b = slice(i * B, (i + 1) * B)
        st, bx, _ = apan.step(N, src[b], dst[b], ts[b], ef[b], st, bx, graph, g, w, fanout=3)
    assert np.array_equal(s0["mem"], st["mem"]) and np.array_equal(b0["mb"], bx["mb"])
    # k = 2: batch 3 reads version 0
    hist = [(oracle.new_state(N, M, He), apan.new_mailbox(N, M, He))]
    for i in range(1, 4):
        b = slice((i - 1) * B, i * B)
        snap = hist[max(0, i - 1 - 2)]
        ns, nb, info = apan.step(N, src[b], dst[b], ts[b], ef[b], snap[0], snap[1], graph, g, w, fanout=3,
                                 latest=hist[-1][0], latest_box=hist[-1][1])
        hist.append((ns, nb))
    ev = info["winner"] >> 1
    from oracle.train import gru_forward, time_encode
    x = np.concatenate([np.zeros((len(ev), 2 * M + He)),
                        time_encode((ts[2 * B:3 * B][ev]).astype(np.float32), g["time_w"], g["time_b"])], 1)
    want, _ = gru_forward(x, np.zeros((len(ev), M)), g)
    assert np.allclose(info["h_new"], want, rtol=0, atol=1e-15)

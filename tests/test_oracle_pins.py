"""Pins of the CPU oracle against things other than itself.

Each test names the pin (P1..P12) and what fixes the expected value: the
definition written out by brute force, a hand-worked example, a closed form,
a library routine (torch.nn.GRUCell, numpy 'inverted_cdf' quantile) or an
invariant.  No expected value here comes from the CUDA path.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
from synth import CONFIGS, edge_features, gru_params, make_events

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _bias_only(M, He, Dt, c):
    """W = 0, b_ih[n-block] = c, other biases 0  =>  r = z = 1/2, n = tanh(c)."""
    Dx = 2 * M + He + Dt
    p = dict(w_ih=np.zeros((3 * M, Dx), np.float32), w_hh=np.zeros((3 * M, M), np.float32),
             b_ih=np.zeros(3 * M, np.float32), b_hh=np.zeros(3 * M, np.float32),
             time_w=np.ones(Dt, np.float32), time_b=np.zeros(Dt, np.float32))
    p["b_ih"][2 * M:] = c
    return p


# ---------------------------------------------------------------- P11 worked example
def test_p11_worked_example_sampler():
    g = _load("worked_example.json")
    ev = g["events"]
    q = g["sampler"]
    roots = [r["root"] for r in q]
    tq = [r["tq"] for r in q]
    for out in (oracle.sample_brute(ev["src"], ev["dst"], ev["ts"], roots, tq, g["fanout"]),
                oracle.Graph(g["num_nodes"], ev["src"], ev["dst"], ev["ts"]).sample(roots, tq, g["fanout"])):
        for i, r in enumerate(q):
            assert out["cnt"][i] == r["cnt"]
            assert list(out["nbr"][i]) == r["nbr"]
            assert list(out["eid"][i]) == r["eid"]
            assert list(out["ts"][i]) == r["ts"]
            assert list(out["dt"][i]) == r["dt"]


def test_p11_worked_example_winners():
    g = _load("worked_example.json")
    ev = g["events"]
    B = g["batch"]
    for b, w in enumerate(g["winners"]):
        s = np.array(ev["src"][b * B:(b + 1) * B])
        d = np.array(ev["dst"][b * B:(b + 1) * B])
        t = np.array(ev["ts"][b * B:(b + 1) * B])
        nodes, win = oracle.dedup(g["num_nodes"], s, d)
        assert list(nodes) == w["nodes"]
        assert list(win) == w["winner"]
        other = [int(d[p >> 1]) if p % 2 == 0 else int(s[p >> 1]) for p in win]
        assert other == w["other"]
        assert [float(t[p >> 1]) for p in win] == w["t"]


@pytest.mark.parametrize("key,k,schedule", [("k0_exact", 0, "exact"), ("k1_exact", 1, "exact"),
                                            ("k1_grouped", 1, "grouped")])
def test_p11_p4_worked_example_bias_closed_form(key, k, schedule):
    g = _load("worked_example.json")
    ev = g["events"]
    exp = g["bias_only_units_of_tanh_c"][key]
    M, He, Dt, c = 4, 3, 2, 0.7
    ef = edge_features(0, 0, 6, He)
    st, _ = oracle.run_stream(4, ev["src"], ev["dst"], ev["ts"], ef, _bias_only(M, He, Dt, c),
                              g["batch"], k, schedule)
    want = np.array(exp["mem"])[:, None] * math.tanh(c)
    assert np.allclose(st["mem"], np.broadcast_to(want, (4, M)), rtol=0, atol=2e-7)
    assert list(st["mem_ts"]) == exp["mem_ts"]
    assert list(st["mail_ts"]) == exp["mem_ts"]


@pytest.mark.parametrize("key,k", [("k0_exact", 0), ("k1_exact", 1)])
def test_p11_worked_example_dt_fed_to_encoder(key, k):
    """Time-block-only GRU (d_t = 1, ω = 1, φ = 0, W_in[time] = 1, b_iz = -40)
    gives h' = tanh(cos(Δt)) + O(e^-40): pins which Δt each winner sees."""
    g = _load("worked_example.json")
    ev = g["events"]
    exp = g["bias_only_units_of_tanh_c"][key]
    M, He, Dt = 2, 1, 1
    B = g["batch"]
    p = _bias_only(M, He, Dt, 0.0)
    p["w_ih"][2 * M:3 * M, 2 * M + He] = 1.0  # n-gate rows read the single time column
    p["b_ih"][M:2 * M] = -40.0                # z ~ 0
    ef = edge_features(0, 0, 6, He)
    for i, dts in enumerate(exp["dt"], start=1):
        v = oracle.snapshot_version(i, k)
        snap, _ = oracle.run_stream(4, ev["src"], ev["dst"], ev["ts"], ef, p, B, k, max_batches=v)
        sl = slice((i - 1) * B, i * B)
        out = oracle.memory_update(4, ev["src"][sl], ev["dst"][sl], ev["ts"][sl], ef[sl], p,
                                   snap["mem"], snap["mem_ts"])
        want = np.tanh(np.cos(np.array(dts, np.float64)))
        assert np.allclose(out["mem"][:, 0], want, atol=1e-6), (i, out["mem"][:, 0], want)


def test_p11_worked_example_mitigation():
    g = _load("worked_example.json")
    ev = g["events"]
    exp = g["mitigation_k0_gamma2.5_lambda0.5"]
    M, He, Dt, c = 3, 2, 2, 0.3
    p = _bias_only(M, He, Dt, c)
    ef = edge_features(0, 0, 6, He)
    mit = dict(lam=0.5, gamma=2.5, n_sim=5)
    st, _ = oracle.run_stream(4, ev["src"], ev["dst"], ev["ts"], ef, p, 2, 0, mitigation=mit, fanout=2)
    assert np.allclose(st["mem"], np.array(exp["mem"])[:, None] * math.tanh(c), atol=2e-7)
    graph = oracle.Graph(4, ev["src"], ev["dst"], ev["ts"])
    for i in range(1, 4):
        snap, _ = oracle.run_stream(4, ev["src"], ev["dst"], ev["ts"], ef, p, 2, 0, mitigation=mit,
                                    fanout=2, max_batches=i - 1)
        sl = slice((i - 1) * 2, i * 2)
        out = oracle.memory_update(4, ev["src"][sl], ev["dst"][sl], ev["ts"][sl], ef[sl], p,
                                   snap["mem"], snap["mem_ts"], mitigation=mit, graph=graph, fanout=2)
        assert list(out["elig"]) == exp["eligible"][i - 1]
        assert list(out["omega"][:, 0]) == exp["omega_first"][i - 1]


# ---------------------------------------------------------------- P1 sampler
def _brute_py(src, dst, ts, root, tq, fanout):
    """The definition once more, in Python, for tiny cases."""
    out = []
    for j in range(len(src) - 1, -1, -1):
        if len(out) == fanout:
            break
        if ts[j] < tq and (src[j] == root or dst[j] == root):
            out.append((int(dst[j] if src[j] == root else src[j]), j))
    return out


def test_p1_spec_examples():
    # cold start, 3 prior events newest first, 12 events keep last 10
    src = [5] * 12 + [7]
    dst = list(range(12)) + [5]
    ts = list(range(1, 14))
    g = oracle.Graph(20, src, dst, ts)
    out = g.sample([9, 5, 5, 19], [100.0, 4.0, 13.0, 13.0], 10)
    assert out["cnt"].tolist() == [1, 3, 10, 0]
    assert out["nbr"][1, :3].tolist() == [2, 1, 0]
    assert out["nbr"][2].tolist() == list(range(11, 1, -1))
    assert (out["ts"][2] < 13).all()


@pytest.mark.parametrize("name", ["tiny", "wiki", "lastfm"])
def test_p1_bsearch_sampler_equals_brute_force(name):
    cfg = CONFIGS[name]
    E = 12_000
    src, dst, ts, neg = make_events(cfg, 0, E)
    rng = np.random.default_rng(3)
    n = 600
    roots = rng.integers(0, cfg.num_nodes, n).astype(np.int32)
    # hot nodes too: take endpoints of events
    roots[: n // 2] = src[rng.integers(0, E, n // 2)]
    qts = ts[rng.integers(0, E, n)] + rng.integers(0, 2, n)  # exact ties and between-tick queries
    g = oracle.Graph(cfg.num_nodes, src, dst, ts)
    for fanout in (1, 3, 10):
        a = oracle.sample_brute(src, dst, ts, roots, qts, fanout)
        b = g.sample(roots, qts, fanout)
        for key in ("nbr", "eid", "ts", "dt", "cnt"):
            assert np.array_equal(a[key], b[key]), (fanout, key)
        valid = a["eid"] >= 0
        assert (a["ts"][valid] < np.repeat(qts[:, None], fanout, 1)[valid]).all()  # causality S:L119
        prior = np.array([np.sum(((src == r) | (dst == r)) & (ts < t)) for r, t in zip(roots, qts)])
        assert np.array_equal(a["cnt"], np.minimum(prior, fanout))
    for i in range(0, n, 37):
        ref = _brute_py(src, dst, ts, roots[i], qts[i], 10)
        assert [(int(x), int(e)) for x, e in zip(a["nbr"][i], a["eid"][i]) if e >= 0] == ref


# ---------------------------------------------------------------- P2 dedup / write-back
def test_p2_dedup_equals_last_occurrence():
    rng = np.random.default_rng(0)
    for trial in range(20):
        N = int(rng.integers(1, 30))
        B = int(rng.integers(1, 200))
        s = rng.integers(0, N, B).astype(np.int32)
        d = rng.integers(0, N, B).astype(np.int32)
        nodes, win = oracle.dedup(N, s, d)
        last = {}
        for a in range(B):
            last[int(s[a])] = 2 * a
            last[int(d[a])] = 2 * a + 1
        ref = sorted(last.items(), key=lambda kv: kv[1])
        assert [n for n, _ in ref] == nodes.tolist()
        assert [p for _, p in ref] == win.tolist()
        assert len(set(nodes.tolist())) == len(nodes)


@pytest.mark.parametrize("k,schedule", [(0, "exact"), (2, "exact"), (1, "grouped")])
def test_p2_final_mem_ts_is_last_event(k, schedule):
    cfg = CONFIGS["tiny"]
    src, dst, ts, _ = make_events(cfg, 0, 3000)
    ef = edge_features(0, 0, 3000, cfg.edge_dim)
    p = gru_params(cfg.mem_dim, cfg.mail_dim, cfg.time_dim)
    st, vers = oracle.run_stream(cfg.num_nodes, src, dst, ts, ef, p, cfg.batch, k, schedule)
    last = np.zeros(cfg.num_nodes)
    for j in range(len(src)):
        last[src[j]] = ts[j]
        last[dst[j]] = ts[j]
    assert np.array_equal(st["mem_ts"], last)
    assert np.array_equal(st["mail_ts"], last)
    # P3 staleness bound per fetch, 1-based iterations
    i = np.arange(1, len(vers) + 1)
    assert ((i - 1 - k <= vers) & (vers <= i - 1)).all()
    if schedule == "exact":
        assert np.array_equal(vers, np.maximum(0, i - 1 - k))
    # |mem| <= 1 (P8): convex combination of tanh and h
    assert np.abs(st["mem"]).max() <= 1.0


def _gru_torch(x, h, p):
    cell = torch.nn.GRUCell(x.shape[1], h.shape[1]).double()
    with torch.no_grad():
        cell.weight_ih.copy_(torch.from_numpy(p["w_ih"].astype(np.float64)))
        cell.weight_hh.copy_(torch.from_numpy(p["w_hh"].astype(np.float64)))
        cell.bias_ih.copy_(torch.from_numpy(p["b_ih"].astype(np.float64)))
        cell.bias_hh.copy_(torch.from_numpy(p["b_hh"].astype(np.float64)))
        return cell(torch.from_numpy(x.astype(np.float64)), torch.from_numpy(h.astype(np.float64))).numpy()


@pytest.mark.parametrize("k", [0, 1])
def test_p2_p5_last_event_value_equals_gru_cell(k):
    """Final mem[w] equals torch.nn.GRUCell(x_w, h_w) (f64, library routine) on
    w's last event, fed from the snapshot S_{v(i*)} the schedule assigns."""
    cfg = CONFIGS["tiny"]
    E, B = 2000, cfg.batch
    src, dst, ts, _ = make_events(cfg, 1, E)
    ef = edge_features(1, 0, E, cfg.edge_dim)
    p = gru_params(cfg.mem_dim, cfg.mail_dim, cfg.time_dim)
    st, _ = oracle.run_stream(cfg.num_nodes, src, dst, ts, ef, p, B, k)
    nb = E // B
    i_last = nb
    v = oracle.snapshot_version(i_last, k)
    snap, _ = oracle.run_stream(cfg.num_nodes, src, dst, ts, ef, p, B, k, max_batches=v)
    sl = slice((i_last - 1) * B, i_last * B)
    out = oracle.memory_update(cfg.num_nodes, src[sl], dst[sl], ts[sl], ef[sl], p, snap["mem"], snap["mem_ts"])
    M = cfg.mem_dim
    dt = (ts[sl][out["winner"] >> 1] - snap["mem_ts"][out["nodes"]]).astype(np.float32)
    enc = np.cos(np.float64(np.float32(p["time_w"][None, :] * dt[:, None]))).astype(np.float32)  # φ = 0
    x = np.concatenate([out["mail"], enc], axis=1)
    h = snap["mem"][out["nodes"]]
    ref = _gru_torch(x, h, p)
    assert np.allclose(out["mem"], ref, rtol=0, atol=2e-7)
    assert np.array_equal(st["mem"][out["nodes"]], out["mem"])
    # mail blocks are the snapshot rows of w and the other endpoint, then ef (G14)
    a = out["winner"] >> 1
    other = np.where(out["winner"] % 2 == 0, dst[sl][a], src[sl][a])
    assert np.array_equal(out["mail"][:, :M], snap["mem"][out["nodes"]])
    assert np.array_equal(out["mail"][:, M:2 * M], snap["mem"][other])
    assert np.array_equal(out["mail"][:, 2 * M:], ef[sl][a])


# ---------------------------------------------------------------- P3 k=0 == sequential
def test_p3_k0_batch1_equals_sequential_tgn():
    """k = 0, B = 1 is plain sequential TGN, Eq. (1) per event,
    here as a straight-line loop with torch.nn.GRUCell in f64."""
    E, N, M, He, Dt = 150, 40, 8, 5, 6
    rng = np.random.default_rng(4)
    src = rng.integers(0, N, E).astype(np.int32)
    dst = rng.integers(0, N, E).astype(np.int32)
    ts = np.floor(np.cumsum(rng.exponential(2.0, E)))
    ef = edge_features(2, 0, E, He)
    p = gru_params(M, 2 * M + He, Dt, seed=9)
    st, _ = oracle.run_stream(N, src, dst, ts, ef, p, 1, 0)
    mem = np.zeros((N, M), np.float32)
    mts = np.zeros(N)
    for j in range(E):
        u, v = int(src[j]), int(dst[j])
        new = {}
        for w, o in ((u, v), (v, u)):
            dt = np.float32(ts[j] - mts[w])
            enc = np.cos(np.float64(np.float32(p["time_w"] * dt) + p["time_b"])).astype(np.float32)
            x = np.concatenate([mem[w], mem[o], ef[j], enc])[None]
            new[w] = _gru_torch(x, mem[w][None], p)[0].astype(np.float32)
        for w, val in new.items():  # dst's message wins for a self-loop: identical anyway
            mem[w] = val
            mts[w] = ts[j]
    assert np.allclose(st["mem"], mem, rtol=0, atol=1e-6)
    assert np.array_equal(st["mem_ts"], mts)


# ---------------------------------------------------------------- P4 bias-only closed form
@pytest.mark.parametrize("k,schedule", [(0, "exact"), (1, "exact"), (3, "exact"), (2, "grouped")])
def test_p4_bias_only_closed_form(k, schedule):
    """mem[w] = tanh(c)(1 - 2^-m_w), m_w an integer replay of the schedule:
    m_w <- m_w(snapshot) + 1 at each commit touching w."""
    cfg = CONFIGS["tiny"]
    E, B, N = 4000, 200, cfg.num_nodes
    src, dst, ts, _ = make_events(cfg, 2, E)
    M, He, Dt, c = 6, 4, 3, 0.9
    p = _bias_only(M, He, Dt, c)
    ef = edge_features(0, 0, E, He)
    st, vers = oracle.run_stream(N, src, dst, ts, ef, p, B, k, schedule)
    hist = [np.zeros(N, np.int64)]
    for i in range(1, E // B + 1):
        v = oracle.snapshot_version(i, k, schedule)
        snap = hist[v]
        live = hist[-1].copy()
        for a in range((i - 1) * B, i * B):
            for w in (src[a], dst[a]):
                live[w] = snap[w] + 1
        hist.append(live)
    want = math.tanh(c) * (1.0 - 2.0 ** (-hist[-1].astype(np.float64)))
    assert np.allclose(st["mem"], want[:, None], rtol=0, atol=3e-7)


# ---------------------------------------------------------------- F1 plan mode (per-iteration k_i)
@pytest.mark.parametrize("plan_k,key", [(1, "k0_exact"), (2, "k1_exact")])
def test_plan_worked_example_constant_plans(plan_k, key):
    """Plan mode with a constant paper staleness k_i: "k=1 represents the
    baseline method of TGL without applying staleness", so k_i = 1 is
    the build-k 0 run and k_i = 2 the build-k 1 run of the hand-worked example
    (C.5 values, golden/worked_example.json)."""
    g = _load("worked_example.json")
    ev = g["events"]
    exp = g["bias_only_units_of_tanh_c"][key]
    M, He, Dt, c = 4, 3, 2, 0.7
    ef = edge_features(0, 0, 6, He)
    st, vers = oracle.run_stream(4, ev["src"], ev["dst"], ev["ts"], ef, _bias_only(M, He, Dt, c),
                                 g["batch"], plan_k - 1, plan=[plan_k] * 3)
    want = np.array(exp["mem"])[:, None] * math.tanh(c)
    assert np.allclose(st["mem"], np.broadcast_to(want, (4, M)), rtol=0, atol=2e-7)
    assert list(st["mem_ts"]) == exp["mem_ts"]
    # Alg. 1 gate: iteration i reads the memory updated through i - k_i
    assert list(vers) == [max(0, i - plan_k) for i in (1, 2, 3)]


@pytest.mark.parametrize("kk", [0, 1, 3])
def test_plan_constant_equals_exact_schedule_bitwise(kk):
    """k_i = k + 1 for every i reads v(i) = max(0, i - 1 - k), the exact
    schedule of build staleness k (G8): the whole state must be the
    same bits with random GRU weights (not only in the closed form)."""
    cfg = CONFIGS["tiny"]
    E, B = 3000, cfg.batch
    src, dst, ts, _ = make_events(cfg, 5, E)
    ef = edge_features(5, 0, E, cfg.edge_dim)
    p = gru_params(cfg.mem_dim, cfg.mail_dim, cfg.time_dim)
    nb = -(-E // B)
    a, va = oracle.run_stream(cfg.num_nodes, src, dst, ts, ef, p, B, kk, "exact")
    b, vb = oracle.run_stream(cfg.num_nodes, src, dst, ts, ef, p, B, kk, plan=[kk + 1] * nb)
    assert np.array_equal(va, vb)
    for key in ("mem", "mem_ts", "mail", "mail_ts"):
        assert np.array_equal(a[key], b[key]), key


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_plan_bias_only_closed_form_random_plans(seed):
    """P4 for plan mode: mem[w] = tanh(c)(1 - 2^-m_w), the integer replay run
    with v(i) = max(0, i - k_i) written out here from Alg. 1's gate
    (P:L844-L847), for random plans with 1 <= k_i <= 4."""
    cfg = CONFIGS["tiny"]
    E, B, N = 4000, 200, cfg.num_nodes
    src, dst, ts, _ = make_events(cfg, 7 + seed, E)
    M, He, Dt, c = 6, 4, 3, 0.9
    prm = _bias_only(M, He, Dt, c)
    ef = edge_features(0, 0, E, He)
    nb = E // B
    rng = np.random.default_rng(seed)
    plan = rng.integers(1, 5, nb).astype(np.int32)
    kmax = int(max(i - max(0, i - int(plan[i - 1])) for i in range(1, nb + 1))) - 1
    st, vers = oracle.run_stream(N, src, dst, ts, ef, prm, B, kmax, plan=plan)
    hist = [np.zeros(N, np.int64)]
    for i in range(1, nb + 1):
        v = max(0, i - int(plan[i - 1]))
        assert vers[i - 1] == v
        snap = hist[v]
        live = hist[-1].copy()
        for a in range((i - 1) * B, i * B):
            for w in (src[a], dst[a]):
                live[w] = snap[w] + 1
        hist.append(live)
    want = math.tanh(c) * (1.0 - 2.0 ** (-hist[-1].astype(np.float64)))
    assert np.allclose(st["mem"], want[:, None], rtol=0, atol=3e-7)


# ---------------------------------------------------------------- P6 message blocks
@pytest.mark.parametrize("block", ["self", "other", "edge"])
def test_p6_message_block_closed_forms(block):
    """W_ih nonzero on exactly one block (identity on its first columns), zero
    biases: r = z = 1/2 and n_j = tanh(block_j), so h' = (tanh(block_j) + h_j)/2."""
    N, M, He, Dt = 12, 4, 6, 3
    Dx = 2 * M + He + Dt
    rng = np.random.default_rng(5)
    p = _bias_only(M, He, Dt, 0.0)
    off = {"self": 0, "other": M, "edge": 2 * M}[block]
    for j in range(M):
        p["w_ih"][2 * M + j, off + j] = 1.0
    mem = rng.uniform(-1, 1, (N, M)).astype(np.float32)
    mts = np.zeros(N)
    src = np.array([0, 3, 5], np.int32)
    dst = np.array([1, 4, 0], np.int32)
    ts = np.array([2.0, 3.0, 4.0])
    ef = rng.uniform(-1, 1, (3, He)).astype(np.float32)
    out = oracle.memory_update(N, src, dst, ts, ef, p, mem, mts)
    for w, pw, hw in zip(out["nodes"], out["winner"], out["mem"]):
        a = pw >> 1
        o = dst[a] if pw % 2 == 0 else src[a]
        blk = {"self": mem[w], "other": mem[o], "edge": ef[a][:M]}[block]
        assert np.allclose(hw, 0.5 * np.tanh(blk.astype(np.float64)) + 0.5 * mem[w], atol=1e-7)


def test_p6_time_block_dt_zero_is_all_ones():
    """enc(0) = cos(φ) = 1 for φ = 0: time-only n-gate rows summing
    the Dt columns give n = tanh(Dt * 1 / Dt) = tanh(1)."""
    N, M, He, Dt = 5, 3, 2, 7
    p = _bias_only(M, He, Dt, 0.0)
    p["w_ih"][2 * M:, 2 * M + He:] = 1.0 / Dt
    mem = np.zeros((N, M), np.float32)
    out = oracle.memory_update(N, np.array([1], np.int32), np.array([2], np.int32), np.array([0.0]),
                               np.zeros((1, He), np.float32), p, mem, np.zeros(N))
    assert np.allclose(out["mem"], 0.5 * math.tanh(1.0), atol=1e-7)


# ---------------------------------------------------------------- P7 mitigation
def _omega_exhaustive(src, dst, ts, w, tstar, mem_ts, gamma, n_sim, fanout):
    """Ω by exhaustive enumeration over ALL nodes, with set intersections built
    from the brute-force sampler (pinned by P1)."""
    def nb(v):
        s = oracle.sample_brute(src, dst, ts, [v], [tstar], fanout)
        return {int(x) for x in s["nbr"][0] if x >= 0}
    n1 = nb(w) - {w}
    scored = []
    for u in range(len(mem_ts)):
        if u == w:
            continue
        c = sum(1 for x in n1 if u in nb(x))
        if c > 0 and mem_ts[u] > mem_ts[w] and tstar - mem_ts[u] < gamma:
            scored.append((-c, -mem_ts[u], u))
    scored.sort()
    return [u for _, _, u in scored[:n_sim]]


def test_p7_mitigation_ranking_exhaustive():
    rng = np.random.default_rng(11)
    N, E = 25, 400
    src = rng.integers(0, N, E).astype(np.int32)
    dst = rng.integers(0, N, E).astype(np.int32)
    ts = np.floor(np.cumsum(rng.exponential(1.0, E)))
    g = oracle.Graph(N, src, dst, ts)
    M = 4
    mem = rng.uniform(-1, 1, (N, M)).astype(np.float32)
    checked = 0
    for trial in range(40):
        tstar = float(ts[rng.integers(50, E)])
        mem_ts = np.where(rng.random(N) < 0.8, tstar - rng.integers(0, 30, N), 0).astype(np.float64)
        mem_ts = np.minimum(mem_ts, tstar)
        ids = np.arange(N, dtype=np.int32)
        gamma = float(rng.integers(3, 15))
        out = g.mitigate(ids, np.full(N, tstar), mem, mem_ts, 0.5, gamma, 3, 4)
        for w in range(N):
            el = tstar - mem_ts[w] > gamma
            assert out["elig"][w] == el
            if not el:
                assert (out["omega"][w] == -1).all()
                assert np.array_equal(out["h"][w], mem[w])
                continue
            om = _omega_exhaustive(src, dst, ts, w, tstar, mem_ts, gamma, 3, 4)
            got = [int(x) for x in out["omega"][w] if x >= 0]
            assert got == om, (trial, w)
            if om:
                checked += 1
                want = 0.5 * mem[w].astype(np.float64) + 0.5 * mem[om].astype(np.float64).mean(0)
                assert np.allclose(out["h"][w], want, atol=1e-7)
                assert (np.minimum(mem[w], mem[om].min(0)) - 1e-7 <= out["h"][w]).all()  # convexity S:L241
                assert (out["h"][w] <= np.maximum(mem[w], mem[om].max(0)) + 1e-7).all()
    assert checked > 10


def _two_node_omega_graph():
    # w = 0 is stale; x = 1 is its neighbour; u = 2 is x's other neighbour (fresh)
    src = np.array([0, 1], np.int32)
    dst = np.array([1, 2], np.int32)
    ts = np.array([1.0, 2.0])
    return src, dst, ts


@pytest.mark.parametrize("lam,want", [(1.0, [1.0, 0.0]), (0.5, [0.5, 1.0]), (0.0, [0.0, 2.0])])
def test_p7_lambda_identities(lam, want):
    """λ=1 -> ŝ = s (P:L554 'reverts to standard MSPipe'); λ=0.5, s=[1,0],
    mean=[0,2] -> [0.5,1]; λ=0 -> the mean."""
    src, dst, ts = _two_node_omega_graph()
    g = oracle.Graph(3, src, dst, ts)
    mem = np.array([[1, 0], [0, 0], [0, 2]], np.float32)
    mem_ts = np.array([0.0, 0.0, 9.0])
    out = g.mitigate([0], [10.0], mem, mem_ts, lam, 5.0, 5, 10)
    assert out["elig"][0] and out["omega"][0].tolist()[:1] == [2]
    assert out["h"][0].tolist() == want


def test_p7_lambda_one_run_equals_mitigation_off():
    """Whole-stream: λ = 1 is bitwise equal to mitigation off."""
    cfg = CONFIGS["tiny"]
    E = 2000
    src, dst, ts, _ = make_events(cfg, 3, E)
    ef = edge_features(3, 0, E, cfg.edge_dim)
    p = gru_params(cfg.mem_dim, cfg.mail_dim, cfg.time_dim)
    a, _ = oracle.run_stream(cfg.num_nodes, src, dst, ts, ef, p, 200, 1)
    b, _ = oracle.run_stream(cfg.num_nodes, src, dst, ts, ef, p, 200, 1,
                             mitigation=dict(lam=1.0, gamma=5.0, n_sim=5))
    for key in a:
        assert np.array_equal(a[key], b[key])


# ---------------------------------------------------------------- P9 sizing, P12 quantile
def test_p9_memory_overhead_upperbound_row():
    g = _load("memory_overhead_upperbound.json")
    for r in g["rows"]:
        mb = oracle.memory_overhead_bound(r["K"], r["B"], 10, r["Hn"], r["He"], 100) / 1e6
        # printed to 3 significant digits; MOOC/LastFM print 44.3 where the formula gives 44.43
        # (a last-digit slip in the paper, recorded in DESIGN.md) -> 0.5 % relative
        assert abs(mb - r["printed_MB"]) <= 0.005 * r["printed_MB"], r


def test_p12_quantile_nearest_rank_equals_numpy_inverted_cdf():
    rng = np.random.default_rng(0)
    for n in (1, 2, 7, 100, 10_000):
        x = (rng.pareto(1.5, n) * 10).round()
        for p in (0.5, 0.9, 0.99, 1.0):
            assert oracle.quantile_nearest_rank(x, p) == np.quantile(x, p, method="inverted_cdf")
    assert oracle.quantile_nearest_rank(np.full(10, 5.0), 0.3) == 5.0


def test_p12_delta_t_population_and_heavy_tail():
    src = np.array([0, 1, 0, 2, 2], np.int32)
    dst = np.array([1, 1, 2, 2, 0], np.int32)
    ts = np.array([1.0, 4.0, 6.0, 7.0, 9.0])
    # gaps: e1 node1 (4-1=3, self-loop once); e2 node0 (5), node2 first; e3 node2 (1, self-loop);
    # e4 node2 (2), node0 (3)
    assert sorted(oracle.delta_t_population(3, src, dst, ts).tolist()) == [1, 2, 3, 3, 5]
    cfg = CONFIGS["wiki"]
    s, d, t, _ = make_events(cfg, 0)
    pop = oracle.delta_t_population(cfg.num_nodes, s, d, t)
    med = oracle.quantile_nearest_rank(pop, 0.5)
    assert oracle.quantile_nearest_rank(pop, 0.99) / max(med, 1.0) > 10  # S:L115 heavy tail


# ------------------------------------------------------------------ row F2
def test_f2_feature_fetch_closed_form():
    """Rows whose values encode their own index (table[i, c] = 1000 i + c): every
    fetched row must read back as 1000 * id + c, pads as zeros."""
    from oracle.features import feature_fetch
    rng = np.random.default_rng(0)
    N, E, Hn, He = 50, 300, 7, 5
    nfeat = (1000.0 * np.arange(N)[:, None] + np.arange(Hn)[None, :]).astype(np.float32)
    efeat = (1000.0 * np.arange(E)[:, None] + np.arange(He)[None, :]).astype(np.float32)
    sub = rng.integers(-1, N, (12, 4))
    eid = rng.integers(-1, E, (12, 3))
    on, oe = feature_fetch(sub, eid, nfeat, efeat)
    for (r, s), v in np.ndenumerate(sub):
        want = np.zeros(Hn) if v < 0 else 1000.0 * v + np.arange(Hn)
        assert np.array_equal(on[r, s], want)
    for (r, s), v in np.ndenumerate(eid):
        want = np.zeros(He) if v < 0 else 1000.0 * v + np.arange(He)
        assert np.array_equal(oe[r, s], want)
    assert feature_fetch(sub, eid)[0] is None


# ------------------------------------------------------------------ row F3
def test_f3_rnn_cell_matches_torch_rnncell():
    """cell="rnn": h' = tanh(W_ih x + b_ih + W_hh h + b_hh) == torch.nn.RNNCell (f64)."""
    import torch
    from synth import rnn_params
    rng = np.random.default_rng(3)
    N, M, He, Dt, B = 40, 8, 6, 4, 10
    p = rnn_params(M, 2 * M + He, Dt, seed=5)
    src, dst = rng.integers(0, N, B).astype(np.int32), rng.integers(0, N, B).astype(np.int32)
    ts = np.sort(rng.uniform(10, 20, B))
    ef = rng.uniform(-1, 1, (B, He)).astype(np.float32)
    mem = rng.uniform(-1, 1, (N, M)).astype(np.float32)
    mem_ts = rng.uniform(0, 9, N)
    out = oracle.memory_update(N, src, dst, ts, ef, p, mem, mem_ts, cell="rnn")
    cell = torch.nn.RNNCell(2 * M + He + Dt, M).double()
    with torch.no_grad():
        for name in ("w_ih", "w_hh", "b_ih", "b_hh"):
            getattr(cell, {"w_ih": "weight_ih", "w_hh": "weight_hh", "b_ih": "bias_ih", "b_hh": "bias_hh"}[name]) \
                .copy_(torch.tensor(p[name], dtype=torch.float64))
    for u, (w, pw) in enumerate(zip(out["nodes"], out["winner"])):
        a = pw >> 1
        o = src[a] if pw & 1 else dst[a]
        dt = np.float32(ts[a] - mem_ts[w])
        arg = (p["time_w"].astype(np.float64) * np.float64(dt) + p["time_b"]).astype(np.float32)  # fmaf
        enc = np.cos(arg.astype(np.float64))
        x = np.concatenate([mem[w], mem[o], ef[a], enc.astype(np.float32)]).astype(np.float64)
        with torch.no_grad():
            want = cell(torch.tensor(x)[None], torch.tensor(mem[w], dtype=torch.float64)[None])[0].numpy()
        assert np.allclose(out["mem"][u], want, rtol=0, atol=2e-7)


def _selector_rnn(M, He, Dt):
    """RNN weights that copy the edge-feature part of x: h'[m] = tanh(x[2M + m])."""
    Dx = 2 * M + He + Dt
    w_ih = np.zeros((M, Dx), np.float32)
    for m in range(min(M, He)):
        w_ih[m, 2 * M + m] = 1.0
    return dict(w_ih=w_ih, w_hh=np.zeros((M, M), np.float32), b_ih=np.zeros(M, np.float32),
                b_hh=np.zeros(M, np.float32), time_w=np.ones(Dt, np.float32), time_b=np.zeros(Dt, np.float32))


@pytest.mark.parametrize("k", [0, 2])
def test_f3_deferred_mailbox_closed_form(k):
    """Edge-feature selector RNN: with the IMMEDIATE mailbox a node's memory is
    tanh(e) of its winning event in its last batch; with the DEFERRED mailbox
    (TGL) it is tanh(e) of its winning event in the latest batch <= v(i) that
    contained it before its last batch i (the stored mail), and 0 when there was
    none.  Integer replay of the batches only; no GRU/GEMM code."""
    rng = np.random.default_rng(7 + k)
    N, M, He, Dt, B, E = 12, 4, 6, 2, 5, 120
    src, dst = rng.integers(0, N, E).astype(np.int32), rng.integers(0, N, E).astype(np.int32)
    ts = np.arange(E, dtype=np.float64)
    ef = rng.uniform(-1, 1, (E, He)).astype(np.float32)
    p = _selector_rnn(M, He, Dt)
    nb = E // B
    win = {}  # (batch, node) -> winning event (most recent pair in the batch)
    for i in range(1, nb + 1):
        for a in range((i - 1) * B, i * B):
            win[(i, int(src[a]))] = a
            win[(i, int(dst[a]))] = a
    for mailbox in ("immediate", "deferred"):
        st, _ = oracle.run_stream(N, src, dst, ts, ef, p, B, k, mailbox=mailbox, cell="rnn")
        for v in range(N):
            batches = [i for i in range(1, nb + 1) if (i, v) in win]
            if not batches:
                assert (st["mem"][v] == 0).all()
                continue
            last = batches[-1]
            if mailbox == "immediate":
                e = ef[win[(last, v)]]
            else:
                vi = max(0, last - 1 - k)  # the version batch `last` reads
                prev = [i for i in batches if i <= vi]
                e = ef[win[(prev[-1], v)]] if prev else np.zeros(He, np.float32)
            assert np.allclose(st["mem"][v], np.tanh(e[:M].astype(np.float64)), rtol=0, atol=1e-7), (mailbox, v)


def test_f3_deferred_with_input_weights_zero_equals_immediate():
    """W_ih = 0: the message (hence the mailbox form) cannot matter — bitwise equal."""
    from synth import gru_params
    rng = np.random.default_rng(1)
    N, M, He, Dt, B, E = 30, 8, 6, 4, 7, 200
    src, dst = rng.integers(0, N, E).astype(np.int32), rng.integers(0, N, E).astype(np.int32)
    ts = np.cumsum(rng.uniform(0, 1, E))
    ef = rng.uniform(-1, 1, (E, He)).astype(np.float32)
    p = gru_params(M, 2 * M + He, Dt)
    p["w_ih"] = np.zeros_like(p["w_ih"])
    a, _ = oracle.run_stream(N, src, dst, ts, ef, p, B, 1)
    b, _ = oracle.run_stream(N, src, dst, ts, ef, p, B, 1, mailbox="deferred")
    assert np.array_equal(a["mem"], b["mem"]) and np.array_equal(a["mem_ts"], b["mem_ts"])


def test_f3_deferred_mail_is_post_update_memory():
    """Deferred mailbox invariant: a node's stored mail starts with its own
    post-update memory of the same batch, i.e. mail[w][:M] == mem[w]."""
    from synth import gru_params
    rng = np.random.default_rng(2)
    N, M, He, Dt, B, E = 25, 8, 6, 4, 9, 300
    src, dst = rng.integers(0, N, E).astype(np.int32), rng.integers(0, N, E).astype(np.int32)
    ts = np.cumsum(rng.uniform(0, 1, E))
    ef = rng.uniform(-1, 1, (E, He)).astype(np.float32)
    st, _ = oracle.run_stream(N, src, dst, ts, ef, gru_params(M, 2 * M + He, Dt), B, 1, mailbox="deferred")
    touched = np.unique(np.concatenate([src, dst]))
    assert np.array_equal(st["mail"][touched, :M], st["mem"][touched])
    assert np.array_equal(st["mail_ts"][touched], st["mem_ts"][touched])

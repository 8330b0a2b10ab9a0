"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Bit-exact for ids, counts, winners, timestamps, Ω,
eligibility and copied rows; values within the north-star tolerance
|g - o| <= 1e-4 |o| + 1e-6 (fp32, teacher-forced).  Expected values come
from oracle/ only."""
import numpy as np
import pytest
import torch

import oracle
from paper_2402_15113_b200 import MemoryStage, StageConfig, _C, build_tcsr
from synth import CONFIGS, edge_features, gru_params, make_events, make_workload

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-4, 1e-6


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    d = torch.device("cuda:0")
    torch.cuda.set_device(d)
    return d


def _close(g, o, rtol=RTOL, atol=ATOL):
    g = np.asarray(g, np.float64)
    o = np.asarray(o, np.float64)
    bad = np.abs(g - o) > rtol * np.abs(o) + atol
    return not bad.any(), float(np.abs(g - o).max(initial=0.0))


def _t(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


# ------------------------------------------------------------------ A1 sampler
@pytest.mark.parametrize("name,E", [("tiny", None), ("wiki", None), ("lastfm", 300_000), ("reddit", 200_000)])
def test_sampler_batch_bit_exact(dev, name, E):
    cfg = CONFIGS[name]
    src, dst, ts, neg = make_events(cfg, 0, E)
    g = build_tcsr(cfg.num_nodes, src, dst, ts, dev)
    og = oracle.Graph(cfg.num_nodes, src, dst, ts)
    B, F = cfg.batch, cfg.fanout
    nb = -(-len(src) // B)
    rng = np.random.default_rng(1)
    picks = sorted(set([1, 2, nb] + rng.integers(1, nb + 1, 12).tolist()))
    for i in picks:
        j0, j1 = (i - 1) * B, min(i * B, len(src))
        n = j1 - j0
        out = _C.alloc_sample(3 * n, F, dev)
        _C.sample_batch(g, _t(src[j0:j1], dev), _t(dst[j0:j1], dev), _t(neg[j0:j1], dev), _t(ts[j0:j1], dev), F, out)
        roots = np.concatenate([src[j0:j1], dst[j0:j1], neg[j0:j1]])
        qts = np.concatenate([ts[j0:j1]] * 3)
        ref = og.sample(roots, qts, F)
        for key in ("nbr", "eid", "ts", "dt", "cnt"):
            assert np.array_equal(out[key].cpu().numpy(), ref[key]), (i, key)
        sub = out["sub"].cpu().numpy()
        assert np.array_equal(sub[:, 0], roots)
        assert np.array_equal(sub[:, 1:], ref["nbr"])
    _C.check()


@pytest.mark.parametrize("fanout", [1, 3, 10, 17, 64])
def test_sampler_recent_arbitrary_queries(dev, fanout):
    cfg = CONFIGS["lastfm"]
    src, dst, ts, _ = make_events(cfg, 2, 100_000)
    g = build_tcsr(cfg.num_nodes, src, dst, ts, dev)
    rng = np.random.default_rng(fanout)
    n = 5003  # ragged tail over 32-root warps
    roots = rng.integers(0, cfg.num_nodes, n).astype(np.int32)
    qts = ts[rng.integers(0, len(ts), n)] + rng.integers(-1, 2, n)
    qts[:5] = [0.0, -1.0, ts[-1] + 10, ts[0], ts[len(ts) // 2]]
    out = _C.alloc_sample(n, fanout, dev)
    _C.sample_recent(g, _t(roots, dev), _t(qts, dev), fanout, out)
    ref = oracle.sample_brute(src, dst, ts, roots[:300], qts[:300], fanout)  # the definition
    ref2 = oracle.Graph(cfg.num_nodes, src, dst, ts).sample(roots, qts, fanout)
    for key in ("nbr", "eid", "ts", "dt", "cnt"):
        got = out[key].cpu().numpy()
        assert np.array_equal(got[:300], ref[key]), key
        assert np.array_equal(got, ref2[key]), key
    _C.check()


def test_sampler_edge_cases(dev):
    src = np.array([0, 1, 2, 2], np.int32)
    dst = np.array([1, 1, 2, 0], np.int32)  # self-loops (1,1), (2,2)
    ts = np.array([1.0, 2.0, 2.0, 3.0])
    g = build_tcsr(5, src, dst, ts, dev)
    empty = _C.alloc_sample(0, 4, dev)
    _C.sample_recent(g, torch.empty(0, dtype=torch.int32, device=dev), torch.empty(0, dtype=torch.float64, device=dev), 4, empty)
    roots = np.array([1, 2, 4, 0], np.int32)
    qts = np.array([5.0, 5.0, 5.0, 1.0])
    out = _C.alloc_sample(4, 4, dev)
    _C.sample_recent(g, _t(roots, dev), _t(qts, dev), 4, out)
    ref = oracle.sample_brute(src, dst, ts, roots, qts, 4)
    for key in ("nbr", "eid", "ts", "dt", "cnt"):
        assert np.array_equal(out[key].cpu().numpy(), ref[key]), key
    assert out["cnt"].cpu().tolist() == [2, 2, 0, 0]  # self-loop once; isolated node; strict ts < t_q
    _C.check()
    bad = _C.alloc_sample(1, 4, dev)
    _C.sample_recent(g, _t(np.array([7], np.int32), dev), _t(np.array([1.0]), dev), 4, bad)
    with pytest.raises(_C.MspipeError) as e:
        _C.check()
    assert e.value.status == _C.ERANGE
    assert bad["cnt"].item() == 0


# ------------------------------------------------------------------ A2-A6 teacher-forced
def _random_state(num_nodes, M, src, dst, ts, j0, seed):
    """Seeded synthetic snapshot: random memory rows; mem_ts = time of each
    node's last event before the batch (0 if none), as a real trajectory has."""
    rng = np.random.default_rng(seed)
    mem = rng.uniform(-1, 1, (num_nodes, M)).astype(np.float32)
    mem_ts = np.zeros(num_nodes)
    mem_ts[src[:j0]] = ts[:j0]  # numpy fancy assignment keeps the last write
    last_dst = np.zeros(num_nodes)
    last_dst[dst[:j0]] = ts[:j0]
    return mem, np.maximum(mem_ts, last_dst)


def _teacher_forced(dev, name, i, mitigation=None, seed=0, E=None, precision=_C.FP32_3XTF32, fused=False):
    cfg = CONFIGS[name]
    src, dst, ts, neg = make_events(cfg, seed, E)
    B, F, M = cfg.batch, cfg.fanout, cfg.mem_dim
    j0, j1 = (i - 1) * B, min(i * B, len(src))
    ef = edge_features(seed, j0, j1 - j0, cfg.edge_dim)
    params = gru_params(M, cfg.mail_dim, cfg.time_dim)
    mem, mem_ts = _random_state(cfg.num_nodes, M, src, dst, ts, j0, seed + i)
    g = build_tcsr(cfg.num_nodes, src, dst, ts, dev)
    sc = StageConfig(cfg.num_nodes, M, cfg.edge_dim, cfg.time_dim, F, B, 0, mitigation=mitigation,
                     precision=precision, fused=fused)
    st = MemoryStage(sc, params, g, dev)
    st.memory.mem.copy_(_t(mem, dev))
    st.memory.mem_ts.copy_(_t(mem_ts, dev))
    x = {k: _t(v[j0:j1], dev) for k, v in dict(src=src, dst=dst, ts=ts, neg=neg).items()}
    x["ef"] = _t(ef, dev)
    st.bind_resident(x["src"], x["dst"], x["ts"], x["neg"], x["ef"])
    st.prep(1)
    sl = st.slots[0]
    n = j1 - j0
    upd = st._upd(1)  # winners from prep's dedup + the update outputs
    if fused:  # mspipe_memory_prep + mspipe_message_build ran in prep(1); mspipe_gru_apply here
        st.update(1)
    else:
        _C.memory_update(st.memory, st.gru, x["src"], x["dst"], x["ts"], x["ef"], sl.mem, sl.mem_ts, F + 1, upd,
                         snap_h=sl.h[: 2 * n] if sl.h is not None else None)
    torch.cuda.synchronize()
    _C.check()
    og = oracle.Graph(cfg.num_nodes, src, dst, ts) if mitigation else None
    ref = oracle.memory_update(cfg.num_nodes, src[j0:j1], dst[j0:j1], ts[j0:j1], ef, params, mem, mem_ts,
                               mitigation=mitigation, graph=og, fanout=F)
    return st, sl, upd, ref, (src[j0:j1], dst[j0:j1], ts[j0:j1], neg[j0:j1]), (mem, mem_ts)


@pytest.mark.parametrize("name,i,E", [("tiny", 1, None), ("tiny", 50, None), ("wiki", 137, None),
                                      ("lastfm", 400, 300_000), ("gdelt", 3, 20_000)])
@pytest.mark.parametrize("precision,fused", [(_C.FP32_3XTF32, True), (_C.FP32_3XTF32, False),
                                             (_C.FP32_SIMT, False)])
def test_update_teacher_forced(dev, name, i, E, precision, fused):
    st, sl, upd, ref, ev, (mem, mem_ts) = _teacher_forced(dev, name, i, E=E, precision=precision, fused=fused)
    U = int(upd["num"].item())
    # A1 outputs of the prep (fused or separate sampler) against the oracle sampler
    cfg = CONFIGS[name]
    roots = np.concatenate([ev[0], ev[1], ev[3]])
    sref = oracle.Graph(cfg.num_nodes, *make_events(cfg, 0, E)[:3]).sample(roots, np.concatenate([ev[2]] * 3),
                                                                           cfg.fanout)
    n3 = len(roots)
    for key in ("nbr", "eid", "ts", "dt", "cnt"):
        assert np.array_equal(sl.samp[key][:n3].cpu().numpy(), sref[key]), key
    assert U == len(ref["nodes"])
    assert np.array_equal(upd["nodes"][:U].cpu().numpy(), ref["nodes"])
    assert np.array_equal(upd["winner"][:U].cpu().numpy(), ref["winner"])
    assert np.array_equal(upd["ts"][:U].cpu().numpy(), ref["ts"])
    Dm = ref["mail"].shape[1]
    mail = upd["mail"][:U].cpu().numpy()
    assert np.array_equal(mail[:, :Dm], ref["mail"])  # copies of snapshot rows + ef
    assert (mail[:, Dm:] == 0).all()
    g64, o64 = upd["mem"][:U].cpu().numpy().astype(np.float64), ref["mem"].astype(np.float64)
    print(f"{name} i={i} fused={fused}: h' max abs err {np.abs(g64 - o64).max():.3g}, "
          f"max err / (1e-4|o| + 1e-6) {(np.abs(g64 - o64) / (1e-4 * np.abs(o64) + 1e-6)).max():.3g}")
    ok, err = _close(upd["mem"][:U].cpu().numpy(), ref["mem"])
    assert ok, f"GRU mismatch max abs {err}"
    # A3 fetch: copied rows are the state rows of the subgraph ids (pads zero)
    ids = sl.samp["sub"][: 3 * len(ev[0])].reshape(-1).cpu().numpy()
    got = sl.mem[: len(ids)].cpu().numpy()
    gts = sl.mem_ts[: len(ids)].cpu().numpy()
    valid = ids >= 0
    assert np.array_equal(got[valid], mem[ids[valid]]) and (got[~valid] == 0).all()
    assert np.array_equal(gts[valid], mem_ts[ids[valid]]) and (gts[~valid] == 0).all()


@pytest.mark.parametrize("name,i,E,p", [("tiny", 30, None, 0.5), ("reddit", 200, 150_000, 0.8),
                                        ("wiki", 100, None, 0.8), ("lastfm", 90, 100_000, 0.9)])
def test_mitigation_teacher_forced(dev, name, i, E, p):
    cfg = CONFIGS[name]
    gamma = oracle.gamma(cfg.num_nodes, *make_events(cfg, 0, E)[:3], p)
    mit = dict(lam=0.95, gamma=gamma, n_sim=5)
    st, sl, upd, ref, ev, (mem, mem_ts) = _teacher_forced(dev, name, i, mitigation=mit, E=E)
    U = int(upd["num"].item())
    n = len(ev[0])
    win = ref["winner"]
    rows = np.where(win % 2 == 0, win // 2, n + win // 2)  # root-layout row of each winner
    elig = sl.elig[: 2 * n].cpu().numpy().astype(bool)[rows]
    omega = sl.omega[: 2 * n].cpu().numpy()[rows]
    h = sl.h[: 2 * n].cpu().numpy()[rows]
    assert np.array_equal(elig, ref["elig"])
    assert elig.sum() >= 3, "test should exercise eligible targets"
    assert np.array_equal(omega, ref["omega"])
    assert (ref["omega"][:, 0] >= 0).sum() >= 1, "test should exercise a non-empty Omega"
    ok, err = _close(h, ref["h"])
    assert ok, err
    ok, err = _close(upd["mem"][:U].cpu().numpy(), ref["mem"])
    assert ok, err
    # all 2B target rows against the oracle's mitigation on explicit targets
    og = oracle.Graph(CONFIGS[name].num_nodes, *make_events(CONFIGS[name], 0, E)[:3])
    ids = np.concatenate([ev[0], ev[1]])
    allref = og.mitigate(ids, np.concatenate([ev[2], ev[2]]), mem, mem_ts, 0.95, gamma, 5, CONFIGS[name].fanout)
    assert np.array_equal(sl.elig[: 2 * n].cpu().numpy().astype(bool), allref["elig"])
    assert np.array_equal(sl.omega[: 2 * n].cpu().numpy(), allref["omega"])
    ok, err = _close(sl.h[: 2 * n].cpu().numpy(), allref["h"])
    assert ok, err


def test_mitigation_lambda_one_is_identity(dev):
    mit = dict(lam=1.0, gamma=1.0, n_sim=5)
    st, sl, upd, ref, ev, (mem, _) = _teacher_forced(dev, "tiny", 30, mitigation=mit)
    n = len(ev[0])
    ids = np.concatenate([ev[0], ev[1]])
    assert np.array_equal(sl.h[: 2 * n].cpu().numpy(), mem[ids])


# ------------------------------------------------------------------ whole streams
def _stream(dev, name, k, schedule="exact", mitigation=None, E=None, seed=0, precision=_C.FP32_3XTF32):
    w = make_workload(name, seed=seed, num_events=E)
    cfg = w["cfg"]
    sc = StageConfig(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.time_dim, cfg.fanout, cfg.batch, k,
                     schedule=schedule, mitigation=mitigation, fetch_mail=True, precision=precision)
    g = build_tcsr(cfg.num_nodes, w["src"], w["dst"], w["ts"], dev)
    st = MemoryStage(sc, w["params"], g, dev)
    t = {kk: _t(w[kk], dev) for kk in ("src", "dst", "ts", "neg", "ef")}
    st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
    st.run()
    torch.cuda.synchronize()
    _C.check()
    ref, vers = oracle.run_stream(cfg.num_nodes, w["src"], w["dst"], w["ts"], w["ef"], w["params"], cfg.batch, k,
                                  schedule, mitigation=mitigation, fanout=cfg.fanout)
    return st, ref, vers, cfg


@pytest.mark.parametrize("name,k,schedule,E", [("tiny", 0, "exact", None), ("tiny", 1, "exact", None),
                                               ("tiny", 2, "grouped", None), ("wiki", 1, "exact", None),
                                               ("lastfm", 2, "exact", 120_000)])
@pytest.mark.parametrize("precision", [_C.FP32_3XTF32, _C.FP32_SIMT])
def test_stream_free_running(dev, name, k, schedule, E, precision):
    st, ref, vers, cfg = _stream(dev, name, k, schedule, E=E, precision=precision)
    assert [st.versions[i] for i in range(1, len(vers) + 1)] == vers.tolist()
    assert np.array_equal(st.memory.mem_ts.cpu().numpy(), ref["mem_ts"])
    assert np.array_equal(st.memory.mail_ts.cpu().numpy(), ref["mail_ts"])
    g = st.memory.mem.cpu().numpy().astype(np.float64)
    o = ref["mem"].astype(np.float64)
    rel = np.linalg.norm(g - o, axis=1) / np.maximum(np.linalg.norm(o, axis=1), 1e-3)
    print(f"{name} k={k} {schedule}: free-running row-rel max {rel.max():.3g} p99 {np.quantile(rel, 0.99):.3g}")
    assert rel.max() <= 1e-4
    Dm = cfg.mail_dim
    ok, err = _close(st.memory.mail.cpu().numpy()[:, :Dm], ref["mail"], rtol=1e-4, atol=1e-5)
    assert ok, err


def test_stream_mitigation_reddit_shaped(dev):
    cfg = CONFIGS["reddit"]
    E = 60_000
    src, dst, ts, _ = make_events(cfg, 0, E)
    gamma = oracle.gamma(cfg.num_nodes, src, dst, ts, 0.99)
    mit = dict(lam=0.95, gamma=gamma, n_sim=5)
    st, ref, vers, cfg = _stream(dev, "reddit", 2, mitigation=mit, E=E)
    assert np.array_equal(st.memory.mem_ts.cpu().numpy(), ref["mem_ts"])
    g = st.memory.mem.cpu().numpy().astype(np.float64)
    o = ref["mem"].astype(np.float64)
    rel = np.linalg.norm(g - o, axis=1) / np.maximum(np.linalg.norm(o, axis=1), 1e-3)
    print(f"reddit k=2 MSPipe-S: free-running row-rel max {rel.max():.3g}")
    assert rel.max() <= 1e-4


def test_bias_only_closed_form_on_gpu(dev):
    """P4 on the GPU path: W = 0, b_in = c => mem[w] = tanh(c)(1 - 2^-m_w),
    m_w from the integer replay of the same schedule (independent of the oracle)."""
    cfg = CONFIGS["tiny"]
    E, B, k = 4000, 200, 2
    src, dst, ts, neg = make_events(cfg, 5, E)
    M, He, Dt, c = cfg.mem_dim, cfg.edge_dim, cfg.time_dim, 0.9
    p = dict(w_ih=np.zeros((3 * M, 2 * M + He + Dt), np.float32), w_hh=np.zeros((3 * M, M), np.float32),
             b_ih=np.zeros(3 * M, np.float32), b_hh=np.zeros(3 * M, np.float32),
             time_w=np.ones(Dt, np.float32), time_b=np.zeros(Dt, np.float32))
    p["b_ih"][2 * M:] = c
    g = build_tcsr(cfg.num_nodes, src, dst, ts, dev)
    st = MemoryStage(StageConfig(cfg.num_nodes, M, He, Dt, 10, B, k), p, g, dev)
    ef = edge_features(5, 0, E, He)
    st.bind_resident(*(_t(a, dev) for a in (src, dst, ts, neg, ef)))
    st.run()
    hist = [np.zeros(cfg.num_nodes, np.int64)]
    for i in range(1, E // B + 1):
        snap = hist[max(0, i - 1 - k)]
        live = hist[-1].copy()
        for a in range((i - 1) * B, i * B):
            for w in (src[a], dst[a]):
                live[w] = snap[w] + 1
        hist.append(live)
    want = np.tanh(c) * (1.0 - 2.0 ** (-hist[-1].astype(np.float64)))
    ok, err = _close(st.memory.mem.cpu().numpy(), np.broadcast_to(want[:, None], (cfg.num_nodes, M)))
    assert ok, err


@pytest.mark.parametrize("k,schedule,precision,fused", [(1, "exact", _C.FP32_3XTF32, True),
                                                         (2, "exact", _C.FP32_3XTF32, True),
                                                         (2, "grouped", _C.FP32_3XTF32, True),
                                                         (1, "exact", _C.FP32_3XTF32, False),
                                                         (3, "exact", _C.FP32_SIMT, False)])
def test_double_buffered_state_equals_single(dev, k, schedule, precision, fused):
    """Two table sets (commit t and fetch t+k on different tables, no wait
    between them) give bit-identical state and fetched snapshots to one set."""
    w = make_workload("lastfm", seed=4, num_events=40_000)  # hot nodes: rows rewritten every batch
    cfg = w["cfg"]
    res = []
    for db in (False, True):
        sc = StageConfig(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.time_dim, cfg.fanout, cfg.batch, k,
                         schedule=schedule, fetch_mail=True, precision=precision, fused=fused, double_buffer=db)
        g = build_tcsr(cfg.num_nodes, w["src"], w["dst"], w["ts"], dev)
        st = MemoryStage(sc, w["params"], g, dev)
        assert st.memory.double_buffer == db
        t = {kk: _t(w[kk], dev) for kk in ("src", "dst", "ts", "neg", "ef")}
        st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
        snaps = []
        for ops in st.step_ops():
            st.run_ops(ops)
            sl = st._slot(ops[-1][1])
            snaps.append(sl.mem_ts.cpu().numpy().copy())
        torch.cuda.synchronize()
        _C.check()
        res.append(({kk: getattr(st.memory, kk).cpu().numpy() for kk in ("mem", "mem_ts", "mail", "mail_ts")},
                    snaps, dict(st.versions)))
    (a, sa, va), (b, sb, vb) = res
    assert va == vb
    for kk in a:
        assert np.array_equal(a[kk], b[kk]), kk
    assert all(np.array_equal(x, y) for x, y in zip(sa, sb))


def test_double_buffer_abi(dev):
    cfg = CONFIGS["tiny"]
    h = _C.MemoryHandle(cfg.num_nodes, 100, 172, 1, dev)
    t1 = [torch.zeros_like(x) for x in (h.mem, h.mem_ts, h.mail, h.mail_ts)]
    upd = _C.alloc_update(200, 100, h.mail_stride, dev)
    _C.memory_writeback(h, 1, upd)
    with pytest.raises(_C.MspipeError) as e:  # only before the first commit
        _C._ck(_C.lib().mspipe_memory_double_buffer(h.h, *(_C.ptr(x) for x in t1)), "double_buffer")
    assert e.value.status == _C.EORDER
    h2 = _C.MemoryHandle(cfg.num_nodes, 100, 172, 1, dev, double_buffer=True)
    with pytest.raises(_C.MspipeError) as e:
        _C._ck(_C.lib().mspipe_memory_double_buffer(h2.h, *(_C.ptr(x) for x in t1)), "double_buffer")
    assert e.value.status == _C.EINVAL
    # version bookkeeping: set 0 holds versions 0, 2, ...; version committed - 1 stays readable
    assert h2.tables(0) is h2._sets[0]
    _C.memory_writeback(h2, 1, upd)
    assert h2.tables() is h2._sets[1] and h2.tables(0) is h2._sets[0]
    with pytest.raises(_C.MspipeError) as e:
        h2.tables(2)
    assert e.value.status == _C.EINVAL
    hw = _C.MemoryHandle(cfg.num_nodes, 100, 172, 1, dev, rank=0, world=2)
    with pytest.raises(_C.MspipeError) as e:
        _C._ck(_C.lib().mspipe_memory_double_buffer(hw.h, *(_C.ptr(x) for x in t1)), "double_buffer")
    assert e.value.status == _C.EUNSUPPORTED


# ------------------------------------------------------------------ ABI contract
def test_abi_staleness_and_order_errors(dev):
    cfg = CONFIGS["tiny"]
    src, dst, ts, neg = make_events(cfg, 0, 1000)
    g = build_tcsr(cfg.num_nodes, src, dst, ts, dev)
    st = MemoryStage(StageConfig(cfg.num_nodes, 100, 172, 100, 10, 200, 1), gru_params(100, 372, 100), g, dev)
    ids = torch.zeros(4, dtype=torch.int32, device=dev)
    om = torch.empty((4, 100), device=dev)
    ots = torch.empty(4, dtype=torch.float64, device=dev)
    assert _C.memory_fetch(st.memory, 1, ids, om, ots) == 0
    assert _C.memory_fetch(st.memory, 2, ids, om, ots) == 0  # k = 1: version 0 is fresh enough for i = 2
    with pytest.raises(_C.MspipeError) as e:
        _C.memory_fetch(st.memory, 3, ids, om, ots)  # needs committed >= 1
    assert e.value.status == _C.ESTALE
    upd = _C.alloc_update(200, 100, st.memory.mail_stride, dev)
    with pytest.raises(_C.MspipeError) as e:
        _C.memory_writeback(st.memory, 2, upd)
    assert e.value.status == _C.EORDER
    _C.memory_writeback(st.memory, 1, upd)  # num = 0 rows
    assert st.memory.committed == 1
    with pytest.raises(_C.MspipeError) as e:
        _C.memory_fetch(st.memory, 1, ids, om, ots)  # would read a version newer than i - 1
    assert e.value.status == _C.ESTALE


@pytest.mark.parametrize("kind", ["torch", "mspipe", "mspipe_staged"])
def test_cuda_graph_replay_equals_eager(dev, kind):
    """Step graphs (torch.cuda.CUDAGraph, or mspipe_util_graph_* as bench.py
    uses them, with resident or pinned-host inputs) replay the eager stream
    bit for bit."""
    w = make_workload("tiny", seed=3, num_events=3000)
    cfg = w["cfg"]
    outs = []
    for use_graph in (False, True):
        sc = StageConfig(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.time_dim, cfg.fanout, cfg.batch, 1)
        g = build_tcsr(cfg.num_nodes, w["src"], w["dst"], w["ts"], dev)
        st = MemoryStage(sc, w["params"], g, dev)
        if use_graph and kind == "mspipe_staged":
            st.bind_host(w["src"], w["dst"], w["ts"], w["neg"], w["ef"])
        else:
            t = {kk: _t(w[kk], dev) for kk in ("src", "dst", "ts", "neg", "ef")}
            st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
        if use_graph:
            steps = st.step_ops()
            s = torch.cuda.Stream()
            graphs = []
            for ops in steps:
                if kind == "torch":
                    gr = torch.cuda.CUDAGraph()
                    with torch.cuda.stream(s), torch.cuda.graph(gr, stream=s):
                        st.run_ops(ops)
                else:
                    gr = _C.StepGraph().capture(lambda: st.run_ops(ops), s)
                graphs.append(gr)
            st.memory.reset()
            with torch.cuda.stream(s):
                for gr in graphs:
                    gr.replay()
            st.memory.set_committed(len(graphs))  # host bookkeeping follows the replayed commits
        else:
            st.run()
        torch.cuda.synchronize()
        _C.check()
        outs.append((st.memory.mem.cpu().numpy(), st.memory.mem_ts.cpu().numpy()))
        if use_graph and kind == "mspipe_staged":
            # e2e read-back: each step reads the previous commit's result; after the
            # last step that is commit nb-1: its unique nodes, in pair order, and h'
            nb = st.num_batches
            B = cfg.batch
            j0, j1 = (nb - 2) * B, (nb - 1) * B
            pairs = np.stack([w["src"][j0:j1], w["dst"][j0:j1]], axis=1).reshape(-1)
            last = {v: p for p, v in enumerate(pairs)}
            want_nodes = [v for p, v in enumerate(pairs) if last[v] == p]
            U, nodes, hrows = st.result()
            assert U == len(want_nodes)
            assert nodes.numpy().tolist() == want_nodes
            assert np.isfinite(hrows.numpy()).all()
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("name,k,gs,staged", [("tiny", 1, 8, False), ("wiki", 1, 8, False), ("wiki", 1, 8, True),
                                              ("lastfm", 2, 5, False)])
def test_multi_step_graphs_equal_oracle(dev, name, k, gs, staged):
    """bench.py's capture: gs consecutive steps per CUDA graph (the epoch's last
    group shorter), replayed over two epochs with a reset between them, ends in
    the oracle's state (versions, mem_ts bit-exact, memory within 1e-4)."""
    w = make_workload(name, seed=11, num_events=24 * 600 + 123 if name != "tiny" else None)
    cfg = w["cfg"]
    sc = StageConfig(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.time_dim, cfg.fanout, cfg.batch, k)
    g = build_tcsr(cfg.num_nodes, w["src"], w["dst"], w["ts"], dev)
    st = MemoryStage(sc, w["params"], g, dev)
    if staged:
        st.bind_host(w["src"], w["dst"], w["ts"], w["neg"], w["ef"])
    else:
        t = {kk: _t(w[kk], dev) for kk in ("src", "dst", "ts", "neg", "ef")}
        st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
    sops = st.step_ops()
    s = torch.cuda.Stream()
    groups = []
    for j in range(0, len(sops), gs):
        def run_group(idx=range(j, min(j + gs, len(sops)))):
            for q in idx:  # as bench.py: the e2e copy streams join only at the graph's end
                st.run_ops(sops[q], join_copies=(q == idx[-1]))
        groups.append(_C.StepGraph().capture(run_group, s))
    for epoch in range(2):
        st.memory.reset()
        with torch.cuda.stream(s):
            for gr in groups:
                gr.replay(s)
        torch.cuda.synchronize()
    st.memory.set_committed(len(sops))
    _C.check()
    ref, vers = oracle.run_stream(cfg.num_nodes, w["src"], w["dst"], w["ts"], w["ef"], w["params"], cfg.batch, k,
                                  "exact", fanout=cfg.fanout)
    assert [st.versions[i] for i in range(1, len(vers) + 1)] == vers.tolist()
    assert np.array_equal(st.memory.mem_ts.cpu().numpy(), ref["mem_ts"])
    gm, om = st.memory.mem.cpu().numpy().astype(np.float64), ref["mem"].astype(np.float64)
    rel = np.linalg.norm(gm - om, axis=1) / np.maximum(np.linalg.norm(om, axis=1), 1e-3)
    assert rel.max() <= 1e-4


def test_determinism_two_runs_bitwise(dev):
    a = _stream(dev, "lastfm", 1, E=30_000)[0].memory
    b = _stream(dev, "lastfm", 1, E=30_000)[0].memory
    for key in ("mem", "mem_ts", "mail", "mail_ts"):
        assert torch.equal(getattr(a, key), getattr(b, key)), key


def test_two_stream_overlap_equals_serial(dev):
    """prep(t+k) on a side stream overlapping update(t) gives bitwise the same state."""
    w = make_workload("lastfm", seed=4, num_events=24_000)
    cfg = w["cfg"]
    outs = []
    for overlap in (False, True):
        sc = StageConfig(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.time_dim, cfg.fanout, cfg.batch, 2)
        g = build_tcsr(cfg.num_nodes, w["src"], w["dst"], w["ts"], dev)
        st = MemoryStage(sc, w["params"], g, dev)
        t = {kk: _t(w[kk], dev) for kk in ("src", "dst", "ts", "neg", "ef")}
        st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
        for ops in st.step_ops():
            st.run_ops(ops, overlap=overlap)
        torch.cuda.synchronize()
        outs.append([getattr(st.memory, k).cpu().numpy() for k in ("mem", "mem_ts", "mail", "mail_ts")])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


# ------------------------------------------------------------------ row F1
@pytest.mark.parametrize("name,E,B", [("tiny", None, 200), ("wiki", None, 600), ("lastfm", 300_000, 600),
                                      ("tiny", 3001, 7)])
def test_stale_histogram_equals_oracle(dev, name, E, B):
    """mspipe_stale_histogram (GPU, T-CSR search) == the oracle's batch replay, bit for bit."""
    from oracle import planner as OP
    cfg = CONFIGS[name]
    src, dst, ts, _ = make_events(cfg, 2, E)
    g = build_tcsr(cfg.num_nodes, src, dst, ts, dev)
    max_d = 40
    h = _C.stale_histogram(g, _t(src, dev), _t(dst, dev), B, max_d).cpu().numpy()
    _, ref = OP.stale_fraction(src, dst, B, [1])
    want = np.zeros(max_d + 2, np.int64)
    for d, c in ref.items():
        want[min(d, max_d + 1)] += c
    assert np.array_equal(h, want)


@pytest.mark.parametrize("name,k,mit,E", [("tiny", 0, False, None), ("tiny", 2, False, None),
                                          ("wiki", 1, False, 60_000), ("reddit", 2, True, 60_000),
                                          ("tiny", 2, True, None)])
def test_staleness_error_series_equals_oracle(dev, name, k, mit, E):
    """Row F1 analytics: the lockstep GPU series (mspipe_staleness_error over the
    stale stage's and a k = 0 stage's fetched rows) against the oracle's dual
    run; k = 0 without MSPipe-S is exactly 0 (two identical deterministic runs)."""
    from paper_2402_15113_b200.planner import staleness_error_series
    w = make_workload(name, seed=6, num_events=E)
    cfg = w["cfg"]
    m = None
    if mit:
        m = dict(lam=cfg.lam, gamma=oracle.gamma(cfg.num_nodes, w["src"], w["dst"], w["ts"], 0.99), n_sim=cfg.n_sim)
    sc = StageConfig(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.time_dim, cfg.fanout, cfg.batch, k, mitigation=m)
    g = build_tcsr(cfg.num_nodes, w["src"], w["dst"], w["ts"], dev)
    t = {kk: _t(w[kk], dev) for kk in ("src", "dst", "ts", "neg", "ef")}
    got = staleness_error_series(sc, w["params"], g, dev, t["src"], t["dst"], t["ts"], t["neg"], t["ef"]).cpu().numpy()
    _C.check()
    ref = oracle.staleness_error_series(cfg.num_nodes, w["src"], w["dst"], w["ts"], w["ef"], w["params"], cfg.batch,
                                        k, mitigation=m, fanout=cfg.fanout)
    assert got.shape == ref.shape
    if k == 0 and not mit:
        assert (got == 0).all() and (ref == 0).all()
    ok, err = _close(got, ref, rtol=1e-4, atol=1e-5)
    print(f"{name} k={k} mit={mit}: staleness error mean {ref.mean():.4g}, max |gpu - oracle| {err:.3g}")
    assert ok, err


@pytest.mark.parametrize("fused", [True, False])
def test_stream_with_plan_equals_oracle(dev, fused):
    """A per-iteration plan k_i (row F1: prep(i) right after commit(i - k_i)) gives
    the oracle's state under the same plan."""
    from paper_2402_15113_b200.planner import stage_config_for_plan
    w = make_workload("lastfm", seed=6, num_events=36_000)
    cfg = w["cfg"]
    nb = -(-36_000 // cfg.batch)
    rng = np.random.default_rng(6)
    plan = [min(i, int(rng.integers(1, 5))) for i in range(1, nb + 1)]
    base = StageConfig(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.time_dim, cfg.fanout, cfg.batch, 0,
                       fetch_mail=True, fused=fused)
    sc = stage_config_for_plan(base, plan)
    g = build_tcsr(cfg.num_nodes, w["src"], w["dst"], w["ts"], dev)
    st = MemoryStage(sc, w["params"], g, dev)
    t = {kk: _t(w[kk], dev) for kk in ("src", "dst", "ts", "neg", "ef")}
    st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
    st.run()
    torch.cuda.synchronize()
    _C.check()
    ref, vers = oracle.run_stream(cfg.num_nodes, w["src"], w["dst"], w["ts"], w["ef"], w["params"], cfg.batch,
                                  sc.k, plan=plan)
    assert [st.versions[i] for i in range(1, nb + 1)] == vers.tolist()
    assert np.array_equal(st.memory.mem_ts.cpu().numpy(), ref["mem_ts"])
    gm, om = st.memory.mem.cpu().numpy().astype(np.float64), ref["mem"].astype(np.float64)
    rel = np.linalg.norm(gm - om, axis=1) / np.maximum(np.linalg.norm(om, axis=1), 1e-3)
    assert rel.max() <= 1e-4


@pytest.mark.parametrize("name,E,fused", [("gdelt", 30_000, True), ("gdelt", 30_000, False), ("tiny", None, True)])
def test_feature_fetch_equals_oracle(dev, name, E, fused):
    """F2 inside the stage (its own stream, forked after the sampler): node-feature
    rows of the subgraph nodes and edge-feature rows of the sampled links equal
    the oracle's gather over the oracle sampler's ids, bit for bit; the state is
    unchanged by it."""
    from oracle.features import feature_fetch
    from synth import node_features
    w = make_workload(name, seed=9, num_events=E)
    cfg = w["cfg"]
    nf = node_features(9, cfg.num_nodes, cfg.node_dim) if cfg.node_dim else None
    B = 500 if name == "gdelt" else cfg.batch
    sc = StageConfig(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.time_dim, cfg.fanout, B, 1, fused=fused,
                     features=True, node_dim=cfg.node_dim)
    g = build_tcsr(cfg.num_nodes, w["src"], w["dst"], w["ts"], dev)
    st = MemoryStage(sc, w["params"], g, dev)
    t = {kk: _t(w[kk], dev) for kk in ("src", "dst", "ts", "neg", "ef")}
    st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
    st.bind_features(nf, t["ef"])
    ops = st.step_ops()
    og = oracle.Graph(cfg.num_nodes, w["src"], w["dst"], w["ts"])
    for o in ops[:6]:
        st.run_ops(o)
    torch.cuda.synchronize()
    _C.check()
    for i in sorted({i for o in ops[:6] for op, i in o if op == "prep"})[-2:]:
        j0, j1 = (i - 1) * B, min(i * B, len(w["src"]))
        roots = np.concatenate([w["src"][j0:j1], w["dst"][j0:j1], w["neg"][j0:j1]])
        s = og.sample(roots, np.concatenate([w["ts"][j0:j1]] * 3), cfg.fanout)
        sub = np.concatenate([roots[:, None], s["nbr"]], axis=1)
        on, oe = feature_fetch(sub, s["eid"], nf, w["ef"])
        sl = st._slot(i)
        R = len(roots)
        assert np.array_equal(sl.efeat[:R].cpu().numpy(), oe)
        if nf is not None:
            assert np.array_equal(sl.nfeat[:R, :, : cfg.node_dim].cpu().numpy(), on)


# ------------------------------------------------------------------ row F3
@pytest.mark.parametrize("name,k,E", [("tiny", 0, None), ("wiki", 1, 60_000), ("lastfm", 2, 80_000)])
@pytest.mark.parametrize("cell,mailbox", [("rnn", "immediate"), ("gru", "deferred"), ("rnn", "deferred")])
def test_updater_variants_free_running(dev, name, k, E, cell, mailbox):
    """Row F3: RNN-cell updater (JODIE) and deferred mailbox (TGL TGN) over whole
    streams against the oracle's variants: timestamps bit-exact, memories and
    mails within the fp32 tolerance."""
    from synth import rnn_params
    w = make_workload(name, seed=11, num_events=E)
    cfg = w["cfg"]
    params = rnn_params(cfg.mem_dim, cfg.mail_dim, cfg.time_dim) if cell == "rnn" else w["params"]
    sc = StageConfig(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.time_dim, cfg.fanout, cfg.batch, k,
                     fetch_mail=True, cell=cell, mailbox=mailbox)
    g = build_tcsr(cfg.num_nodes, w["src"], w["dst"], w["ts"], dev)
    st = MemoryStage(sc, params, g, dev)
    t = {kk: _t(w[kk], dev) for kk in ("src", "dst", "ts", "neg", "ef")}
    st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
    st.run()
    torch.cuda.synchronize()
    _C.check()
    ref, vers = oracle.run_stream(cfg.num_nodes, w["src"], w["dst"], w["ts"], w["ef"], params, cfg.batch, k,
                                  mailbox=mailbox, cell=cell)
    assert np.array_equal(st.memory.mem_ts.cpu().numpy(), ref["mem_ts"])
    assert np.array_equal(st.memory.mail_ts.cpu().numpy(), ref["mail_ts"])
    gm, om = st.memory.mem.cpu().numpy().astype(np.float64), ref["mem"].astype(np.float64)
    rel = np.linalg.norm(gm - om, axis=1) / np.maximum(np.linalg.norm(om, axis=1), 1e-3)
    print(f"{name} k={k} {cell}/{mailbox}: row-rel max {rel.max():.3g}")
    assert rel.max() <= 1e-4
    Dm = cfg.mail_dim
    ok, err = _close(st.memory.mail.cpu().numpy()[:, :Dm], ref["mail"], rtol=1e-4, atol=1e-5)
    assert ok, err


def test_updater_variant_abi(dev):
    from synth import rnn_params
    cfg = CONFIGS["tiny"]
    p = rnn_params(cfg.mem_dim, cfg.mail_dim, cfg.time_dim)
    with pytest.raises(_C.MspipeError) as e:  # variants are tensor-core only
        _C.GruHandle(cfg.mem_dim, cfg.edge_dim, cfg.time_dim, p, dev, _C.FP32_SIMT, cell=_C.CELL_RNN)
    assert e.value.status == _C.EUNSUPPORTED
    gd = _C.GruHandle(cfg.mem_dim, cfg.edge_dim, cfg.time_dim, gru_params(cfg.mem_dim, cfg.mail_dim, cfg.time_dim),
                      dev, mailbox=_C.MAILBOX_DEFERRED)
    h = _C.MemoryHandle(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, 0, dev)
    x = torch.zeros(4, dtype=torch.int32, device=dev)
    upd = _C.alloc_update(4, cfg.mem_dim, h.mail_stride, dev)
    with pytest.raises(_C.MspipeError) as e:  # the immediate-message entry points refuse a deferred handle
        _C.memory_update(h, gd, x, x, x.double(), torch.zeros((4, cfg.edge_dim), device=dev),
                         torch.zeros((12 * 11, cfg.mem_dim), device=dev), torch.zeros(12 * 11, dtype=torch.float64,
                                                                                      device=dev), 11, upd)
    assert e.value.status == _C.EUNSUPPORTED
    with pytest.raises(_C.MspipeError) as e:  # mail rows follow commit `committed`, not another version
        _C.memory_mail_deferred(h, 3, x, x, x.double(), torch.zeros((4, cfg.edge_dim), device=dev), upd["nodes"],
                                upd["winner"], upd["num"])
    assert e.value.status == _C.EORDER


# ------------------------------------------------------------------ bf16 updater
BF16_TOL = 2e-2  # north star: "2e-2 if a bf16 GRU path is enabled"
BF16_ATOL = 1e-3  # per element |g - o| <= 2e-2 |o| + 1e-3 (bf16 mode)


def _bf16_ok(g, o, label):
    """C.6's per-element bf16 rule; prints the worst element's share of its bound."""
    g, o = np.asarray(g, np.float64), np.asarray(o, np.float64)
    share = np.abs(g - o) / (BF16_TOL * np.abs(o) + BF16_ATOL)
    print(f"{label}: max abs err {np.abs(g - o).max():.3g}, worst element at {share.max():.3g} of its "
          f"2e-2|o| + 1e-3 bound")
    return share.max() <= 1.0


@pytest.mark.parametrize("name,i,E", [("tiny", 1, None), ("wiki", 137, None), ("gdelt", 3, 20_000)])
def test_update_teacher_forced_bf16(dev, name, i, E):
    """MSPIPE_BF16 (tcgen05 kind::f16, bf16 operands, fp32 accumulation): h' within
    2e-2 of the f64-accumulated oracle; everything integer or copied stays exact."""
    st, sl, upd, ref, ev, (mem, mem_ts) = _teacher_forced(dev, name, i, E=E, precision=_C.BF16, fused=True)
    U = int(upd["num"].item())
    assert np.array_equal(upd["nodes"][:U].cpu().numpy(), ref["nodes"])
    assert np.array_equal(upd["ts"][:U].cpu().numpy(), ref["ts"])
    Dm = ref["mail"].shape[1]
    assert np.array_equal(upd["mail"][:U].cpu().numpy()[:, :Dm], ref["mail"])
    g, o = upd["mem"][:U].cpu().numpy().astype(np.float64), ref["mem"].astype(np.float64)
    assert _bf16_ok(g, o, f"{name} bf16 teacher-forced")


@pytest.mark.parametrize("name,k,E,cell", [("wiki", 1, 60_000, "gru"), ("lastfm", 2, 60_000, "gru"),
                                           ("tiny", 0, None, "rnn")])
def test_stream_free_running_bf16(dev, name, k, E, cell):
    from synth import rnn_params
    w = make_workload(name, seed=12, num_events=E)
    cfg = w["cfg"]
    params = rnn_params(cfg.mem_dim, cfg.mail_dim, cfg.time_dim) if cell == "rnn" else w["params"]
    sc = StageConfig(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.time_dim, cfg.fanout, cfg.batch, k,
                     precision=_C.BF16, cell=cell)
    g = build_tcsr(cfg.num_nodes, w["src"], w["dst"], w["ts"], dev)
    st = MemoryStage(sc, params, g, dev)
    t = {kk: _t(w[kk], dev) for kk in ("src", "dst", "ts", "neg", "ef")}
    st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
    st.run()
    torch.cuda.synchronize()
    _C.check()
    ref, _ = oracle.run_stream(cfg.num_nodes, w["src"], w["dst"], w["ts"], w["ef"], params, cfg.batch, k, cell=cell)
    assert np.array_equal(st.memory.mem_ts.cpu().numpy(), ref["mem_ts"])
    assert _bf16_ok(st.memory.mem.cpu().numpy(), ref["mem"], f"{name} k={k} {cell} bf16 free-running")


# ------------------------------------------------------------------ bench launch configuration
@pytest.mark.parametrize("name,E,gru", [("wiki", None, "tc"), ("gdelt", 80_000, "tc"), ("reddit", 60_000, "tc"),
                                        ("wiki", None, "bf16")])
def test_bench_configuration_matches_oracle(dev, name, E, gru):
    """The configuration bench.py times — per-step graphs (mspipe_util_graph_*)
    replayed after a reset, the config's own batch and staleness k, double-
    buffered tables, fused kernels, two streams, MSPipe-S where the config has
    it — at the workload's full size (GDELT / Reddit: a prefix), against the
    oracle: timestamps bit-exact, memories within the tolerance."""
    from paper_2402_15113_b200 import gamma_quantile
    w = make_workload(name, seed=0, num_events=E)
    cfg = w["cfg"]
    mit = None
    if cfg.mitigation:
        mit = dict(lam=cfg.lam, gamma=gamma_quantile(cfg.num_nodes, w["src"], w["dst"], w["ts"], cfg.quantile_p),
                   n_sim=cfg.n_sim)
    sc = StageConfig(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.time_dim, cfg.fanout, cfg.batch,
                     cfg.staleness_k, mitigation=mit, precision=_C.BF16 if gru == "bf16" else _C.FP32_3XTF32)
    g = build_tcsr(cfg.num_nodes, w["src"], w["dst"], w["ts"], dev)
    st = MemoryStage(sc, w["params"], g, dev)
    assert st.memory.double_buffer == (cfg.staleness_k >= 1)
    t = {kk: _t(w[kk], dev) for kk in ("src", "dst", "ts", "neg", "ef")}
    st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
    s = torch.cuda.Stream()
    graphs = [_C.StepGraph().capture(lambda: st.run_ops(ops), s) for ops in st.step_ops()]
    st.memory.reset()
    with torch.cuda.stream(s):
        for gr in graphs:
            gr.replay()
    st.memory.set_committed(len(graphs))
    torch.cuda.synchronize()
    _C.check()
    ref, _ = oracle.run_stream(cfg.num_nodes, w["src"], w["dst"], w["ts"], w["ef"], w["params"], cfg.batch,
                               cfg.staleness_k, mitigation=mit, fanout=cfg.fanout)
    assert np.array_equal(st.memory.mem_ts.cpu().numpy(), ref["mem_ts"])
    gm, om = st.memory.mem.cpu().numpy().astype(np.float64), ref["mem"].astype(np.float64)
    if gru == "bf16":
        assert _bf16_ok(gm, om, f"{name} bench configuration bf16")
    else:
        rel = np.linalg.norm(gm - om, axis=1) / np.maximum(np.linalg.norm(om, axis=1), 1e-3)
        print(f"{name} bench configuration: row-rel max {rel.max():.3g}")
        assert rel.max() <= 1e-4



# ------------------------------------------------- sizes and degenerate batches
def _run_stream(dev, w, B, k, schedule="exact", **kw):
    cfg = w["cfg"]
    sc = StageConfig(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.time_dim, cfg.fanout, B, k, schedule=schedule,
                     **kw)
    g = build_tcsr(cfg.num_nodes, w["src"], w["dst"], w["ts"], dev)
    st = MemoryStage(sc, w["params"], g, dev)
    t = {kk: _t(w[kk], dev) for kk in ("src", "dst", "ts", "neg", "ef")}
    st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
    st.run()
    torch.cuda.synchronize()
    _C.check()
    ref, vers = oracle.run_stream(cfg.num_nodes, w["src"], w["dst"], w["ts"], w["ef"], w["params"], B, k, schedule,
                                  fanout=cfg.fanout)
    assert [st.versions[i] for i in range(1, len(vers) + 1)] == vers.tolist()
    assert np.array_equal(st.memory.mem_ts.cpu().numpy(), ref["mem_ts"])
    assert np.array_equal(st.memory.mail_ts.cpu().numpy(), ref["mail_ts"])
    gm, om = st.memory.mem.cpu().numpy().astype(np.float64), ref["mem"].astype(np.float64)
    rel = np.linalg.norm(gm - om, axis=1) / np.maximum(np.linalg.norm(om, axis=1), 1e-3)
    assert rel.max() <= 1e-4, rel.max()
    ok, err = _close(st.memory.mail.cpu().numpy()[:, :cfg.mail_dim], ref["mail"], rtol=1e-4, atol=1e-5)
    assert ok, err
    return rel.max()


@pytest.mark.parametrize("clusters", [0, 1, 3])
def test_max_batch_ragged_tail_and_tile_loop(dev, clusters, monkeypatch):
    """The largest batch the fused prep takes (B = 8192: U up to 16,384 GEMM rows,
    up to 128 M tiles x 7 hidden tiles) on a GDELT-shaped stream with a ragged
    last batch, k = 1; with the persistent GEMM forced onto 1 or 3 clusters, one
    cluster walks dozens of tiles (stage phases, the early loads of the next
    tile and the two receive buffers all cycle).  Equals the oracle."""
    if clusters:
        monkeypatch.setenv("MSPIPE_TC_CLUSTERS", str(clusters))
    w = make_workload("gdelt", seed=5, num_events=3 * 8192 + 17)
    rel = _run_stream(dev, w, 8192, 1)
    print(f"B=8192 clusters={clusters or 'auto'}: row-rel max {rel:.3g}")


def test_degenerate_batches(dev):
    """Batches whose events all repeat one pair (U = 2), self-loops (a node is
    both endpoints: one winner per event), a node hit by every event of a batch
    (LastFM's hot node at its extreme), and a one-event last batch; k = 0 and 2."""
    cfg = CONFIGS["tiny"]
    B = 64
    src = np.concatenate([np.full(B, 3), np.arange(B) % 7, np.full(B, 5), np.arange(B) + 100, [9]]).astype(np.int32)
    dst = np.concatenate([np.full(B, 4), np.arange(B) % 7, (np.arange(B) * 13) % 997, np.full(B, 100), [9]])
    dst = dst.astype(np.int32)
    E = len(src)
    ts = np.floor(np.cumsum(np.random.default_rng(3).exponential(0.7, E))).astype(np.float64)
    neg = np.random.default_rng(4).integers(0, cfg.num_nodes, E).astype(np.int32)
    w = dict(cfg=cfg, src=src, dst=dst, ts=ts, neg=neg, ef=edge_features(7, 0, E, cfg.edge_dim),
             params=gru_params(cfg.mem_dim, cfg.mail_dim, cfg.time_dim))
    for k in (0, 2):
        _run_stream(dev, w, B, k)


@pytest.mark.parametrize("env", [{"MSPIPE_SPLIT_COMMIT": "0"}, {"MSPIPE_SAMPLE_HINT": "0"},
                                 {"MSPIPE_TC_SPLITS": "1"}, {"MSPIPE_TC_SPLITS": "2"}, {"MSPIPE_TC_BIG_S": "4"},
                                 {"MSPIPE_PREP_SMEM": "0", "MSPIPE_PREP_BPS": "4"}, {"MSPIPE_BUILD_ROW": "1"}, {"MSPIPE_BUILD_CHUNKS": "2"}, {"MSPIPE_BUILD_CHUNKS": "4"},
                                 {"MSPIPE_WB_FIRST": "0"}, {"MSPIPE_WB_FIRST": "1"}, {"MSPIPE_GRAPH_PRIO": "1"}, {"MSPIPE_PREP_STCS": "1"},
                                 {"MSPIPE_TCSR_LDCS": "1"}, {"MSPIPE_TCSR_LDCS": "0", "MSPIPE_PREP_STCS": "0"}])
def test_switch_variants_equal_oracle(dev, env, monkeypatch):
    """The library's experiment switches (read at every launch) keep the oracle's
    results: the GEMM epilogue writing mem_ts / mail itself (no write-back
    branch), the sampler without its per-node search hints, S = 1 and 2 at wiki size (three and
    two K chunks per TMEM buffer; default 4), S = 4 at GDELT size (default 2), the dedup table
    in global memory."""
    for kk, v in env.items():
        monkeypatch.setenv(kk, v)
    name = "gdelt" if "MSPIPE_TC_BIG_S" in env else "wiki"
    w = make_workload(name, seed=13, num_events=12 * (4000 if name == "gdelt" else 600) + 77)
    _run_stream(dev, w, w["cfg"].batch, 1)

"""GPU parity at the sizes bench.py times.

* Whole streams through bench.py's launch configuration (8 steps per CUDA
  graph, fused kernels, two streams, double-buffered tables, the epoch reset
  issued inside the replay stream's context as bench.py does, two epochs):
  Reddit (672,447 events, MSPipe-S, k = 2), LastFM (1,293,103 events, hot
  nodes, k = 2), Wikipedia (157,474, k = 1), and GDELT's first 1,000 batches
  (4M events, k = 3) over the T-CSR of the WHOLE 191M-event stream.
  Timestamps bit-exact; memory row-relative drift max <= 1e-4, max and p99
  reported (C.6 "free-running trajectory").
* The A3s output — the 3B(𝒩+1) subgraph ids and the snapshot rows S_{v(i)}
  gathered for them — compared with the oracle's, bit for bit, batch by batch,
  with double-buffered tables (catch-up active) and with one table set.
* The full-length GDELT T-CSR under the sampler: roots at query times spread
  over the whole stream (rows of up to 39M entries), bit-exact vs the oracle.

Expected values come from oracle/ only."""
import numpy as np
import pytest
import torch

import oracle
from paper_2402_15113_b200 import MemoryStage, StageConfig, _C, build_tcsr, gamma_quantile
from synth import CONFIGS, make_workload

pytestmark = pytest.mark.gpu

GDELT_PREFIX = 4_000_000  # bench.py's GDELT window: the first 1,000 batches


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    d = torch.device("cuda:0")
    torch.cuda.set_device(d)
    return d


@pytest.fixture(scope="module")
def gdelt(dev):
    """GDELT's first 4M events + the T-CSR of the whole 191M-event stream (device)."""
    w = make_workload("gdelt", seed=0, num_events=GDELT_PREFIX, tcsr_events=CONFIGS["gdelt"].num_events)
    g = build_tcsr(w["cfg"].num_nodes, *w["tcsr"], dev)
    return w, g


def _t(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def _mit(w):
    cfg = w["cfg"]
    if not cfg.mitigation:
        return None
    return dict(lam=cfg.lam, gamma=gamma_quantile(cfg.num_nodes, w["src"], w["dst"], w["ts"], cfg.quantile_p),
                n_sim=cfg.n_sim)


def _drift(gm, om):
    gm, om = gm.astype(np.float64), om.astype(np.float64)
    rel = np.linalg.norm(gm - om, axis=1) / np.maximum(np.linalg.norm(om, axis=1), 1e-3)
    return float(rel.max()), float(np.quantile(rel, 0.99))


def _bench_path(dev, w, g, k, mit, gs=8, epochs=2):
    """bench.py's timed configuration: gs steps per CUDA graph, replayed from a
    reset issued inside the replay stream's context, `epochs` times."""
    cfg = w["cfg"]
    sc = StageConfig(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.time_dim, cfg.fanout, cfg.batch, k,
                     mitigation=mit)
    st = MemoryStage(sc, w["params"], g, dev)
    assert st.fused and st.memory.double_buffer == (k >= 1)
    t = {kk: _t(w[kk], dev) for kk in ("src", "dst", "ts", "neg", "ef")}
    st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
    sops = st.step_ops()
    s = torch.cuda.Stream()
    groups = []
    for j in range(0, len(sops), gs):
        def run_group(idx=range(j, min(j + gs, len(sops)))):
            for q in idx:
                st.run_ops(sops[q], join_copies=(q == idx[-1]))
        groups.append(_C.StepGraph().capture(run_group, s))
    with torch.cuda.stream(s):
        for _ in range(epochs):
            st.memory.reset()  # on the current (replay) stream, as bench.py does
            for gr in groups:
                gr.replay(s)
    torch.cuda.synchronize()
    st.memory.set_committed(len(sops))
    _C.check()
    return st


def _check_stream(st, w, k, mit, label):
    cfg = w["cfg"]
    ref, vers = oracle.run_stream(cfg.num_nodes, w["src"], w["dst"], w["ts"], w["ef"], w["params"], cfg.batch, k,
                                  mitigation=mit, fanout=cfg.fanout)
    assert [st.versions[i] for i in range(1, len(vers) + 1)] == vers.tolist()
    assert np.array_equal(st.memory.mem_ts.cpu().numpy(), ref["mem_ts"])
    assert np.array_equal(st.memory.mail_ts.cpu().numpy(), ref["mail_ts"])
    mx, p99 = _drift(st.memory.mem.cpu().numpy(), ref["mem"])
    nb = len(vers)
    print(f"{label}: {len(w['src'])} events, {nb} batches, k={k}{' MSPipe-S' if mit else ''}: "
          f"free-running row-rel drift max {mx:.3g} p99 {p99:.3g}")
    assert mx <= 1e-4
    mail_mx, _ = _drift(st.memory.mail.cpu().numpy()[:, :cfg.mail_dim], ref["mail"])
    assert mail_mx <= 1e-4


@pytest.mark.parametrize("name", ["reddit", "lastfm", "wiki"])
def test_whole_stream_bench_path(dev, name):
    w = make_workload(name, seed=0)
    cfg = w["cfg"]
    mit = _mit(w)
    g = build_tcsr(cfg.num_nodes, w["src"], w["dst"], w["ts"], dev)
    st = _bench_path(dev, w, g, cfg.staleness_k, mit)
    _check_stream(st, w, cfg.staleness_k, mit, name)


def test_gdelt_bench_window_over_full_tcsr(dev, gdelt):
    """bench.py's GDELT workload exactly: 1,000 batches of 4,000 events, k = 3,
    sampler over the whole-stream T-CSR; the oracle runs the same prefix (its
    sampler sees only strictly earlier events, so the prefix suffices)."""
    w, g = gdelt
    st = _bench_path(dev, w, g, 3, None, epochs=1)
    _check_stream(st, w, 3, None, "gdelt (first 1,000 batches, 191M-event T-CSR)")


def test_gdelt_full_tcsr_sampler(dev, gdelt):
    """A1 on GDELT's full-length rows (mean 22,934 entries, max ~39M: a 33-ary
    search of up to five rounds) at query times spread over the whole stream."""
    w, g = gdelt
    cfg = w["cfg"]
    src, dst, ts = w["tcsr"]
    rng = np.random.default_rng(5)
    n = 20_000
    E = len(src)
    j = rng.integers(0, E, n)
    roots = np.where(rng.random(n) < 0.5, src[j], dst[j]).astype(np.int32)
    roots[: n // 10] = rng.integers(0, cfg.num_nodes, n // 10)
    qts = ts[j] + rng.integers(0, 2, n) * 15.0  # tick ties and the next tick
    out = _C.alloc_sample(n, cfg.fanout, dev)
    _C.sample_recent(g, _t(roots, dev), _t(qts, dev), cfg.fanout, out)
    ref = oracle.Graph(cfg.num_nodes, src, dst, ts).sample(roots, qts, cfg.fanout)
    for key in ("nbr", "eid", "ts", "dt", "cnt"):
        assert np.array_equal(out[key].cpu().numpy(), ref[key]), key
    _C.check()
    print(f"gdelt full T-CSR: {n} roots, mean cnt {ref['cnt'].mean():.2f}")


# ------------------------------------------------------------ A3s rows vs the oracle
@pytest.mark.parametrize("name,E,k", [("wiki", None, 1), ("lastfm", 150_000, 2), ("reddit", 120_000, 2),
                                      ("tiny", None, 0)])
def test_subgraph_rows_equal_oracle_snapshot(dev, name, E, k):
    """The A3s output of the dumped batches against the oracle's S_{v(i)}: the
    3B(𝒩+1) subgraph ids and the rows' mem_ts bit-exact, the memory rows within
    the free-running tolerance (the state they copy is itself a GPU trajectory,
    ~1e-7 from the oracle's); and, with the double-buffered tables' catch-up
    active, the fetched rows bitwise equal to those of a one-table-set run."""
    w = make_workload(name, seed=3, num_events=E)
    g = build_tcsr(w["cfg"].num_nodes, w["src"], w["dst"], w["ts"], dev)
    a = _subgraph_rows(dev, w, g, k, False, _mit(w))
    if k >= 1:
        b = _subgraph_rows(dev, w, g, k, True, _mit(w))
        for i in a:
            for x, y in zip(a[i][:3], b[i][:3]):  # ids, rows, mem_ts
                assert np.array_equal(x, y), i


def test_subgraph_rows_equal_oracle_snapshot_gdelt(dev, gdelt):
    w, g = gdelt
    nb = 40
    ww = dict(w, src=w["src"][: nb * 4000], dst=w["dst"][: nb * 4000], ts=w["ts"][: nb * 4000],
              neg=w["neg"][: nb * 4000], ef=w["ef"][: nb * 4000])
    _subgraph_rows(dev, ww, g, 3, True, None)


def _subgraph_rows(dev, w, g, k, db, mit):
    cfg = w["cfg"]
    B, F = cfg.batch, cfg.fanout
    sc = StageConfig(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.time_dim, F, B, k, mitigation=mit,
                     double_buffer=db)
    st = MemoryStage(sc, w["params"], g, dev)
    assert st.memory.double_buffer == db
    t = {kk: _t(w[kk], dev) for kk in ("src", "dst", "ts", "neg", "ef")}
    st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
    nb = st.num_batches
    rng = np.random.default_rng(nb)
    want = sorted(set([1, 2, k + 2, nb] + rng.integers(1, nb + 1, 6).tolist()))
    got = {}
    for ops in st.step_ops():
        st.run_ops(ops)
        for op, i in ops:
            # the slot of a batch is rewritten k+1 preps later: read right after its step
            if op == "prep" and i in want:
                torch.cuda.synchronize()
                sl = st._slot(i)
                n = min(B, len(w["src"]) - (i - 1) * B)
                m = 3 * n * (F + 1)
                got[i] = (sl.samp["sub"][: 3 * n].cpu().numpy().reshape(-1), sl.mem[:m].cpu().numpy(),
                          sl.mem_ts[:m].cpu().numpy(),
                          {kk: sl.samp[kk][: 3 * n].cpu().numpy() for kk in ("nbr", "eid", "ts", "dt", "cnt")})
    torch.cuda.synchronize()
    _C.check()
    _, vers, dump = oracle.run_stream(cfg.num_nodes, w["src"], w["dst"], w["ts"], w["ef"], w["params"], B, k,
                                      mitigation=mit, fanout=F, neg=w["neg"], dump_batches=want)
    worst = 0.0
    og = oracle.Graph(cfg.num_nodes, w["src"], w["dst"], w["ts"])
    for q, i in enumerate(dump["batches"]):
        ids, rows, mts, samp = got[int(i)]
        j0, j1 = (int(i) - 1) * B, min(int(i) * B, len(w["src"]))
        roots = np.concatenate([w["src"][j0:j1], w["dst"][j0:j1], w["neg"][j0:j1]])
        sref = og.sample(roots, np.concatenate([w["ts"][j0:j1]] * 3), F)  # A1 of the fused prep (hinted search)
        for kk in ("nbr", "eid", "ts", "dt", "cnt"):
            assert np.array_equal(samp[kk], sref[kk]), (i, kk)
        m = len(ids)
        assert np.array_equal(ids, dump["sub_ids"][q][:m]), i
        assert np.array_equal(mts, dump["mem_ts"][q][:m]), i
        o = dump["mem"][q][:m].astype(np.float64)
        err = np.abs(rows.astype(np.float64) - o)
        assert (err <= 1e-4 * np.abs(o) + 1e-5).all(), (i, err.max())
        assert (rows[ids == -1] == 0).all()  # pads are zero rows
        worst = max(worst, float(err.max()))
        assert st.versions[int(i)] == vers[int(i) - 1]
    print(f"{cfg.name} k={k} db={db}: subgraph ids / mem_ts of batches {want} bit-exact, rows max |gpu - oracle| "
          f"{worst:.3g}")
    return got

"""Row F3 APAN on the GPU (mspipe_message_build_apan + the GRU GEMM +
mspipe_apan_deliver, through the stage) against oracle/apan.py: winners,
mem_ts, mailbox times / positions / counts bit-exact; memory and mailbox rows
within 1e-4 (fp32 projections and the 3xTF32 GRU against f64)."""
import numpy as np
import pytest
import torch

import oracle
from oracle import apan as oa
from paper_2402_15113_b200 import MemoryStage, StageConfig, _C, build_tcsr
from synth import CONFIGS, edge_features, gru_params, make_events

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    d = torch.device("cuda:0")
    torch.cuda.set_device(d)
    return d


def _t(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def _weights(M, Dm, seed=21):
    rng = np.random.default_rng(seed)
    return dict(w_q=rng.uniform(-1, 1, (M, M)).astype(np.float32) / np.sqrt(M),
                w_k=rng.uniform(-1, 1, (M, Dm)).astype(np.float32) / np.sqrt(Dm))


def _stage(dev, cfg, gp, ap, src, dst, ts, neg, ef, k=0):
    sc = StageConfig(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.time_dim, cfg.fanout, cfg.batch, k, fused=True,
                     mailbox="apan", apan=dict(ap, slots=oa.SLOTS))
    g = build_tcsr(cfg.num_nodes, src, dst, ts, dev)
    st = MemoryStage(sc, gp, g, dev)
    return st, g


@pytest.mark.parametrize("name,i,E", [("tiny", 7, None), ("wiki", 60, 60_000), ("gdelt", 3, 20_000)])
def test_apan_teacher_forced(dev, name, i, E):
    """One batch from a random memory + random partly filled mailboxes."""
    cfg = CONFIGS[name]
    src, dst, ts, neg = make_events(cfg, 0, E)
    B, M, Dm = cfg.batch, cfg.mem_dim, cfg.mail_dim
    j0, j1 = (i - 1) * B, min(i * B, len(src))
    ef = edge_features(0, j0, j1 - j0, cfg.edge_dim)
    gp = gru_params(M, Dm, cfg.time_dim)
    ap = _weights(M, Dm)
    rng = np.random.default_rng(i)
    N, S = cfg.num_nodes, oa.SLOTS
    state = oracle.new_state(N, M, cfg.edge_dim)
    state["mem"][:] = rng.uniform(-1, 1, (N, M)).astype(np.float32)
    state["mem_ts"][:] = np.minimum(rng.uniform(0, ts[j0], N), ts[j0])
    box = oa.new_mailbox(N, M, cfg.edge_dim)
    box["mb_cnt"][:] = rng.integers(0, S + 1, N)
    box["mb_pos"][:] = np.where(box["mb_cnt"] < S, box["mb_cnt"], rng.integers(0, S, N))
    box["mb"][:] = rng.uniform(-1, 1, box["mb"].shape).astype(np.float32)
    box["mb_ts"][:] = rng.uniform(0, ts[j0], box["mb_ts"].shape)
    st, _ = _stage(dev, cfg, gp, ap, src, dst, ts, neg, ef)
    st.memory.mem.copy_(_t(state["mem"], dev))
    st.memory.mem_ts.copy_(_t(state["mem_ts"], dev))
    for k in ("mb", "mb_ts", "mb_pos", "mb_cnt"):
        getattr(st.apan, k).copy_(_t(box[k], dev))
    st.apan.refresh_keys()
    x = {k: _t(v[j0:j1], dev) for k, v in dict(src=src, dst=dst, ts=ts, neg=neg).items()}
    x["ef"] = _t(ef, dev)
    st.bind_resident(x["src"], x["dst"], x["ts"], x["neg"], x["ef"])
    st.prep(1)
    st.commit(1)
    torch.cuda.synchronize()
    _C.check()
    new, nb, info = oa.step(N, src[j0:j1], dst[j0:j1], ts[j0:j1], ef, state, box, oracle.Graph(N, src, dst, ts), gp,
                            ap, fanout=cfg.fanout)
    _compare(st, new, nb)


def _compare(st, new, nb, tol=1e-4):
    assert np.array_equal(st.memory.mem_ts.cpu().numpy(), new["mem_ts"])
    dm = np.abs(st.memory.mem.cpu().numpy() - new["mem"]).max()
    assert dm <= tol, dm
    for k in ("mb_pos", "mb_cnt", "mb_ts"):
        assert np.array_equal(getattr(st.apan, k).cpu().numpy(), nb[k]), k
    db = np.abs(st.apan.mb.cpu().numpy() - nb["mb"]).max()
    assert db <= tol, db
    print(f"memory {dm:.1e}, mailbox rows {db:.1e}")


@pytest.mark.parametrize("name,nb_,k,staged", [("tiny", 50, 0, False), ("wiki", 15, 0, False), ("tiny", 30, 1, False),
                                               ("tiny", 30, 3, False), ("wiki", 12, 2, False), ("gdelt", 6, 3, False),
                                               ("reddit", 10, 1, False), ("lastfm", 10, 1, False),
                                               ("wiki", 10, 1, True)])
def test_apan_stream_free_running(dev, name, nb_, k, staged):
    """Free-running under the exact staleness schedule (k >= 1: two streams, one
    table set; the commit waits for the fetch and the APAN build of the later batch)."""
    cfg = CONFIGS[name]
    E = nb_ * cfg.batch
    src, dst, ts, neg = make_events(cfg, 0, E)
    ef = edge_features(0, 0, E, cfg.edge_dim)
    gp = gru_params(cfg.mem_dim, cfg.mail_dim, cfg.time_dim)
    ap = _weights(cfg.mem_dim, cfg.mail_dim)
    st, _ = _stage(dev, cfg, gp, ap, src, dst, ts, neg, ef, k=k)
    if staged:  # e2e: pinned host records
        st.bind_host(src, dst, ts, neg, ef)
    else:
        t = {kk: _t(v, dev) for kk, v in dict(src=src, dst=dst, ts=ts, neg=neg, ef=ef).items()}
        st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
    st.run()
    torch.cuda.synchronize()
    _C.check()
    assert [st.versions[i] for i in range(1, nb_ + 1)] == [max(0, i - 1 - k) for i in range(1, nb_ + 1)]
    new, nb = oa.run_stream(cfg.num_nodes, src, dst, ts, ef, gp, ap, cfg.batch, fanout=cfg.fanout, k=k)
    _compare(st, new, nb, tol=1e-3)
    if nb_ >= 12:
        assert int(st.apan.mb_cnt.max().item()) == oa.SLOTS  # some rings wrapped

"""Row F4 GPU parity: the training stage (mspipe_train_step / _sgd through the
C ABI) against the f64 numpy oracle (oracle/train.py) on the same seeded
inputs.  Loss, logits and every gradient tensor within
  max |g - o| <= 1e-4 max |o|   (per tensor; fp32 GEMMs and
the 3xTF32 GRU against f64), trajectories with SGD within 1e-3.  Expected
values come from oracle/ only."""
import numpy as np
import pytest
import torch

import oracle
from oracle import train as ot
from paper_2402_15113_b200 import MemoryStage, StageConfig, _C, build_tcsr
from synth import CONFIGS, edge_features, gru_params, make_events, train_params

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    d = torch.device("cuda:0")
    torch.cuda.set_device(d)
    return d


def _t(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def _random_state(num_nodes, M, src, dst, ts, j0, seed):
    rng = np.random.default_rng(seed)
    mem = rng.uniform(-1, 1, (num_nodes, M)).astype(np.float32)
    mem_ts = np.zeros(num_nodes)
    mem_ts[src[:j0]] = ts[:j0]
    last = np.zeros(num_nodes)
    last[dst[:j0]] = ts[:j0]
    return mem, np.maximum(mem_ts, last)


def _worst(g, o):
    g, o = np.asarray(g, np.float64), np.asarray(o, np.float64)
    return float(np.abs(g - o).max()) / max(float(np.abs(o).max()), 1e-30)


def _teacher_forced(dev, name, i, E, seed=0, lr=0.0, sgd=False):
    cfg = CONFIGS[name]
    src, dst, ts, neg = make_events(cfg, seed, E)
    B, F, M = cfg.batch, cfg.fanout, cfg.mem_dim
    j0, j1 = (i - 1) * B, min(i * B, len(src))
    ef = edge_features(seed, j0, j1 - j0, cfg.edge_dim)
    gp = gru_params(M, cfg.mail_dim, cfg.time_dim)
    tp = train_params(M, cfg.time_dim, 100)
    mem, mem_ts = _random_state(cfg.num_nodes, M, src, dst, ts, j0, seed + i)
    g = build_tcsr(cfg.num_nodes, src, dst, ts, dev)
    sc = StageConfig(cfg.num_nodes, M, cfg.edge_dim, cfg.time_dim, F, B, 0, fused=True,
                     train=dict(params=tp, lr=lr, sgd=sgd))
    st = MemoryStage(sc, gp, g, dev)
    st.memory.mem.copy_(_t(mem, dev))
    st.memory.mem_ts.copy_(_t(mem_ts, dev))
    x = {k: _t(v[j0:j1], dev) for k, v in dict(src=src, dst=dst, ts=ts, neg=neg).items()}
    x["ef"] = _t(ef, dev)
    st.bind_resident(x["src"], x["dst"], x["ts"], x["neg"], x["ef"])
    st.prep(1)
    st.commit(1)
    torch.cuda.synchronize()
    _C.check()
    ref = ot.train_step(cfg.num_nodes, src[j0:j1], dst[j0:j1], neg[j0:j1], ts[j0:j1], ef, mem, mem_ts,
                        oracle.Graph(cfg.num_nodes, src, dst, ts), gp, tp, fanout=F)
    return st, ref, (gp, tp)


@pytest.mark.parametrize("name,i,E", [("tiny", 1, None), ("tiny", 30, None), ("wiki", 90, 60_000),
                                      ("lastfm", 60, 60_000), ("reddit", 80, 60_000), ("gdelt", 3, 20_000)])
def test_train_step_matches_oracle(dev, name, i, E):
    st, ref, _ = _teacher_forced(dev, name, i, E)
    tr = st.trainer
    loss = float(tr.losses[0].item())
    assert abs(loss - ref["loss"]) <= TOL * abs(ref["loss"]), (loss, ref["loss"])
    B = len(ref["logit"]) // 2
    assert _worst(tr.logits[: 2 * B].cpu().numpy(), ref["logit"]) <= TOL
    report = {}
    for k in _C.TRAIN_TENSORS:
        w = _worst(tr.tensor(k, "grads").cpu().numpy(), ref["grads"][k])
        report[k] = w
        assert w <= TOL, (k, w)
        assert np.abs(ref["grads"][k]).max() > 0, k
    print(f"{name} i={i}: loss {loss:.6f} (oracle {ref['loss']:.6f}); worst grad error / max|o|:",
          {k: f"{v:.1e}" for k, v in report.items()})


def test_train_step_deterministic(dev):
    a, _, _ = _teacher_forced(dev, "wiki", 50, 40_000)
    b, _, _ = _teacher_forced(dev, "wiki", 50, 40_000)
    assert torch.equal(a.trainer.grads, b.trainer.grads)
    assert torch.equal(a.trainer.losses[:1], b.trainer.losses[:1])


def test_sgd_updates_params_and_the_updater(dev):
    """params -= lr * grads on every tensor, and the GRU's tensor-core images follow
    the master weights: a second teacher-forced GEMM with the updated weights equals
    the oracle GRU with those weights."""
    lr = 0.05
    st, ref, (gp, tp) = _teacher_forced(dev, "tiny", 5, None, lr=lr, sgd=True)
    tr = st.trainer
    for k in _C.TRAIN_TENSORS:
        p0 = tp[k] if k in tp else gp[k]
        want = (np.asarray(p0, np.float64) - lr * tr.tensor(k, "grads").cpu().numpy().astype(np.float64))
        assert np.allclose(tr.tensor(k).cpu().numpy(), want, rtol=1e-6, atol=1e-7), k
    # the updater now runs with the new weights
    new_gp = dict(gp, **{k: tr.tensor(k).cpu().numpy() for k in ("w_ih", "w_hh", "b_ih", "b_hh")})
    x = st.inputs(1)
    mem = st.memory.mem.cpu().numpy().copy()
    mem_ts = st.memory.mem_ts.cpu().numpy().copy()
    st.memory.set_committed(0)
    st.prep(1)
    st.commit(1)
    torch.cuda.synchronize()
    upd = st._upd(1)
    U = int(upd["num"].item())
    o = oracle.memory_update(CONFIGS["tiny"].num_nodes, x["src"].cpu().numpy(), x["dst"].cpu().numpy(),
                             x["ts"].cpu().numpy(), x["ef"].cpu().numpy(), new_gp, mem, mem_ts)
    got = upd["mem"][:U].cpu().numpy()
    assert np.array_equal(upd["nodes"][:U].cpu().numpy(), o["nodes"])
    assert np.all(np.abs(got - o["mem"]) <= 1e-4 * np.abs(o["mem"]) + 1e-6)


@pytest.mark.parametrize("name,k,nb,lr,tail,staged", [("tiny", 0, 12, 1e-2, 0, False), ("tiny", 1, 12, 1e-2, 0, False),
                                                      ("wiki", 1, 8, 1e-3, 0, False), ("tiny", 2, 7, 1e-2, 123, False),
                                                      ("gdelt", 3, 5, 1e-3, 0, False), ("wiki", 1, 6, 1e-3, 0, True)])
def test_training_trajectory_matches_oracle(dev, name, k, nb, lr, tail, staged):
    """Stage + training over nb batches with SGD (weights change every step,
    memory committed from the updated GRU): per-batch losses, final memory and
    final parameters against the oracle run in the same order (exact schedule:
    batch i reads S_{max(0, i-1-k)} and the weights after SGD of batch i-1)."""
    cfg = CONFIGS[name]
    E = nb * cfg.batch - tail  # tail > 0: a ragged last batch
    src, dst, ts, neg = make_events(cfg, 0, E)
    ef = edge_features(0, 0, E, cfg.edge_dim)
    M, F, B = cfg.mem_dim, cfg.fanout, cfg.batch
    gp = gru_params(M, cfg.mail_dim, cfg.time_dim)
    tp = train_params(M, cfg.time_dim, 100)
    g = build_tcsr(cfg.num_nodes, src, dst, ts, dev)
    sc = StageConfig(cfg.num_nodes, M, cfg.edge_dim, cfg.time_dim, F, B, k, fused=True, train=dict(params=tp, lr=lr))
    st = MemoryStage(sc, gp, g, dev)
    if staged:  # e2e: inputs from pinned host records, results read back (the bench's e2e path)
        st.bind_host(src, dst, ts, neg, ef)
    else:
        t = {kk: _t(v, dev) for kk, v in dict(src=src, dst=dst, ts=ts, neg=neg, ef=ef).items()}
        st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
    st.run()
    torch.cuda.synchronize()
    _C.check()
    graph = oracle.Graph(cfg.num_nodes, src, dst, ts)
    states = [oracle.new_state(cfg.num_nodes, M, cfg.edge_dim)]
    gru, prm = dict(gp), dict(tp)
    losses = []
    for i in range(1, nb + 1):
        b = slice((i - 1) * B, min(i * B, E))
        snap = states[max(0, i - 1 - k)]
        out = ot.train_step(cfg.num_nodes, src[b], dst[b], neg[b], ts[b], ef[b], snap["mem"], snap["mem_ts"], graph,
                            gru, prm, fanout=F)
        losses.append(out["loss"])
        nxt = {kk: v.copy() for kk, v in states[-1].items()}
        nxt["mem"][out["nodes"]] = out["h_new"].astype(np.float32)
        nxt["mem_ts"][out["nodes"]] = ts[b][out["winner"] >> 1]
        states.append(nxt)
        gru = ot.sgd(gru, {kk: out["grads"][kk] for kk in ot.GRU_KEYS}, lr)
        prm = ot.sgd(prm, out["grads"], lr)
    got = st.trainer.losses[:nb].cpu().numpy()
    worst = np.abs(got - np.array(losses)) / np.abs(np.array(losses))
    assert worst.max() <= 1e-3, worst
    assert np.array_equal(st.memory.mem_ts.cpu().numpy(), states[-1]["mem_ts"])
    dm = np.abs(st.memory.mem.cpu().numpy() - states[-1]["mem"]).max()
    assert dm <= 1e-3, dm
    for kk in _C.TRAIN_TENSORS:
        ref = (prm if kk in prm else gru)[kk]
        assert _worst(st.trainer.tensor(kk).cpu().numpy(), ref) <= 1e-4, kk
    print(f"{name} k={k}: losses {got[0]:.4f} -> {got[-1]:.4f}, worst loss rel err {worst.max():.1e}, memory {dm:.1e}")


def test_train_abi_errors(dev):
    cfg = CONFIGS["tiny"]
    M = cfg.mem_dim
    gp = gru_params(M, cfg.mail_dim, cfg.time_dim)
    n, _ = _C.train_layout(M, cfg.edge_dim, cfg.time_dim, 100)
    p = torch.zeros(n, device=dev)
    gr = torch.zeros(n, device=dev)
    bf = _C.GruHandle(M, cfg.edge_dim, cfg.time_dim, gp, dev, _C.BF16, max_events=200)
    with pytest.raises(_C.MspipeError) as e:
        _C.TrainHandle(bf, cfg.num_nodes, 100, 10, 200, p, gr)
    assert e.value.status == _C.EUNSUPPORTED
    tc = _C.GruHandle(M, cfg.edge_dim, cfg.time_dim, gp, dev, _C.FP32_3XTF32, max_events=200)
    with pytest.raises(_C.MspipeError) as e:
        _C.TrainHandle(tc, cfg.num_nodes, 100, 10, 400, p, gr)  # more events than the updater holds
    assert e.value.status == _C.EINVAL
    with pytest.raises(_C.MspipeError) as e:
        _C.TrainHandle(tc, cfg.num_nodes, 100, 40, 200, p, gr)  # fanout > 31
    assert e.value.status == _C.EINVAL


def test_train_single_event_batch(dev):
    """Degenerate batch: one event (2 winners, 3 roots) on a fresh stage."""
    cfg = CONFIGS["tiny"]
    src, dst, ts, neg = make_events(cfg, 0, 50)
    M = cfg.mem_dim
    gp = gru_params(M, cfg.mail_dim, cfg.time_dim)
    tp = train_params(M, cfg.time_dim, 100)
    ef = edge_features(0, 0, 50, cfg.edge_dim)
    g = build_tcsr(cfg.num_nodes, src, dst, ts, dev)
    st = MemoryStage(StageConfig(cfg.num_nodes, M, cfg.edge_dim, cfg.time_dim, cfg.fanout, 1, 0, fused=True,
                                 train=dict(params=tp, lr=0.0, sgd=False)), gp, g, dev)
    j = 40
    x = {k: _t(v[j:j + 1], dev) for k, v in dict(src=src, dst=dst, ts=ts, neg=neg, ef=ef).items()}
    st.bind_resident(x["src"], x["dst"], x["ts"], x["neg"], x["ef"])
    st.prep(1)
    st.commit(1)
    torch.cuda.synchronize()
    _C.check()
    zero = oracle.new_state(cfg.num_nodes, M, cfg.edge_dim)
    ref = ot.train_step(cfg.num_nodes, src[j:j + 1], dst[j:j + 1], neg[j:j + 1], ts[j:j + 1], ef[j:j + 1], zero["mem"],
                        zero["mem_ts"], oracle.Graph(cfg.num_nodes, src, dst, ts), gp, tp, fanout=cfg.fanout)
    assert abs(float(st.trainer.losses[0].item()) - ref["loss"]) <= TOL * ref["loss"]
    for k in _C.TRAIN_TENSORS:
        assert _worst(st.trainer.tensor(k, "grads").cpu().numpy(), ref["grads"][k]) <= TOL, k


def test_train_step_with_mitigation(dev):
    """MSPipe-S (A4) feeding the training stage: the GRU's hidden input is the
    blended row, so its backward (dW_hh, via h read from the GEMM operand) must
    follow the oracle run with the same mitigation (Reddit shape)."""
    from paper_2402_15113_b200 import gamma_quantile
    cfg = CONFIGS["reddit"]
    E, i = 60_000, 80
    src, dst, ts, neg = make_events(cfg, 0, E)
    B, F, M = cfg.batch, cfg.fanout, cfg.mem_dim
    j0, j1 = (i - 1) * B, i * B
    ef = edge_features(0, j0, B, cfg.edge_dim)
    gp = gru_params(M, cfg.mail_dim, cfg.time_dim)
    tp = train_params(M, cfg.time_dim, 100)
    mem, mem_ts = _random_state(cfg.num_nodes, M, src, dst, ts, j0, 7)
    mit = dict(lam=cfg.lam, gamma=gamma_quantile(cfg.num_nodes, src, dst, ts, cfg.quantile_p) * 0.05, n_sim=cfg.n_sim)
    g = build_tcsr(cfg.num_nodes, src, dst, ts, dev)
    st = MemoryStage(StageConfig(cfg.num_nodes, M, cfg.edge_dim, cfg.time_dim, F, B, 0, fused=True, mitigation=mit,
                                 train=dict(params=tp, lr=0.0, sgd=False)), gp, g, dev)
    st.memory.mem.copy_(_t(mem, dev))
    st.memory.mem_ts.copy_(_t(mem_ts, dev))
    x = {k: _t(v[j0:j1], dev) for k, v in dict(src=src, dst=dst, ts=ts, neg=neg).items()}
    x["ef"] = _t(ef, dev)
    st.bind_resident(x["src"], x["dst"], x["ts"], x["neg"], x["ef"])
    st.prep(1)
    st.commit(1)
    torch.cuda.synchronize()
    _C.check()
    graph = oracle.Graph(cfg.num_nodes, src, dst, ts)
    ref = ot.train_step(cfg.num_nodes, src[j0:j1], dst[j0:j1], neg[j0:j1], ts[j0:j1], ef, mem, mem_ts, graph, gp, tp,
                        fanout=F, mitigation=mit)
    plain = ot.train_step(cfg.num_nodes, src[j0:j1], dst[j0:j1], neg[j0:j1], ts[j0:j1], ef, mem, mem_ts, graph, gp,
                          tp, fanout=F)
    assert np.abs(ref["grads"]["w_hh"] - plain["grads"]["w_hh"]).max() > 0  # the blend is on the path
    assert abs(float(st.trainer.losses[0].item()) - ref["loss"]) <= TOL * ref["loss"]
    for k in _C.TRAIN_TENSORS:
        assert _worst(st.trainer.tensor(k, "grads").cpu().numpy(), ref["grads"][k]) <= TOL, k

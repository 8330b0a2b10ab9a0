"""Pins of the F1 planner oracle (oracle/planner.py) against what the paper and
plain arithmetic fix: Eq. 3-4 evaluated by hand, an independent event-driven
simulation of the same resources, brute-force minimality of the solver, the
paper's Table 1 stage shares against its Table 2 speedups
 and its "range from 2 to 4", and the stale-node fraction
against a from-scratch replay."""
import math

import numpy as np
import pytest

from oracle import planner as P

# Table `tab:breakdown`: TGN stage shares (%), and Table 2
# MSPipe speedups over TGL on the same datasets
TABLE1 = {"REDDIT": [9.5, 12.6, 5.7, 46.9, 25.3], "WIKI": [6.6, 5.8, 5.8, 51.5, 30.3],
          "MOOC": [9.7, 3.0, 2.5, 53.1, 31.7], "LASTFM": [11.5, 9.1, 8.5, 43.0, 26.8],
          "GDELT": [17.6, 12.8, 10.5, 37.5, 21.6]}
TABLE2_SPEEDUP = {"REDDIT": 1.77, "WIKI": 1.54, "MOOC": 1.50, "LASTFM": 2.00, "GDELT": 2.36}


def test_timeline_single_iteration_is_prefix_sums():
    tau = [3.0, 1.5, 2.0, 7.0, 0.5]
    b, e = P.timeline(tau, 1)
    assert np.allclose(b[1][1:], np.concatenate([[0], np.cumsum(tau)[:-1]]))
    assert np.allclose(e[1][1:], np.cumsum(tau))


def test_timeline_worked_by_hand():
    """tau = 1 everywhere, Eq. 3 as printed: iteration 1 starts (0,1,2,3,4);
    iteration 2: b^(1) = e_1^(1) = 1, b^(2) = max(e_2^(1) = 2, e_1^(3) = 3) = 3,
    b^(3) = max(e_2^(2) = 4, e_1^(3) = 3) = 4, b^(4) = max(5, 4) = 5, b^(5) = 6."""
    b, e = P.timeline([1.0] * 5, 2)
    assert b[1][1:].tolist() == [0, 1, 2, 3, 4]
    assert b[2][1:].tolist() == [1, 3, 4, 5, 6]
    assert (e - b)[1:, 1:].tolist() == [[1.0] * 5] * 2


def test_timeline_with_gate_worked_by_hand():
    """Synchronous plan k_i = 1 (TGL): fetch i waits for update i-1.
    tau = (1,1,1,1,1): b_2^(3) = max(4, 3, e_1^(5) = 5) = 5."""
    b, e = P.timeline([1.0] * 5, 2, k=[1, 1])
    assert b[2][3] == 5 and b[2][4] == 6 and b[2][5] == 7


@pytest.mark.parametrize("seed", range(6))
def test_timeline_equals_event_driven_simulation(seed):
    rng = np.random.default_rng(seed)
    for _ in range(40):
        tau = rng.uniform(1, 100, 5)
        E = int(rng.integers(1, 25))
        k = None if rng.random() < 0.3 else [int(rng.integers(1, i + 1)) for i in range(1, E + 1)]
        b, e = P.timeline(tau, E, k)
        bd, ed = P.des(tau, E, k)
        assert np.allclose(b, bd) and np.allclose(e, ed)


def _c2_holds(tau, plan_prefix, i, cand):
    """C2 for iteration i with k_i = cand, evaluated from scratch with timeline():
    e_{i-cand}^(5) <= b_i^(4) - tau^(3), b_i^(4) from the schedule with the gate of i relaxed."""
    _, e = P.timeline(tau, i, plan_prefix + [i])
    b_free, _ = P.timeline(tau, i, plan_prefix + [i])
    return e[i - cand][5] <= b_free[i][4] - tau[2]


@pytest.mark.parametrize("seed", range(4))
def test_solver_minimality_brute_force(seed):
    rng = np.random.default_rng(100 + seed)
    for _ in range(15):
        tau = list(rng.uniform(1, 100, 5))
        E, kmax = int(rng.integers(2, 20)), int(rng.integers(2, 7))
        k, status = P.solve(tau, E, kmax)
        for i in range(1, E + 1):
            cands = [c for c in range(1, min(i, kmax)) if _c2_holds(tau, k[: i - 1], i, c)]
            if cands:
                assert k[i - 1] == min(cands)
            elif i > kmax:
                assert status is not None and status[2] == "C2"


def test_steady_state_closed_form():
    """Training dominates: (k-1) tau^(4) >= tau^(3) + tau^(5) gives k = 2 for (1,1,1,100,1)."""
    k, status = P.solve([1, 1, 1, 100, 1], 30, 10)
    assert status is None and set(k[2:]) == {2}


def test_infeasible_reports_c2():
    k, status = P.solve([1, 1, 50, 2, 50], 20, 2)
    assert status is not None and status[0] == "infeasible" and status[2] == "C2"


@pytest.mark.parametrize("name", list(TABLE1))
def test_table1_rows_give_paper_k_range_and_no_stall(name):
    """minimal staleness bounds "range from 2 to 4"; under the solved
    plan training runs back to back (b_i^(4) = e_{i-1}^(4)) after warm-up, while
    the synchronous plan (k_i = 1, TGL) stalls it."""
    tau = TABLE1[name]
    E = 60
    k, status = P.solve(tau, E, 10)
    assert status is None
    assert 2 <= min(k[10:]) and max(k[10:]) <= 4
    b, e = P.timeline(tau, E, k)
    assert all(abs(b[i][4] - e[i - 1][4]) < 1e-9 for i in range(10, E + 1))
    bs, es = P.timeline(tau, E, [1] * E)
    assert any(bs[i][4] > es[i - 1][4] + 1e-9 for i in range(10, E + 1))


@pytest.mark.parametrize("name", list(TABLE1))
def test_speedup_bound_dominates_paper_speedup(name):
    """The analytic bound from Table 1's shares is >= the speedup Table 2 measured,
    and it ranks GDELT first, as Table 2 does."""
    bound = P.speedup_bound(TABLE1[name])
    assert bound >= TABLE2_SPEEDUP[name]
    assert max(TABLE1, key=lambda n: P.speedup_bound(TABLE1[n])) == "GDELT"


def test_speedup_bound_reddit_value():
    assert P.speedup_bound(TABLE1["REDDIT"]) == pytest.approx(100 / 46.9)
    assert P.speedup_bound([0, 0, 0, 5, 0]) == 1.0


def _stale_replay(src, dst, B, kk):
    """From scratch: for every batch, scan back batch by batch for each node."""
    nb = -(-len(src) // B)
    batches = [set(src[(i - 1) * B:i * B]) | set(dst[(i - 1) * B:i * B]) for i in range(1, nb + 1)]
    stale = total = 0
    for i in range(1, nb + 1):
        for v in batches[i - 1]:
            total += 1
            for d in range(1, i):
                if v in batches[i - 1 - d]:
                    stale += 1 if d <= kk - 1 else 0
                    break
    return stale / total


@pytest.mark.parametrize("seed", range(3))
def test_stale_fraction_equals_replay(seed):
    rng = np.random.default_rng(seed)
    E, N, B = 600, 40, 17
    src, dst = rng.integers(0, N, E), rng.integers(0, N, E)
    fr, hist = P.stale_fraction(src, dst, B, [1, 2, 3, 5, 9])
    for kk, f in zip([1, 2, 3, 5, 9], fr):
        assert f == pytest.approx(_stale_replay(src, dst, B, kk))
    assert fr[0] == 0.0 and all(np.diff(fr) >= 0)


def test_stale_fraction_closed_forms():
    # fresh nodes every event: nothing is ever stale
    E = 100
    fr, _ = P.stale_fraction(np.arange(E), np.arange(E) + E, 10, [2, 5])
    assert (fr == 0).all()
    # one edge repeated, one event per batch: every batch after the first re-updates {0, 1}
    fr, hist = P.stale_fraction(np.zeros(E, int), np.ones(E, int), 1, [1, 2, 3])
    assert fr.tolist() == [0.0, 2 * (E - 1) / (2 * E), 2 * (E - 1) / (2 * E)]
    assert hist == {0: 2, 1: 2 * (E - 1)}


def test_k_max_rule():
    assert P.k_max_from_fraction({1: 0.0, 2: 0.3, 3: 0.5, 4: 0.6}) == 4
    assert P.k_max_from_fraction({2: 0.9}) == 1


# ---------------------------------------------------------------- staleness error (F1 analytics)
def _bias_only(M, He, Dt, c):
    Dx = 2 * M + He + Dt
    p = dict(w_ih=np.zeros((3 * M, Dx), np.float32), w_hh=np.zeros((3 * M, M), np.float32),
             b_ih=np.zeros(3 * M, np.float32), b_hh=np.zeros(3 * M, np.float32),
             time_w=np.ones(Dt, np.float32), time_b=np.zeros(Dt, np.float32))
    p["b_ih"][2 * M:] = c
    return p


def test_staleness_error_k0_is_zero():
    """k = 0 run vs itself -> 0 for random weights."""
    import oracle
    from synth import make_workload
    w = make_workload("tiny", seed=1, num_events=3000)
    c = w["cfg"]
    e = oracle.staleness_error_series(c.num_nodes, w["src"], w["dst"], w["ts"], w["ef"], w["params"], c.batch, 0)
    assert len(e) == 15 and (e == 0.0).all()


@pytest.mark.parametrize("k,schedule", [(1, "exact"), (3, "exact"), (2, "grouped")])
def test_staleness_error_bias_only_closed_form(k, schedule):
    """Bias-only GRU (W = 0, b_in = c): a node's memory after m updates is
    tanh(c)(1 - 2^-m) (pin P4), so the error of iteration i is
    sqrt(sum_w M tanh(c)^2 (2^-m~_w - 2^-m_w)^2) over the batch's update
    targets, m~ from the stale run's integer replay read at v(i) and m from the
    k = 0 replay read at i - 1 (both written out here from Eq. 2)."""
    import oracle
    from synth import CONFIGS, edge_features, make_events
    cfg = CONFIGS["tiny"]
    E, B, N = 3000, 150, cfg.num_nodes
    src, dst, ts, _ = make_events(cfg, 4, E)
    M, He, Dt, c = 5, 3, 2, 0.8
    ef = edge_features(0, 0, E, He)
    got = oracle.staleness_error_series(N, src, dst, ts, ef, _bias_only(M, He, Dt, c), B, k, schedule)
    stale = [np.zeros(N, np.int64)]
    ref = np.zeros(N, np.int64)
    want = []
    for i in range(1, E // B + 1):
        v = max(0, i - 1 - k) if schedule == "exact" else (k + 1) * ((i - 1) // (k + 1))
        snap = stale[v]
        targets = sorted(set(src[(i - 1) * B:i * B].tolist()) | set(dst[(i - 1) * B:i * B].tolist()))
        d = np.array([2.0 ** -snap[w] - 2.0 ** -ref[w] for w in targets])
        want.append(math.sqrt(M * math.tanh(c) ** 2 * float((d * d).sum())))
        live = stale[-1].copy()
        new_ref = ref.copy()
        for a in range((i - 1) * B, i * B):
            for w in (src[a], dst[a]):
                live[w] = snap[w] + 1
                new_ref[w] = ref[w] + 1
        stale.append(live)
        ref = new_ref
    assert np.allclose(got, want, rtol=1e-6, atol=1e-6)
    assert (got > 0).any()


def test_staleness_error_mitigated_not_above_unmitigated_in_mean():
    """on a toy run with k = 2 the per-iteration series is finite and
    bounded, and the MSPipe-S series is <= the unmitigated one in mean (the
    property Fig. `fig:staleness_error` shows)."""
    import oracle
    from synth import make_workload
    w = make_workload("tiny", seed=0, num_events=6000)
    c = w["cfg"]
    mit = dict(lam=0.95, gamma=oracle.gamma(c.num_nodes, w["src"], w["dst"], w["ts"], 0.99), n_sim=5)
    a = oracle.staleness_error_series(c.num_nodes, w["src"], w["dst"], w["ts"], w["ef"], w["params"], c.batch, 2)
    b = oracle.staleness_error_series(c.num_nodes, w["src"], w["dst"], w["ts"], w["ef"], w["params"], c.batch, 2,
                                      mitigation=mit)
    assert np.isfinite(a).all() and np.isfinite(b).all()
    # |x - s| <= 2 per element (P8: memories in [-1, 1]): ||.||_F <= 2 sqrt(U M)
    assert a.max() <= 2 * math.sqrt(2 * c.batch * c.mem_dim)
    assert b.mean() <= a.mean()


def test_library_stale_fractions_equal_oracle():
    """mspipe_plan_stale_fractions (host, in the library) on the oracle's C3
    histogram gives the oracle's fractions bit for bit (reading F6)."""
    from oracle import planner as OP
    from paper_2402_15113_b200 import _C
    from synth import CONFIGS, make_events
    cfg = CONFIGS["wiki"]
    src, dst, _, _ = make_events(cfg, 2, 60_000)
    ks = list(range(1, 12))
    fr, hist = OP.stale_fraction(src, dst, 600, ks)
    max_d = 40
    h = np.zeros(max_d + 2, np.int64)
    for d, n in hist.items():
        h[min(d, max_d + 1)] += n
    assert np.array_equal(_C.plan_stale_fractions(h, ks), fr)

"""Row F1 on the library side, CPU only: the C-ABI planner (host code in
libmspipe.so) against the oracle (oracle/planner.py), and the stream order a
plan produces against the oracle's per-iteration versions."""
import numpy as np
import pytest

import oracle
from oracle import planner as P
from paper_2402_15113_b200 import _C
from paper_2402_15113_b200.stage import plan_versions, schedule_ops, snapshot_versions

from test_planner_pins import TABLE1


@pytest.mark.parametrize("seed", range(5))
def test_lib_timeline_equals_oracle(seed):
    rng = np.random.default_rng(seed)
    for _ in range(30):
        tau = rng.uniform(0, 50, 5)
        E = int(rng.integers(1, 40))
        k = None if rng.random() < 0.3 else [int(rng.integers(1, i + 1)) for i in range(1, E + 1)]
        b, e = _C.plan_timeline(tau, E, k)
        bo, eo = P.timeline(tau, E, k)
        assert np.array_equal(b, bo[1:, 1:]) and np.array_equal(e, eo[1:, 1:])


@pytest.mark.parametrize("seed", range(5))
def test_lib_solver_equals_oracle(seed):
    rng = np.random.default_rng(50 + seed)
    for _ in range(30):
        tau = list(rng.uniform(0.1, 100, 5))
        E, kmax = int(rng.integers(1, 50)), int(rng.integers(1, 8))
        k, bad = _C.plan_min_staleness(tau, E, kmax)
        ko, status = P.solve(tau, E, kmax)
        assert k.tolist() == ko
        assert bad == (0 if status is None else status[1])


@pytest.mark.parametrize("name", list(TABLE1))
def test_lib_solver_table1(name):
    k, bad = _C.plan_min_staleness(TABLE1[name], 100, 10)
    assert bad == 0 and 2 <= k[10:].min() and k[10:].max() <= 4


def test_lib_planner_errors():
    with pytest.raises(_C.MspipeError) as e:
        _C.plan_timeline([1, 1, -1, 1, 1], 3)
    assert e.value.status == _C.EINVAL
    with pytest.raises(_C.MspipeError) as e:
        _C.plan_timeline([1] * 5, 3, [1, 0, 1])
    assert e.value.status == _C.EINVAL
    with pytest.raises(_C.MspipeError) as e:
        _C.plan_min_staleness([1] * 5, 3, 0)
    assert e.value.status == _C.EINVAL


@pytest.mark.parametrize("seed", range(4))
def test_plan_schedule_reads_the_oracle_versions(seed):
    """schedule "plan" enqueues prep(i) right after commit(v(i)); the versions the
    stream order reads equal the oracle's v(i) = max(0, i - k_i)."""
    rng = np.random.default_rng(seed)
    nb, K = 40, 4
    plan = [min(i, int(rng.integers(1, K + 1))) if i > 1 else 1 for i in range(1, nb + 1)]
    v = snapshot_versions(nb, K - 1, "plan", plan)
    assert v == plan_versions(plan, nb)
    ops = schedule_ops(nb, K - 1, "plan", plan)
    assert [i for o, i in ops if o == "commit"] == list(range(1, nb + 1))
    seen = set()
    for o, i in ops:
        if o == "commit":
            assert i in seen
        seen.add(i)
    # the oracle's stream under the same plan reports the same versions
    w_src = rng.integers(0, 30, nb * 5).astype(np.int32)
    w_dst = rng.integers(0, 30, nb * 5).astype(np.int32)
    ts = np.arange(nb * 5, dtype=np.float64)
    M, He, Dt = 8, 4, 4
    params = dict(w_ih=np.zeros((3 * M, 2 * M + He + Dt), np.float32), w_hh=np.zeros((3 * M, M), np.float32),
                  b_ih=np.zeros(3 * M, np.float32), b_hh=np.zeros(3 * M, np.float32),
                  time_w=np.ones(Dt, np.float32), time_b=np.zeros(Dt, np.float32))
    _, vers = oracle.run_stream(30, w_src, w_dst, ts, np.zeros((nb * 5, He), np.float32), params, 5, K - 1,
                                plan=plan)
    assert vers.tolist() == v
    with pytest.raises(ValueError):
        schedule_ops(nb, 1, "plan", plan)  # K - 1 = 3 needed

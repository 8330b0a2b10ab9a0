"""Oracle for SURVEY.md §8 row F1: the minimal-staleness planner (MSPipe §3.2).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import this module.  It shares no code
with the library (paper_2402_15113_b200/csrc/planner.cpp, stale.cu).

Plain Python, written from PAPER.md in the paper's notation (P:Lnnn = line):

* ``timeline``   Eq. 3-4: start/end times b_i^(j), e_i^(j) of the
                 five stages j = 1..5 (sample, fetch feature, fetch memory, train,
                 update memory) of iterations i = 1..E, plus the staleness gate
                 of Alg. 1 L8-L11 when a plan k_i is given.
* ``des``        the same schedule from an event-driven simulation of the
                 resources of Fig. 5 / P:L230-L233 (an independent formulation,
                 used to pin ``timeline``).
* ``solve``      the optimisation of P:L300-L307: minimal k_i subject to C1-C3.
* ``stale_fraction`` Fig. `fig:overlap` / C3: share of the nodes a batch
                 updates whose memory is stale under staleness k.
* ``speedup_bound``, ``bubbles``: analysis helpers (F1).

Readings (F-readings):
  F1  paper staleness k_i (>= 1; k = 1 is "TGL without staleness");
      iteration i fetches memory updated through iteration i - k_i.
  F2  C1 is the gate of Alg. 1 (``while i - i_upd > k_i: wait``): the fetch of
      iteration i starts no earlier than e_{i-k_i}^(5); P:L293 prints the
      inequality the other way round, the prose and Alg. 1 fix this reading.
  F3  C2 is checked against the training start of the ungated schedule:
      e_{i-k}^(5) <= b_i^(4) - tau^(3) with b_i^(4) computed with the gate of
      iteration i relaxed (the fetch then fits before training, no stall).
  F4  iterations with no k in [1, min(i, k_max)) (i = 1, and any i <= the
      first feasible window) are warm-up: they fetch with k_i = i (the initial
      state, "will not wait").
  F5  C3: k_max = 1 + max{k : stale_fraction(k) <= 0.5}, so every allowed
      k_i < k_max keeps the stale share within 50 %.
  F6  stale nodes of batch i under staleness k: the distinct src/dst nodes of
      the batch whose previous update happened in iterations i-k+1 .. i-1
      (those commits are not yet visible to a fetch of version i-k).
"""
from __future__ import annotations

import heapq

import numpy as np

STAGES = ("sample", "fetch_feature", "fetch_memory", "train", "update_memory")


def timeline(tau, E, k=None):
    """Eq. 3-4.  tau: 5 stage durations; k: None (Eq. 3 as printed, no memory
    gate) or per-iteration k_i (list indexed i-1).  Returns (b, e), arrays
    [E+1, 6] with row 0 / column 0 unused (1-based i and j as in the paper)."""
    b = np.zeros((E + 1, 6))
    e = np.zeros((E + 1, 6))
    for i in range(1, E + 1):
        for j in range(1, 6):
            if j == 1:
                start = e[i - 1][1]                               # b_i^(1) = e_{i-1}^(1)
            elif j == 2:
                start = max(e[i][1], e[i - 1][3])                 # PCIe shared with stage 3
            else:
                start = max(e[i][j - 1], e[i - 1][j])             # j in [3, 5]
            if j == 3 and k is not None:
                ki = k[i - 1]
                if i - ki >= 1:
                    start = max(start, e[i - ki][5])              # Alg. 1 L8-L11 gate (F2)
            b[i][j] = start
            e[i][j] = start + tau[j - 1]
    return b, e


def des(tau, E, k=None):
    """Event-driven simulation of the same pipeline: resources sampler (stage 1),
    PCIe (stages 2 and 3, FIFO over (i, j)), GPU (stage 4), D2H (stage 5);
    a stage starts when its resource is free, the previous stage of its
    iteration is done and (stage 3) the gate i - i_upd <= k_i holds."""
    res_of = {1: "sampler", 2: "pcie", 3: "pcie", 4: "gpu", 5: "d2h"}
    queues = {"sampler": [(i, 1) for i in range(1, E + 1)],
              "pcie": [(i, j) for i in range(1, E + 1) for j in (2, 3)],
              "gpu": [(i, 4) for i in range(1, E + 1)],
              "d2h": [(i, 5) for i in range(1, E + 1)]}
    head = {r: 0 for r in queues}
    busy_until = {r: 0.0 for r in queues}
    busy = {r: False for r in queues}
    done = {}
    b = np.zeros((E + 1, 6))
    e = np.zeros((E + 1, 6))
    ev = []  # (time, seq, resource, (i, j)) completions
    seq = 0
    now = 0.0
    i_upd_time = {0: 0.0}  # iteration -> time its update finished

    def ready(i, j, t):
        if j > 1 and (i, j - 1) not in done:
            return False
        if j == 3 and k is not None and i - k[i - 1] >= 1:
            if (i - k[i - 1], 5) not in done:
                return False
        return True

    def start_of(i, j):
        t = busy_until[res_of[j]]
        if j > 1:
            t = max(t, done[(i, j - 1)])
        if j == 3 and k is not None and i - k[i - 1] >= 1:
            t = max(t, done[(i - k[i - 1], 5)])
        return t

    while len(done) < 5 * E:
        progressed = True
        while progressed:
            progressed = False
            for r, q in queues.items():
                if busy[r] or head[r] >= len(q):
                    continue
                i, j = q[head[r]]
                if ready(i, j, now):
                    t0 = start_of(i, j)
                    b[i][j] = t0
                    e[i][j] = t0 + tau[j - 1]
                    busy[r] = True
                    head[r] += 1
                    heapq.heappush(ev, (e[i][j], seq, r, (i, j)))
                    seq += 1
                    progressed = True
        if not ev:
            raise RuntimeError("deadlock")
        t, _, r, (i, j) = heapq.heappop(ev)
        now = t
        busy[r] = False
        busy_until[r] = t
        done[(i, j)] = t
        if j == 5:
            i_upd_time[i] = t
    return b, e


def solve(tau, E, k_max):
    """per i, the minimal k_i in [1, min(i, k_max)) with C2
    e_{i-k}^(5) <= b_i^(4) - tau^(3), where b_i^(4) is the training start with
    iteration i's gate relaxed (F3); C1 is then enforced as the gate.  Warm-up
    iterations (no k in range) get k_i = i (F4).  Returns (k list, status)
    where status is None or ("infeasible", i, "C2")."""
    k = []
    b = np.zeros((E + 1, 6))
    e = np.zeros((E + 1, 6))

    def stage_times(i, ki):
        bi, ei = np.zeros(6), np.zeros(6)
        for j in range(1, 6):
            if j == 1:
                s = e[i - 1][1]
            elif j == 2:
                s = max(ei[1], e[i - 1][3])
            else:
                s = max(ei[j - 1], e[i - 1][j])
            if j == 3 and ki is not None and i - ki >= 1:
                s = max(s, e[i - ki][5])
            bi[j], ei[j] = s, s + tau[j - 1]
        return bi, ei

    status = None
    for i in range(1, E + 1):
        b_free, _ = stage_times(i, None)  # gate relaxed
        hi = min(i, k_max)
        chosen = None
        for cand in range(1, hi):  # 1 <= k_i < min(i, k_max)
            if e[i - cand][5] <= b_free[4] - tau[2]:
                chosen = cand
                break
        if chosen is None:
            if hi > 1 and status is None and i > k_max:
                status = ("infeasible", i, "C2")
            chosen = i if hi <= 1 or i <= k_max else hi - 1
        k.append(chosen)
        b[i], e[i] = stage_times(i, chosen)
    return k, status


def bubbles(b, e):
    """gap_i^(j) = b_i^(j) - max(e_i^(j-1), e_{i-1}^(j)) (>= 0), j = 2..5 (stage
    2's resource predecessor is e_{i-1}^(3))."""
    E = b.shape[0] - 1
    g = np.zeros((E + 1, 6))
    for i in range(1, E + 1):
        for j in range(2, 6):
            prev = e[i - 1][3] if j == 2 else e[i - 1][j]
            g[i][j] = b[i][j] - max(e[i][j - 1], prev)
    return g


def speedup_bound(tau):
    """Serial time over the steady-state period of the pipelined schedule: the
    busiest resource per iteration (stage 1; stages 2 + 3 on PCIe; 4; 5)."""
    t = list(tau)
    return sum(t) / max(t[0], t[1] + t[2], t[3], t[4])


def stale_fraction(src, dst, batch, k_values):
    """F6: for each k in k_values, sum over batches of the distinct src/dst
    nodes whose previous update is in iterations i-k+1..i-1, over the sum of
    distinct src/dst nodes per batch.  Returns (fractions, hist) where hist[d]
    counts (batch, node) pairs whose previous update was d iterations earlier
    (d = 0: never updated before)."""
    src = np.asarray(src)
    dst = np.asarray(dst)
    n = int(max(src.max(initial=0), dst.max(initial=0))) + 1
    last = np.zeros(n, np.int64)  # iteration of the last update, 0 = none
    E = len(src)
    nb = -(-E // batch)
    hist = {}
    total = 0
    for i in range(1, nb + 1):
        j0, j1 = (i - 1) * batch, min(i * batch, E)
        nodes = np.unique(np.concatenate([src[j0:j1], dst[j0:j1]]))
        prev = last[nodes]
        d = np.where(prev > 0, i - prev, 0)
        for x in d:
            hist[int(x)] = hist.get(int(x), 0) + 1
        total += len(nodes)
        last[nodes] = i
    fr = []
    for kk in k_values:
        stale = sum(c for d, c in hist.items() if 1 <= d <= kk - 1)
        fr.append(stale / total if total else 0.0)
    return np.array(fr), hist


def k_max_from_fraction(fractions_by_k: dict):
    """F5: 1 + the largest k whose stale fraction is <= 50 %."""
    ok = [kk for kk, f in fractions_by_k.items() if f <= 0.5]
    return 1 + max(ok) if ok else 1

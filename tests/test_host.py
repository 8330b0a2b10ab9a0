"""CPU-only checks of the host logic and of the C-ABI library's surface
(no compute calls: there is no GPU here)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from paper_2402_15113_b200 import _C, build_tcsr_host, gamma_quantile, schedule_ops, snapshot_versions
from synth import CONFIGS, make_events

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    names = set()
    for f in os.listdir(os.path.join(ROOT, "include")):
        if f.endswith(".h"):
            txt = open(os.path.join(ROOT, "include", f)).read()
            names |= set(re.findall(r"MSPIPE_API\s+[\w\s\*]+?\b(mspipe_\w+)\s*\(", txt))
    return names


def test_library_exports_every_declared_symbol():
    from paper_2402_15113_b200.build import build
    build()
    lib = _C.lib()  # loads and checks the ABI version (host-only call)
    declared = _declared_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert set(_C.EXPORTS) == declared
    assert lib.mspipe_abi_version() == _C.ABI_VERSION


def test_library_is_sm100a_only():
    from paper_2402_15113_b200.build import LIB
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_host_status_paths_without_gpu():
    """Argument validation returns statuses before any CUDA call."""
    lib = _C.lib()
    h = ctypes.c_void_p()
    rc = lib.mspipe_memory_create(ctypes.byref(h), 10, 6, 4, 0, None, None, None, None, 16, 0, 1, None)
    assert rc == _C.EINVAL and "mem_dim" in _C.last_error()
    rc = lib.mspipe_memory_create(ctypes.byref(h), 10, 8, 4, 0, ctypes.c_void_p(16), ctypes.c_void_p(16),
                                  ctypes.c_void_p(16), ctypes.c_void_p(16), 20, 2, 2, None)
    assert rc == _C.EINVAL and "rank" in _C.last_error()  # rank outside [0, world)
    rc = lib.mspipe_sample_recent(None, None, None, 1, 10, None, None, None, None, None, None, None)
    assert rc == _C.EINVAL
    rc = lib.mspipe_shard_loopback(None, 2, 0, None)
    assert rc == _C.EINVAL
    rc = lib.mspipe_shard_exchange(None, 0, None)
    assert rc == _C.EINVAL


def test_shard_partition_tiles_the_global_batch():
    """Row E host logic: the G local batches of iteration i tile [(i-1)GB, iGB) and
    key_base + local pair index = global pair index of the single-GPU batch G·B."""
    from paper_2402_15113_b200.shard import key_base, local_range, num_global_batches
    for G in (1, 2, 3, 8):
        for E, B in ((10_000, 200), (1234, 50), (7, 3)):
            nb = num_global_batches(E, G, B)
            covered = []
            for i in range(1, nb + 1):
                for g in range(G):
                    j0, j1 = local_range(i, g, G, B, E)
                    covered.extend(range(j0, j1))
                    for a in range(j1 - j0):
                        for role in (0, 1):
                            assert key_base(i, g, G, B) + 2 * a + role == 2 * (j0 + a) + role
            assert covered == list(range(E))


@pytest.mark.parametrize("schedule", ["exact", "grouped"])
@pytest.mark.parametrize("k", [0, 1, 2, 3, 5])
def test_schedule_reads_the_oracle_version(k, schedule):
    """The stream order of prep/commit realises v(i) of the oracle (G8) and
    satisfies the gate i-1-k <= v(i) <= i-1."""
    for nb in (1, 2, 3, 7, 20):
        v = snapshot_versions(nb, k, schedule)
        assert v == [oracle.snapshot_version(i, k, schedule) for i in range(1, nb + 1)]
        ops = schedule_ops(nb, k, schedule)
        assert sorted(i for o, i in ops if o == "commit") == list(range(1, nb + 1))
        assert [i for o, i in ops if o == "commit"] == list(range(1, nb + 1))  # commits in order
        seen = set()
        for o, i in ops:
            if o == "commit":
                assert i in seen  # prepared before committed
            seen.add(i)


def test_tcsr_rows_are_time_sorted_incident_lists():
    cfg = CONFIGS["tiny"]
    src, dst, ts, _ = make_events(cfg, 0, 5000)
    h = build_tcsr_host(cfg.num_nodes, src, dst, ts)
    deg = np.bincount(src, minlength=cfg.num_nodes) + np.bincount(dst[dst != src], minlength=cfg.num_nodes)
    assert np.array_equal(np.diff(h["indptr"]), deg)
    for v in range(0, cfg.num_nodes, 7):
        a, b = h["indptr"][v], h["indptr"][v + 1]
        e = h["eid"][a:b]
        assert (np.diff(e) > 0).all()
        assert np.array_equal(h["ts"][a:b], ts[e])
        assert ((src[e] == v) | (dst[e] == v)).all()
        assert np.array_equal(h["nbr"][a:b], np.where(src[e] == v, dst[e], src[e]))
    # the device builder (torch sort; run here on the CPU) gives the same arrays
    from paper_2402_15113_b200.graph import build_tcsr_torch
    t = build_tcsr_torch(cfg.num_nodes, src, dst, ts, "cpu")
    for key in ("indptr", "nbr", "eid", "ts"):
        assert np.array_equal(t[key].numpy(), h[key]), key


@pytest.mark.parametrize("name", ["wiki", "reddit"])
def test_gamma_helper_matches_oracle(name):
    cfg = CONFIGS[name]
    src, dst, ts, _ = make_events(cfg, 0, 100_000)
    assert gamma_quantile(cfg.num_nodes, src, dst, ts, 0.99) == oracle.gamma(cfg.num_nodes, src, dst, ts, 0.99)


def test_header_is_plain_c(tmp_path):
    """include/mspipe.h is a C ABI: it compiles as strict C11 (gcc -pedantic) and as C++17."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        import pytest
        pytest.skip("no gcc")
    inc = os.path.join(ROOT, "include")
    src = tmp_path / "h.c"
    src.write_text('#include "mspipe.h"\nint main(void) { return mspipe_abi_version() == MSPIPE_ABI_VERSION ? 0 : 1; }\n')
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I", inc, "-c", str(src), "-o",
                    str(tmp_path / "h.o")], check=True)
    subprocess.run(["g++", "-std=c++17", "-Wall", "-Werror", "-I", inc, "-x", "c++", "-c", str(src), "-o",
                    str(tmp_path / "h2.o")], check=True)

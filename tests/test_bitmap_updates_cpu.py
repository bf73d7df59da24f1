"""The device allocator's pending-update queue (csrc/bitmap_updates.hpp) on a
CPU-only box, through a test-only C shim (tests/native/bitmap_shim.cpp, g++).

Model: a host shadow (the set of free ids, lowest-first allocation, R2) and a
simulated device bitmap that only changes when a batch of taken updates is
applied -- in a random order, as the GPU's atomics would.  Host frees call
on_free; host-side allocations (mp_alloc_mem, no kernel) call on_claim; a
"device scan" (a transfer's receiver allocation) first applies every pending
update, then takes the lowest set bits, which must be exactly the host's
lowest-first choice.  After every application the simulated bitmap must equal
the host's free set, and every taken batch must touch each id at most once
(frees and claims are order-free)."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "tests", "native", "bitmap_shim.cpp")
CSRC = os.path.join(ROOT, "paper_2406_17565_b200", "csrc")


@pytest.fixture(scope="module")
def lib(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("bu") / "bu.so")
    subprocess.run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-I", CSRC, SHIM, "-o", out],
                   check=True)
    L = C.CDLL(out)
    L.bu_new.restype = C.c_void_p
    L.bu_new.argtypes = [C.c_int64]
    L.bu_free.argtypes = [C.c_void_p]
    L.bu_on_free.argtypes = [C.c_void_p, C.c_int32]
    L.bu_on_claim.argtypes = [C.c_void_p, C.c_int32]
    L.bu_queued.restype = C.c_int64
    L.bu_queued.argtypes = [C.c_void_p]
    L.bu_compact.argtypes = [C.c_void_p]
    L.bu_take.restype = C.c_int64
    L.bu_take.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    return L


def take(L, u, cap):
    buf = np.zeros(max(cap, 1), np.int32)
    k = L.bu_take(u, buf.ctypes.data, len(buf))
    assert k >= 0
    return buf[:k]


def apply(device, upd, rng):
    ids = np.where(upd >= 0, upd, -upd - 1)
    assert len(set(ids.tolist())) == len(ids), "an id updated twice in one batch"
    for e in rng.permutation(upd):           # any order: the GPU applies them with atomics
        if e >= 0:
            assert not device[e], "free of a bit already set"
            device[e] = True
        else:
            assert device[-e - 1], "claim of a bit already clear"
            device[-e - 1] = False


@pytest.mark.parametrize("seed", range(6))
def test_queue_keeps_device_bitmap_equal_to_host_shadow(lib, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.choice([64, 300, 1024]))
    u = lib.bu_new(n)
    host_free = np.ones(n, bool)              # host shadow: True = free
    device = np.ones(n, bool)                 # simulated device bitmap
    owned = []
    for step in range(1500):
        op = rng.integers(0, 10)
        nfree = int(host_free.sum())
        if op < 4 and nfree:                  # mp_alloc_mem: host picks, device learns later
            k = int(rng.integers(1, min(nfree, 40) + 1))
            ids = np.flatnonzero(host_free)[:k]
            host_free[ids] = False
            for i in ids:
                lib.bu_on_claim(u, int(i))
            owned += ids.tolist()
        elif op < 8 and owned:                # free_mem / eviction: any owned ids
            sel = rng.random(len(owned)) < rng.uniform(0.05, 0.6)
            for i, s in zip(owned, sel):
                if s:
                    host_free[i] = True
                    lib.bu_on_free(u, int(i))
            owned = [i for i, s in zip(owned, sel) if not s]
        elif op == 8 and nfree:               # device scan: apply pending, lowest set bits
            apply(device, take(lib, u, 4 * n), rng)
            assert np.array_equal(device, host_free)
            k = int(rng.integers(1, min(nfree, 40) + 1))
            dev_pick = np.flatnonzero(device)[:k]
            host_pick = np.flatnonzero(host_free)[:k]
            assert np.array_equal(dev_pick, host_pick)  # R2 lowest-first on both sides
            device[dev_pick] = False
            host_free[host_pick] = False
            owned += host_pick.tolist()
        elif rng.random() < 0.5:              # a sync: the queue is flushed
            apply(device, take(lib, u, 4 * n), rng)
            assert np.array_equal(device, host_free)
        else:                                 # host-side compaction: nothing applied
            lib.bu_compact(u)
            assert lib.bu_queued(u) <= n      # one entry per block at most
        assert lib.bu_queued(u) <= 4 * n
    apply(device, take(lib, u, 4 * n), rng)
    assert np.array_equal(device, host_free)
    lib.bu_free(u)


def test_cancellation_leaves_nothing_to_apply(lib):
    u = lib.bu_new(16)
    lib.bu_on_claim(u, 3)
    lib.bu_on_free(u, 3)                      # claim then free before any apply
    lib.bu_on_free(u, 5)
    lib.bu_on_claim(u, 5)                     # free then re-claim
    assert list(take(lib, u, 16)) == []
    lib.bu_on_claim(u, 7)
    lib.bu_on_free(u, 7)
    lib.bu_on_claim(u, 7)                     # net: one claim
    assert list(take(lib, u, 16)) == [-8]
    lib.bu_free(u)


def test_compaction_keeps_live_updates_once(lib):
    """compact() (host only) drops stale and duplicate entries: taking after
    it gives the same updates as taking without it, each id once."""
    rng = np.random.default_rng(11)
    for _ in range(50):
        n = 200
        a, b = lib.bu_new(n), lib.bu_new(n)
        for _ in range(int(rng.integers(10, 400))):
            i = int(rng.integers(n))
            f = lib.bu_on_free if rng.random() < 0.5 else lib.bu_on_claim
            f(a, i)
            f(b, i)
        lib.bu_compact(b)
        assert lib.bu_queued(b) <= n
        ta, tb = take(lib, a, 4 * n), take(lib, b, 4 * n)
        assert sorted(ta.tolist()) == sorted(tb.tolist())
        assert len(set(np.where(tb >= 0, tb, -tb - 1).tolist())) == len(tb)
        lib.bu_free(a)
        lib.bu_free(b)

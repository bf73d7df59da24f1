"""The product's host prompt index (paper_2406_17565_b200/csrc/index.hpp) on a
CPU-only box, through a test-only C shim (tests/native/index_shim.cpp, built
with g++ -- no CUDA), against the oracle's prefix map on randomized
insert / match(pin) / delete / evict / swap-victim sequences (S:632 shape:
<= 100 stored sequences, lengths <= 512, B in {8, 16}).

Compared exactly after every op: duplicate blocks of an insert (R4
keep-existing), matched prefixes (R5), blocks unlinked by delete and whether
they are freed or orphaned (R6), LRU eviction order (R8), the HBM-frontier
swap victim (R9), the eviction-feasibility count (R2), the logical clock (R7),
and the full index dump (prefix tokens, medium, block, last_access, ref,
terminal)."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "tests", "native", "index_shim.cpp")
CSRC = os.path.join(ROOT, "paper_2406_17565_b200", "csrc")


@pytest.fixture(scope="module")
def lib(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("ix") / "ix.so")
    subprocess.run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-I", CSRC, SHIM, "-o", out],
                   check=True)
    L = C.CDLL(out)
    P = C.c_void_p
    pi = C.POINTER(C.c_int32)
    L.ix_new.restype = P
    L.ix_new.argtypes = [C.c_int, C.c_int64, C.c_int64]
    L.ix_free.argtypes = [P]
    L.ix_clock.restype = C.c_uint64
    L.ix_clock.argtypes = [P]
    L.ix_insert.restype = C.c_int64
    L.ix_insert.argtypes = [P, pi, C.c_int64, pi, pi, pi, pi]
    L.ix_match.restype = C.c_int64
    L.ix_match.argtypes = [P, pi, C.c_int64, C.c_int, pi, pi]
    L.ix_erase.restype = C.c_int64
    L.ix_erase.argtypes = [P, pi, C.c_int64, pi, pi, pi]
    L.ix_evict.restype = C.c_int
    L.ix_evict.argtypes = [P, C.c_int, pi]
    L.ix_frontier.restype = C.c_int
    L.ix_frontier.argtypes = [P, pi]
    L.ix_rebind.argtypes = [P, C.c_int, C.c_int32, C.c_int, C.c_int32]
    L.ix_evictable.restype = C.c_int64
    L.ix_evictable.argtypes = [P, C.c_int]
    L.ix_evictable_leaves.restype = C.c_int64
    L.ix_evictable_leaves.argtypes = [P, C.c_int]
    L.ix_evictable_pinned.restype = C.c_int64
    L.ix_evictable_pinned.argtypes = [P, C.c_int, C.POINTER(C.c_int32), C.c_int64,
                                      C.POINTER(C.c_int)]
    L.ix_evictable_at_least.restype = C.c_int
    L.ix_evictable_at_least.argtypes = [P, C.c_int, C.c_int64]
    L.ix_dump.restype = C.c_int64
    L.ix_dump.argtypes = [P, C.c_char_p, C.c_int64]
    return L


def arr(x, dtype=np.int32):
    a = np.ascontiguousarray(np.asarray(x, dtype=dtype))
    return a, a.ctypes.data_as(C.POINTER(C.c_int32))


def dump(L, h):
    n = L.ix_dump(h, None, 0)
    buf = C.create_string_buffer(n + 1)
    L.ix_dump(h, buf, n + 1)
    rows = []
    for line in buf.value.decode().splitlines():
        d, med, idx, la, ref, term, toks = line.split("\t")
        rows.append((tuple(int(x) for x in toks.split(",")), int(med), int(idx), int(la),
                     int(ref), term == "1"))
    return sorted(rows)


def gen(rng, stored, vocab, maxlen):
    if stored and rng.random() < 0.7:
        base = stored[rng.integers(len(stored))]
        cut = int(rng.integers(0, len(base) + 1))
        tail = rng.integers(0, vocab, size=int(rng.integers(0, max(1, maxlen - cut + 1))))
        return np.concatenate([np.asarray(base[:cut], np.int32), tail.astype(np.int32)])
    return rng.integers(0, vocab, size=int(rng.integers(0, maxlen + 1))).astype(np.int32)


def run(L, seed, B, n_ops):
    rng = np.random.default_rng(seed)
    pool = O.OraclePool(0, 1, 1, 8, B, n_hbm=6000, n_dram=6000)
    h = L.ix_new(B, 6000, 6000)
    stored = []
    vocab = int(rng.integers(2, 6))
    scratch = [np.zeros(600, np.int32) for _ in range(3)]
    ptrs = [s.ctypes.data_as(C.POINTER(C.c_int32)) for s in scratch]
    try:
        for step in range(n_ops):
            op = rng.random()
            if op < 0.35 and len(stored) < 100:
                t = gen(rng, stored, vocab, 512 if rng.random() < 0.2 else 96)
                k = len(t) // B
                addrs = pool.alloc_mem(k, O.HBM)
                ta, tp = arr(t)
                med, mp_ = arr([a[1] for a in addrs] or [0])
                idx, ip = arr([a[2] for a in addrs] or [0])
                before = list(pool.state[O.HBM])
                pool.insert(t, addrs)
                want = [a[2] for a in addrs if pool.state[O.HBM][a[2]] == O.FREE]
                nd = L.ix_insert(h, tp, len(t), mp_, ip, ptrs[0], ptrs[1])
                assert list(scratch[1][:nd]) == want
                if k:
                    stored.append(t[: k * B])
            elif op < 0.6:
                t = gen(rng, stored, vocab, 128)
                pin = rng.random() < 0.2
                mt, addrs = pool.match(t, O.FLAG_MATCH_PIN if pin else 0)
                ta, tp = arr(t)
                k = L.ix_match(h, tp, len(t), int(pin), ptrs[0], ptrs[1])
                assert k * B == mt
                assert [(int(scratch[0][i]), int(scratch[1][i])) for i in range(k)] == \
                       [(a[1], a[2]) for a in addrs]
            elif op < 0.75 and stored:
                t = stored[rng.integers(len(stored))]
                before = {m: list(pool.state[m]) for m in (O.HBM, O.DRAM)}
                pool.delete(t)
                gone = sorted((m, i) for m in (O.HBM, O.DRAM)
                              for i, (a, b) in enumerate(zip(before[m], pool.state[m]))
                              if a == O.INDEXED and b != O.INDEXED)
                ta, tp = arr(t)
                n = L.ix_erase(h, tp, len(t), ptrs[0], ptrs[1], ptrs[2])
                got = sorted((int(scratch[0][i]), int(scratch[1][i])) for i in range(n))
                assert got == gone
                for i in range(n):
                    m, x, ref = int(scratch[0][i]), int(scratch[1][i]), int(scratch[2][i])
                    assert pool.state[m][x] == (O.FREE if ref == 0 else O.ORPHAN)
            elif op < 0.85:
                med = int(rng.integers(2))
                n = int(rng.integers(1, 6))
                want = [a[2] for a in pool.evict(n, med)]
                got = []
                x = C.c_int32(0)
                for _ in range(n):
                    if not L.ix_evict(h, med, C.byref(x)):
                        break
                    got.append(x.value)
                assert got == want
            else:
                moved = pool.swap_out(1)
                x = C.c_int32(0)
                have = L.ix_frontier(h, C.byref(x))
                if moved:
                    (old, new), = moved
                    assert have and x.value == old[2]
                    L.ix_rebind(h, O.HBM, old[2], O.DRAM, new[2])
                else:
                    assert not have
            assert L.ix_clock(h) == pool.clock
            if step % 20 == 0:
                for med in (O.HBM, O.DRAM):
                    trial = pool._clone_meta()
                    full = len(trial._evict(10 ** 9, med))
                    assert L.ix_evictable(h, med) == full
                    # the fast feasibility bound (unpinned leaves) never over-promises
                    assert 0 <= L.ix_evictable_leaves(h, med) <= full
                    # the early-stopping peel decides "at least k" exactly
                    for k in {0, 1, full // 2, full, full + 1}:
                        assert L.ix_evictable_at_least(h, med, k) == (full >= k)
                    if stored:   # with a stored prefix pinned (the receiver's match, R12)
                        t = stored[rng.integers(len(stored))]
                        t = t[: int(rng.integers(0, len(t) + 1))]
                        ta, tp = arr(t)
                        agree = C.c_int(0)
                        L.ix_evictable_pinned(h, med, tp, len(t), C.byref(agree))
                        assert agree.value == 1
        assert dump(L, h) == pool.dump_index()
    finally:
        L.ix_free(h)


@pytest.mark.parametrize("B", [8, 16, 32])
def test_index_vs_oracle(lib, B):
    for seed in range(25):
        run(lib, 1000 * B + seed, B, 60)


def test_index_long_runs(lib):
    """Long op sequences: the child table grows past its initial size and the
    path memo is invalidated by many deletes / evictions in between."""
    for seed in range(2):
        run(lib, 77 + seed, 8, 250)

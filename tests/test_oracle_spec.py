"""Oracle vs SPEC.md's worked examples and the kvgen generator's
published splitmix64 test vectors.  Each test cites the SPEC example it pins."""
import numpy as np
import pytest

from oracle import (HBM, DRAM, MIXED, FREE, MPError, OraclePool, FLAG_MATCH_PIN,
                    FLAG_INS_ERR_ON_CONFLICT)
from workloads import kvgen


def mk(n_hbm=100, n_dram=10, B=16, inst=0):
    return OraclePool(inst, 2, 2, 64, B, n_hbm=n_hbm, n_dram=n_dram, seed=1)


def T(*r):
    return np.arange(*r, dtype=np.int32)


def test_splitmix64_vectors():
    # Vigna's splitmix64 with state 0: successive outputs are
    # 0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4 (reference C implementation).
    g = 0x9E3779B97F4A7C15
    out = kvgen.splitmix64(np.array([0, g], dtype=np.uint64))
    assert int(out[0]) == 0xE220A8397B1DCDAF
    assert int(out[1]) == 0x6E789E6AA1B965F4


def test_alloc_examples():
    p = mk()
    # S:131 (3, HBM) on a fresh pool of 100 -> {0,1,2}
    assert [a[2] for a in p.alloc_mem(3, HBM)] == [0, 1, 2]
    # S:132 (5, Mixed) with 2 HBM free, 10 DRAM free -> 2 HBM + 3 DRAM
    q = mk(n_hbm=2, n_dram=10)
    out = q.alloc_mem(5, MIXED)
    assert [(a[1], a[2]) for a in out] == [(HBM, 0), (HBM, 1), (DRAM, 0), (DRAM, 1), (DRAM, 2)]
    # S:133 (1, HBM) with 0 free and all blocks pinned -> OOM
    r = mk(n_hbm=2, n_dram=0)
    a = r.alloc_mem(2, HBM)
    r.insert(T(0, 32), a)
    r.match(T(0, 32), flags=FLAG_MATCH_PIN)
    with pytest.raises(MPError) as e:
        r.alloc_mem(1, HBM)
    assert e.value.name == "OOM"


def test_free_examples():
    p = mk()
    before = list(p.state[HBM])
    a = p.alloc_mem(3, HBM)
    p.free_mem(a)                       # S:141 round trip
    assert p.state[HBM] == before
    a = p.alloc_mem(3, HBM)
    p.free_mem(a[:1])                   # S:142 partial free
    assert [p.state[HBM][i] for i in (0, 1, 2)] == [FREE, "active", "active"]
    with pytest.raises(MPError) as e:   # S:143 double free
        p.free_mem(a[:1])
    assert e.value.name == "DOUBLE_FREE"
    with pytest.raises(MPError) as e:   # S:139 InvalidAddr
        p.free_mem([(0, HBM, 100)])
    assert e.value.name == "INVALID_ADDR"


def test_insert_match_examples():
    p = mk()
    a, b, c = p.alloc_mem(3, HBM)
    p.insert(T(1, 33), [a, b])
    assert p.match(T(1, 33)) == (32, [a, b])
    q = mk()
    a2, b2 = q.alloc_mem(2, HBM)
    q.insert(T(1, 41), [a2, b2])                        # 40 tokens index 32
    assert q.match(T(1, 41))[0] == 32
    with pytest.raises(MPError) as e:                   # S:149 AddrCountMismatch
        q.insert(T(1, 41), [a2])
    assert e.value.name == "ADDR_COUNT"
    # S:153 shared 16-token prefix, two 16-token children
    r = mk()
    a, b, c = r.alloc_mem(3, HBM)
    t1 = T(1, 33)
    t2 = np.concatenate([T(1, 17), T(1017, 1033)])
    r.insert(t1, [a, b])
    r.insert(t2, [a, c])
    d = r.dump_index()
    assert [(len(k), i) for k, _m, i, *_ in d] == [(16, 0), (32, 1), (32, 2)]
    # S:161-163
    assert mk().match(T(1, 33)) == (0, [])
    assert r.match(np.concatenate([T(1, 25), T(5000, 5040)])) == (16, [a])
    assert r.match(T(1, 65)) == (32, [a, b])


def test_conflict_flag():
    p = mk()
    a, b, c = p.alloc_mem(3, HBM)
    p.insert(T(0, 32), [a, b])
    with pytest.raises(MPError) as e:
        p.insert(T(0, 32), [a, c], flags=FLAG_INS_ERR_ON_CONFLICT)
    assert e.value.name == "CONFLICT"
    assert p.state[HBM][c[2]] == "active"
    assert p.insert(T(0, 32), [a, c]) == 1               # keep-existing frees c
    assert p.state[HBM][c[2]] == FREE
    assert p.insert(T(0, 32), [a, b]) == 0               # S:208 idempotent


def test_delete_examples():
    p = mk()
    a, b = p.alloc_mem(2, HBM)
    p.insert(T(0, 32), [a, b])
    p.delete(T(0, 32))
    assert p.match(T(0, 32))[0] == 0
    assert p.free_count(HBM) == 100
    q = mk()
    a, b, c = q.alloc_mem(3, HBM)
    t1 = T(0, 32)
    t2 = np.concatenate([T(0, 16), T(500, 516)])
    q.insert(t1, [a, b])
    q.insert(t2, [a, c])
    q.delete(t1)
    assert q.match(t2) == (32, [a, c])
    before = q.dump_index()
    q.delete(T(900, 940))                                # S:173 no-op
    assert q.dump_index() == before
    # terminal rule (R6): deleting [p, q] keeps a separately stored [p]
    r = mk()
    a, b = r.alloc_mem(2, HBM)
    r.insert(T(0, 16), [a])
    r.insert(T(0, 32), [a, b])
    r.delete(T(0, 32))
    assert r.match(T(0, 32)) == (16, [a])


def test_evict_examples():
    p = mk()
    a, b, c = p.alloc_mem(3, HBM)
    t1 = T(0, 32)
    t2 = np.concatenate([T(0, 16), T(500, 516)])
    p.insert(t1, [a, b])           # t=1
    p.insert(t2, [a, c])           # t=2 (touches a)
    p.match(t2)                    # t=3 touches a, c
    assert p.evict(1, HBM) == [b]  # the older leaf's last block
    q = mk()
    x, y = q.alloc_mem(2, HBM)
    q.insert(T(0, 32), [x, y])
    q.match(T(0, 32), flags=FLAG_MATCH_PIN)
    assert q.evict(10, HBM) == []  # S:182 all pinned
    assert p.match(t1)[0] == 16    # S:183 shorter match


def test_swap_examples():
    p = mk(n_hbm=8, n_dram=4)
    a = p.alloc_mem(3, HBM)
    p.insert(T(0, 48), a)
    m0 = p.match(T(0, 48))[0]
    moved = p.swap_out(2)
    assert p.match(T(0, 48))[0] == m0
    media = [x[1] for x in p.match(T(0, 48))[1]]
    assert media == [HBM, DRAM, DRAM]
    back = p.swap_in([n for _o, n in moved][::-1])       # S:201 round trip
    assert [x[1] for x in back] == [HBM, HBM]
    with pytest.raises(MPError) as e:
        p.swap_in([a[0]])
    assert e.value.name == "PRECONDITION"
    # S:193 pinned blocks are never moved
    q = mk(n_hbm=4, n_dram=4)
    b = q.alloc_mem(2, HBM)
    q.insert(T(0, 32), b)
    q.match(T(0, 32), flags=FLAG_MATCH_PIN)
    assert q.swap_out(5) == []


def test_swap_content_preserved():
    p = OraclePool(0, 2, 2, 64, 16, n_hbm=8, n_dram=4, seed=3, materialize=True)
    a = p.alloc_mem(3, HBM)
    p.fill(a)
    p.insert(T(0, 48), a)
    want = {x[2]: p.hbm_bytes[:, x[2]].copy() for x in a}
    moved = p.swap_out(3)
    for o, n in moved:                                   # S:192 tags preserved
        assert np.array_equal(p.dram_bytes[n[2]], want[o[2]])
        assert np.array_equal(p.block_bytes(n), want[o[2]])
    back = p.swap_in([n for _o, n in moved])
    for (o, _n), h in zip(moved, back):
        assert np.array_equal(p.hbm_bytes[:, h[2]], want[o[2]])

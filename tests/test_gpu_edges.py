"""Edge cases on the GPU path, each compared with the oracle through the twin
harness: empty and sub-block inputs, the last block id of a pool, a pool so
full that the receiver must evict (and one where it cannot: DST_OOM with no
state change), DRAM exhaustion (NO_DRAM), the largest pools the content model
allows, and argument errors that must fail identically and change nothing."""
import numpy as np
import pytest

import oracle as O
from paper_2406_17565_b200 import mempool as M
from tests.twin import Twin, connect, transfer, transfer_with_insert
from workloads.configs import TINY

pytestmark = pytest.mark.gpu
B = TINY.block_tokens


def pair(n=16, n_dram=4, **kw):
    P, D = Twin(0, TINY, n, n_dram, **kw), Twin(1, TINY, n, n_dram, **kw)
    connect(P, D)
    return P, D


def prefill(X, toks):
    _, m = X.match(toks)
    new = X.alloc(-(-len(toks) // B) - len(m))
    X.fill(new)
    X.insert(toks, (m + new)[: len(toks) // B])
    return m + new


def test_empty_and_sub_block_inputs():
    P, D = pair()
    assert transfer(P, D, []) == []                                  # nothing to move
    assert P.alloc(0) == []
    P.free([])
    assert P.match(np.zeros(0, np.int32)) == (0, [])
    short = np.arange(5, 5 + B - 3, dtype=np.int32)                  # < one block
    src = prefill(P, short)
    assert len(src) == 1                                             # one partial block
    final, moved, _ = transfer_with_insert(P, D, short, src)         # moved, not indexed
    assert moved == 1 and D.o.dump_index() == []
    assert transfer_with_insert(P, D, np.zeros(0, np.int32), [])[:2] == ([], 0)
    P.check_state()
    D.check_state()


def test_last_block_and_full_pool_eviction():
    P, D = pair(n=16)
    seqs = [np.arange(100 * i, 100 * i + 4 * B, dtype=np.int32) for i in range(4)]
    for s in seqs:                          # D: 16/16 blocks indexed (evictable)
        src = prefill(P, s)
        transfer_with_insert(P, D, s, src)
    assert D.o.free_count(O.HBM) == 0
    assert sorted(a[2] for s in seqs for a in D.match(s)[1])[-1] == 15   # the last id is used
    P2 = Twin(2, TINY, 16)
    connect(P2, D)
    src = prefill(P2, np.arange(9000, 9000 + 3 * B, dtype=np.int32))
    # the receiver evicts its LRU leaves to make room (R2, R8)
    transfer_with_insert(P2, D, np.arange(9000, 9000 + 3 * B, dtype=np.int32), src)
    D.check_state()
    # now pin everything D holds: no room, DST_OOM, nothing changes
    for s in seqs:
        D.match(s, O.FLAG_MATCH_PIN)
    snap = D.o.dump_index()
    big = np.arange(7000, 7000 + 16 * B, dtype=np.int32)
    src = prefill(P, big[: 12 * B]) if P.o.free_count(O.HBM) >= 12 else None
    if src:
        with pytest.raises(O.MPError) as e:
            transfer_with_insert(P, D, big[: 12 * B], src)
        assert e.value.name == "DST_OOM"
        assert D.o.dump_index() == snap
    D.check_state()
    P.check_state()


def test_no_dram_and_errors():
    P, D = pair(n=16, n_dram=2)
    s = np.arange(0, 6 * B, dtype=np.int32)
    prefill(P, s)
    moved = P.swap_out(4)                   # DRAM holds 2: its LRU leaf is evicted when full
    assert len(moved) == 4
    assert P.match(s)[0] == 4 * B           # blocks 4, 5 went to DRAM and were evicted
    # chain A lives in DRAM and is pinned; chain B is in HBM: swapping B out
    # needs a DRAM block and no DRAM leaf may be evicted -> NO_DRAM
    P.match(s, O.FLAG_MATCH_PIN)
    prefill(P, np.arange(500, 500 + 2 * B, dtype=np.int32))
    with pytest.raises(O.MPError) as e:
        P.swap_out(1)
    assert e.value.name == "NO_DRAM"
    s = s[:4 * B]
    for bad in ([(1, O.HBM, 0)], [(0, O.HBM, 99)], [(0, 7, 0)]):
        with pytest.raises(O.MPError) as e:
            P.free(bad)
        assert e.value.name == "INVALID_ADDR"
    a = P.alloc(1)
    with pytest.raises(O.MPError) as e:
        P.free(a + a)
    assert e.value.name == "DOUBLE_FREE"
    with pytest.raises(O.MPError) as e:
        transfer(P, D, a + a)
    assert e.value.name == "PRECONDITION"
    with pytest.raises(O.MPError) as e:
        transfer_with_insert(P, D, s[:B], a + a)                     # more blocks than ceil
    assert e.value.name == "ADDR_COUNT"
    P.check_state()
    D.check_state()
    with pytest.raises(M.MempoolError) as e:                         # unknown peer
        P.g.transfer(5, M.np.array([M.make_addr(0, 0, a[0][2])], np.uint64))
    assert e.value.name == "DST_UNREACHABLE"


def test_largest_pools():
    # 16384 blocks = the content model's limit (block < 2^14): 512-word bitmap,
    # lowest-first allocation verified against the host shadow (verify mode)
    P = Twin(0, TINY, 16384)
    D = Twin(1, TINY, 16384)
    connect(P, D)
    a = P.alloc(16000)
    P.fill(a[-50:])
    P.free(a[:15000])
    b = P.alloc(15100)                       # wraps past the freed range
    assert [x[2] for x in b[:3]] == [0, 1, 2] and b[-1][2] == 16099
    out = transfer(P, D, a[-50:])
    assert [x[2] for x in out] == list(range(50))
    D.check_bytes()

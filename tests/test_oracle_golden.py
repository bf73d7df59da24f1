"""Oracle vs the hand-computed golden worked example (tests/golden/golden_tiny.yaml,
SURVEY.md §8(c)).  Pins allocator order (R2), insert/keep-existing (R4),
transfer_with_insert with and without DEDUP (R3), frontier-LRU swap (R9),
leaf-LRU evict (R8) and migration bytes (closed form dst[d] == src[s])."""
import os

import numpy as np
import pytest
import yaml

from oracle import (HBM, DRAM, FLAG_DEDUP, OraclePool, transfer_with_insert,
                    ACTIVE, INDEXED, FREE)
from workloads.configs import TINY
from workloads.traces import golden_prompts

GOLD = yaml.safe_load(open(os.path.join(os.path.dirname(__file__), "golden",
                                        "golden_tiny.yaml")))


def mk(inst, n_dram=64):
    s = TINY
    return OraclePool(inst, s.layers, s.kv_heads, s.head_dim, s.block_tokens,
                      n_hbm=64, n_dram=n_dram, seed=17565, materialize=True)


def ids(addrs):
    return [a[2] for a in addrs]


def run_golden(dedup):
    S, p1, p2, p3 = golden_prompts()
    P, D = mk(0), mk(1)
    flags = FLAG_DEDUP if dedup else 0
    res = []
    for step, p in enumerate((p1, p2, p3), start=1):
        mt, matched = P.match(p)
        ceil_b = -(-len(p) // 16)
        new = P.alloc_mem(ceil_b - len(matched), HBM)
        P.fill(new)
        full = matched + new
        P.insert(p, full[: len(p) // 16])
        pg = GOLD["p_side"][f"step{step}"]
        assert mt == pg["match_tokens"]
        assert ids(new) == pg["alloc"]
        assert P.clock == pg["clock_after"]
        assert ids(full) == pg["src"]
        final, moved, dup = transfer_with_insert(P, D, p, full, flags=flags)
        res.append((final, moved, dup, D.clock))
    return P, D, res


def states(pool):
    st = pool.state[HBM]
    return ([i for i, s in enumerate(st) if s != FREE],
            [i for i, s in enumerate(st) if s == INDEXED],
            [i for i, s in enumerate(st) if s == ACTIVE],
            sum(1 for s in st if s == FREE))


@pytest.mark.parametrize("dedup", [False, True])
def test_golden_transfer(dedup):
    P, D, res = run_golden(dedup)
    g = GOLD["d_side_dedup" if dedup else "d_side_no_dedup"]
    for step, (final, moved, dup, clk) in enumerate(res, start=1):
        e = g[f"step{step}"]
        assert ids(final) == e["returns"]
        assert moved == e["moved"]
        assert clk == e["clock_after"]
        if "dup_freed" in e:
            assert dup == e["dup_freed"]
    pf = GOLD["p_side"]["final"]
    assert states(P) == (pf["allocated"], pf["indexed"], pf["active"], pf["free"])
    df = g["final"]
    assert states(D) == (df["allocated"], df["indexed"], df["active"], df["free"])
    # bytes: the closed form dst[d] == src[s] on the materialised byte path,
    # and both equal the generator's content for the source's tags
    for d, s in g["copies"]:
        assert np.array_equal(D.hbm_bytes[:, d], P.hbm_bytes[:, s])
        assert np.array_equal(D.block_bytes((1, HBM, d)), P.hbm_bytes[:, s])
    P.check_invariants()
    D.check_invariants()
    if not dedup:
        S, p1, p2, p3 = golden_prompts()
        for name, p in (("p1", p1), ("p2", p2), ("p3", p3), ("S", S)):
            mt, addrs = D.match(p)
            assert [mt, ids(addrs)] == g["matches"][name]


def test_golden_swap_and_evict():
    S, p1, p2, p3 = golden_prompts()
    P, _, _ = run_golden(False)
    before = P.hbm_bytes[:, 2].copy()
    E = P._clone_meta()  # independent copy for the evict branch
    g = GOLD["p_swap"]
    moved = P.swap_out(2)
    assert [[o[2], n[2]] for o, n in moved] == g["swap_out_2"]
    assert all(o[1] == HBM and n[1] == DRAM for o, n in moved)
    mt, addrs = P.match(p1)
    assert [mt, [[a[1], a[2]] for a in addrs]] == g["match_p1"]
    mt, addrs = P.match(p2)
    assert [mt, [[a[1], a[2]] for a in addrs]] == g["match_p2"]
    new = P.swap_in([(0, DRAM, 0)])
    assert ids(new) == g["swap_in_R0"]
    assert np.array_equal(P.hbm_bytes[:, 2], before)
    mt, addrs = P.match(p1)
    assert mt == 48 and ids(addrs) == [0, 1, 2] and all(a[1] == HBM for a in addrs)
    P.check_invariants()
    # evict branch on the pre-swap state
    freed = E.evict(1, HBM)
    assert ids(freed) == GOLD["p_evict"]["evict_1_hbm"]
    assert E.match(p1)[0] == GOLD["p_evict"]["match_p1_after"]
    E.check_invariants()

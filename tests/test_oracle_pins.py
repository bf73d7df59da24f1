"""Independent pins of the oracle's readings where the paper names a policy
but not its details: R7-R8 (LRU eviction, "evict"),
R9 (swap-out victims), R2 (evict before OOM) and R3
(transfer_with_insert's reuse of the receiver's cached prefix, P:364,
P:495).  None of these re-types the oracle's rule; each derives the expected
outcome another way:

  * R7/R8 -- the last use of every cached prefix is recomputed from the OP
    HISTORY (the op index of the last insert covering it or match reaching
    it), and the evicted block must be the least-recently-used unpinned leaf
    of the CURRENT index (leaf = no cached prefix extends it);
  * R9 -- same history, victim = least-recently-used unpinned HBM block with
    no HBM child (the HBM frontier), one swap at a time;
  * R2 -- the most blocks eviction can free is the largest set of unpinned
    cached prefixes closed under "extends" (a prefix can go only after every
    longer cached prefix), found by enumerating subsets of tiny indexes;
    alloc_mem must succeed exactly up to free + that number;
  * R3 -- after transfer_with_insert with DEDUP the receiver's bytes of every
    block equal the sender's, every block the receiver already cached is
    reused rather than moved (moved + reused == sent), and no receiver block
    is leaked.
"""
import itertools

import numpy as np
import pytest

from oracle import (DRAM, FLAG_DEDUP, FLAG_MATCH_PIN, FREE, HBM, MPError, OraclePool,
                    transfer_with_insert)


def prefixes(seq, B, k=None):
    k = len(seq) // B if k is None else k
    return [tuple(int(x) for x in seq[: i * B]) for i in range(1, k + 1)]


def gen(rng, stored, vocab, maxlen):
    if stored and rng.random() < 0.7:
        base = stored[rng.integers(len(stored))]
        cut = int(rng.integers(0, len(base) + 1))
        tail = [int(t) for t in rng.integers(0, vocab, int(rng.integers(0, maxlen - cut + 1)))]
        return list(base[:cut]) + tail
    return [int(t) for t in rng.integers(0, vocab, int(rng.integers(1, maxlen + 1)))]


class History:
    """Op index of the last use of every prefix, from the op log alone."""

    def __init__(self):
        self.t = 0
        self.last = {}

    def use(self, prefs):
        self.t += 1
        for p in prefs:
            self.last[p] = self.t


def children(index, B):
    kids = {}
    for key in index:
        if len(key) > B:
            kids.setdefault(key[:-B], []).append(key)
    return kids


def lru_pick(pool, hist, medium, frontier):
    """The expected victim: among unpinned cached prefixes of `medium` with no
    cached child (leaf) / no HBM child (frontier), least (last use, block)."""
    kids = children(pool.index, pool.B)
    best = None
    for key, e in pool.index.items():
        if e.addr[1] != medium or e.ref != 0:
            continue
        ks = kids.get(key, [])
        if frontier:
            if any(pool.index[c].addr[1] == HBM for c in ks):
                continue
        elif ks:
            continue
        cand = (hist.last[key], e.addr[2], key)
        best = cand if best is None or cand < best else best
    return best


def random_history_run(seed, B, n_ops, swap):
    rng = np.random.default_rng(seed)
    pool = OraclePool(0, 1, 1, 8, B, n_hbm=48, n_dram=48 if swap else 0)
    hist = History()
    stored = []
    vocab = int(rng.integers(2, 4))
    checked = 0
    for _ in range(n_ops):
        op = rng.random()
        if op < 0.4:
            s = gen(rng, stored, vocab, 6 * B)
            k = len(s) // B
            _, m = pool.match(np.array(s, np.int32))
            hist.use(prefixes(s, B, len(m)))
            try:
                new = pool.alloc_mem(k - len(m), HBM)
            except MPError:
                continue
            # an allocation may have evicted: the victims' history is moot
            pool.insert(np.array(s, np.int32), list(m) + new)
            hist.use(prefixes(s, B))
            if k:
                stored.append(s[: k * B])
        elif op < 0.6:
            q = gen(rng, stored, vocab, 6 * B)
            pin = rng.random() < 0.15
            mt, addrs = pool.match(np.array(q, np.int32), FLAG_MATCH_PIN if pin else 0)
            hist.use(prefixes(q, B, mt // B))
            if pin and addrs and rng.random() < 0.5:
                pool.unpin(addrs)
        elif op < 0.7 and stored:
            pool.delete(np.array(stored.pop(int(rng.integers(len(stored)))), np.int32))
        elif not swap or op < 0.85:
            want = lru_pick(pool, hist, HBM, frontier=False)
            got = pool.evict(1, HBM)
            if want is None:
                assert got == []
            else:
                assert got == [(0, HBM, want[1])], (got, want)
                checked += 1
        else:
            want = lru_pick(pool, hist, HBM, frontier=True)
            if pool.free_count(DRAM) == 0:
                continue
            moved = pool.swap_out(1)
            if want is None:
                assert moved == []
            else:
                (old, new), = moved
                assert old == (0, HBM, want[1]), (old, want)
                assert pool.index[want[2]].addr == new   # same prefix, now in DRAM
                checked += 1
    return checked


@pytest.mark.parametrize("B", [2, 4])
def test_lru_evict_matches_history(B):
    """R7 + R8: evict() always takes the least-recently-used unpinned leaf,
    with recency recomputed from the op history."""
    checked = sum(random_history_run(1000 + s, B, 120, swap=False) for s in range(25))
    assert checked > 100


@pytest.mark.parametrize("B", [2, 4])
def test_swap_out_victim_matches_history(B):
    """R7 + R9: swap_out() takes the least-recently-used unpinned block of the
    HBM frontier (no child in HBM), recency from the op history."""
    checked = sum(random_history_run(2000 + s, B, 120, swap=True) for s in range(25))
    assert checked > 50


def max_evictable(pool, medium):
    """Largest set S of unpinned `medium` prefixes such that every cached
    child of a member is a member (brute force over subsets)."""
    kids = children(pool.index, pool.B)
    cand = [k for k, e in pool.index.items() if e.addr[1] == medium and e.ref == 0]
    for r in range(len(cand), -1, -1):
        for S in itertools.combinations(cand, r):
            s = set(S)
            if all(c in s for k in s for c in kids.get(k, [])):
                return r
    return 0


def test_evict_before_oom_bruteforce():
    """R2: alloc_mem(n) succeeds iff n <= free + the largest
    eviction-closed set of unpinned blocks; evict(inf) frees exactly that."""
    rng = np.random.default_rng(7)
    B = 2
    cases = 0
    for _ in range(150):
        pool = OraclePool(0, 1, 1, 8, B, n_hbm=10)
        stored = []
        for _ in range(int(rng.integers(1, 6))):
            s = gen(rng, stored, 2, 8)
            k = len(s) // B
            _, m = pool.match(np.array(s, np.int32))
            if pool.free_count(HBM) < k - len(m):
                continue
            new = pool.alloc_mem(k - len(m), HBM)
            pool.insert(np.array(s, np.int32), list(m) + new)
            stored.append(s)
        if stored and rng.random() < 0.5:
            pool.match(np.array(stored[rng.integers(len(stored))], np.int32), FLAG_MATCH_PIN)
        if len(pool.index) > 10:
            continue
        best = max_evictable(pool, HBM)
        free = pool.free_count(HBM)
        trial = pool._clone_meta()
        assert len(trial.evict(10 ** 6, HBM)) == best
        ok = pool._clone_meta()
        assert len(ok.alloc_mem(free + best, HBM)) == free + best
        too_many = pool._clone_meta()
        with pytest.raises(MPError, match="OOM"):
            too_many.alloc_mem(free + best + 1, HBM)
        cases += 1
    assert cases > 100


def test_dedup_reuses_cached_prefix_and_moves_bytes():
    """R3 against the paper's statement of the workflow:
    the receiver ends up holding the sender's bytes for every block, indexes
    the prompt, moves only what it did not cache, and leaks nothing."""
    rng = np.random.default_rng(11)
    B = 4
    for trial in range(40):
        P = OraclePool(0, 1, 2, 8, B, n_hbm=64, materialize=True, seed=3)
        D = OraclePool(1, 1, 2, 8, B, n_hbm=64, materialize=True, seed=3)
        stored = []
        for _ in range(8):
            t = gen(rng, stored, 2, 10 * B)
            stored.append(t)
            toks = np.array(t, np.int32)
            ceil_b = -(-len(t) // B)
            _, m = P.match(toks)
            new = P.alloc_mem(ceil_b - len(m), HBM)
            P.fill(new)
            src = list(m) + new
            P.insert(toks, src[: len(t) // B])
            before = {e.addr for e in D.index.values()}
            d_used = sum(1 for s in D.state[HBM] if s != FREE)
            final, moved, _dup = transfer_with_insert(P, D, toks, src, flags=FLAG_DEDUP)
            # bytes: every block of the prompt at D equals P's
            for s_a, d_a in zip(src, final):
                assert np.array_equal(D.block_bytes(d_a), P.block_bytes(s_a))
            # D indexes the prompt's full blocks at exactly those addresses
            mt, dm = D.match(toks)
            assert mt == (len(t) // B) * B and list(dm) == list(final[: len(t) // B])
            # reuse: blocks D had cached are not moved again
            reused = sum(1 for a in final if a in before)
            assert moved + reused == len(src)
            # conservation: D grew by exactly the moved blocks
            assert sum(1 for s in D.state[HBM] if s != FREE) == d_used + moved
            # the trailing partial block is D's (active), free it like an engine
            if len(t) % B:
                D.free_mem([final[-1]])
                P.free_mem([src[-1]])
            P.check_invariants()
            D.check_invariants()

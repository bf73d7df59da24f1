"""Oracle pins of the block aggregation (§5.2; SPEC.md
S:277-278 examples, acceptance criterion 2 at S:633).

* Call counts: the paper's instance -- a 2048-token prompt (the NCCL study's
  prompt), B = 16, L = 40 (Llama2-13B) -- needs 10,240
  network calls with the discrete layout ("each call only transmits a single
  block") and 128 aggregated ("reduces the number of network API calls
  by 2*L times"): exactly 80x.  Property-tested over 200 random
  (n_tokens, B, L): discrete = 2L x aggregated, by-layer-agg = L.
* Layout: every mode's calls tile the request's bytes exactly once, and an
  aggregated block i starts at byte i*Pb; the oracle's pack (A4) puts block
  i's 2L chunks there, layer-major, K before V (R11) -- cross-checked against
  np.take over the per-layer slabs (a library routine, not the oracle's own
  block_bytes path) and against the oracle's DRAM pool, which uses the same
  aggregated layout after a swap_out.
"""
import numpy as np
import pytest

import oracle as O

C13B = 16 * 40 * 128 * 2          # chunk c of the Llama-2-13B shape (B H D elem)


def test_paper_instance_call_counts():
    disc = O.network_calls(2048, 16, 40, C13B, "by_request")
    agg = O.network_calls(2048, 16, 40, C13B, "by_request_agg")
    assert len(disc) == 10_240                    # S:277 = 128 blocks x 2L
    assert len(agg) == 128
    assert len(disc) == 2 * 40 * len(agg)         # P:550 "by 2*L times"
    # "regardless of whether the by-layer or by-request approach is used"
    assert len(O.network_calls(2048, 16, 40, C13B, "by_layer")) == 10_240
    # by-layer needs "at least L times": one aggregated call per layer
    assert len(O.network_calls(2048, 16, 40, C13B, "by_layer_agg")) == 40
    # aggregated block i at i*Pb, Pb = 2*L*c = 12.5 MiB
    Pb = 2 * 40 * C13B
    assert Pb == 13_107_200
    assert [o for o, _ in agg] == [i * Pb for i in range(128)]
    assert all(s == Pb for _, s in agg)


def _tiles(calls, total):
    pos = 0
    for off, size in sorted(calls):
        if off != pos:
            return False
        pos += size
    return pos == total


def test_call_count_property():
    rng = np.random.default_rng(633)
    for _ in range(200):
        n_tok = int(rng.integers(0, 5000))
        B = int(rng.choice([1, 4, 8, 16, 32]))
        L = int(rng.integers(1, 81))
        c = 16 * int(rng.integers(1, 64))
        nb = -(-n_tok // B)                       # R1: the partial block moves too
        d = O.network_calls(n_tok, B, L, c, "by_request")
        a = O.network_calls(n_tok, B, L, c, "by_request_agg")
        la = O.network_calls(n_tok, B, L, c, "by_layer_agg")
        assert len(d) == 2 * L * nb and len(a) == nb
        assert len(d) == 2 * L * len(a)
        assert len(la) == (L if nb else 0)
        for calls in (d, a, la):
            assert _tiles(calls, nb * 2 * L * c)
        assert [o for o, _ in a] == [i * 2 * L * c for i in range(nb)]


def test_unknown_mode_is_config():
    with pytest.raises(O.MPError):
        O.network_calls(16, 16, 2, 4096, "by_token")


def _filled_pool(L=3, H=2, D=8, B=4, n=12, seed=5):
    P = O.OraclePool(0, L, H, D, B, n, n_dram=n, seed=seed, materialize=True)
    a = P.alloc_mem(n, O.HBM)
    P.fill(a[: n // 2])
    P.fill(a[n // 2:])                            # two epochs: distinct content
    return P, a


def test_pack_layout_matches_take_over_slabs():
    P, a = _filled_pool()
    rng = np.random.default_rng(1)
    pick = [a[i] for i in rng.permutation(len(a))[:7]]     # scattered ids
    ids = [x[2] for x in pick]
    st = O.pack(P, pick)
    assert st.shape == (7, P.L, 2, P.W)
    for l in range(P.L):
        for kv in (0, 1):
            np.testing.assert_array_equal(st[:, l, kv], np.take(P.hbm_bytes[2 * l + kv], ids,
                                                                axis=0))
    # byte view: block i starts at i*Pb and is [L][2][c] contiguous
    flat = st.reshape(-1).view(np.uint8)
    Pb = 2 * P.L * P.chunk_bytes
    for i, x in enumerate(ids):
        blk = flat[i * Pb:(i + 1) * Pb].view(np.uint64).reshape(2 * P.L, P.W)
        np.testing.assert_array_equal(blk, P.hbm_bytes[:, x])
    # by-layer staging of layers [1, 3): [n][2][2][W], the calls of by_layer_agg
    sl = O.pack(P, pick, 1, 3)
    np.testing.assert_array_equal(sl, st[:, 1:3])
    with pytest.raises(O.MPError):
        O.pack(P, pick, 2, 2)


def test_pack_equals_dram_aggregated_layout():
    """The DRAM pool keeps blocks aggregated: after swap_out the
    DRAM block's words equal the pack of the HBM block it came from."""
    P, a = _filled_pool()
    toks = np.arange(len(a) * P.B, dtype=np.int32)
    P.insert(toks, a)
    before = {x[2]: O.pack(P, [x])[0].copy() for x in a}
    moved = P.swap_out(3)
    assert len(moved) == 3
    for h, d in moved:
        np.testing.assert_array_equal(P.dram_bytes[d[2]].reshape(P.L, 2, P.W), before[h[2]])
        np.testing.assert_array_equal(O.pack(P, [d])[0], before[h[2]])

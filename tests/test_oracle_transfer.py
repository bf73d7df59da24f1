"""Oracle transfer / transfer_with_insert semantics (§4.3 P:360-369,
R3, R13) and the byte-path closed forms (SURVEY.md §8(c) pins):
pack == np.take(slab, ids) per (layer, kv); unpack o pack == identity on the
chosen blocks; by-layer moves only its layer range."""
import numpy as np
import pytest

from oracle import (HBM, DRAM, FLAG_DEDUP, FLAG_DST_GIVEN, FLAG_INS_ERR_ON_CONFLICT,
                    MPError, OraclePool, transfer, transfer_with_insert)


def mk(inst, n=32, L=3):
    return OraclePool(inst, L, 2, 16, 8, n_hbm=n, n_dram=8, seed=5, materialize=True)


def T(*r):
    return np.arange(*r, dtype=np.int32)


def test_transfer_bytes_closed_form():
    P, D = mk(0), mk(1)
    src = P.alloc_mem(10, HBM)
    P.fill(src)
    rng = np.random.default_rng(0)
    order = [src[i] for i in rng.permutation(10)]
    D.alloc_mem(3, HBM)                      # so dst ids differ from src ids
    out = transfer(P, D, order, priv=b"req-7")
    sid = [a[2] for a in order]
    did = [a[2] for a in out]
    for j in range(P.nch):
        # pack of the source = np.take over the slab (library cross-check)
        packed = np.take(P.hbm_bytes[j], sid, axis=0)
        np.testing.assert_array_equal(np.take(D.hbm_bytes[j], did, axis=0), packed)
    assert D.inbox[-1][:3] == ("transfer", 0, b"req-7")
    assert all(D.state[HBM][i] == "active" for i in did)


def test_by_layer_dst_given():
    P, D = mk(0), mk(1)
    src = P.alloc_mem(4, HBM)
    P.fill(src)
    dst = D.alloc_mem(4, HBM)
    D.fill(dst)
    old = D.hbm_bytes.copy()
    transfer(P, D, src, dst, flags=FLAG_DST_GIVEN, layer_begin=1, layer_end=2)
    for s, d in zip(src, dst):
        for j in range(D.nch):
            want = P.hbm_bytes[j, s[2]] if 2 <= j < 4 else old[j, d[2]]
            np.testing.assert_array_equal(D.hbm_bytes[j, d[2]], want)
    with pytest.raises(MPError) as e:        # dst must be caller-owned (ACTIVE)
        transfer(P, D, src[:1], [(1, HBM, 20)], flags=FLAG_DST_GIVEN)
    assert e.value.name == "PRECONDITION"


def test_transfer_errors_no_state_change():
    P, D = mk(0), mk(1, n=4)
    src = P.alloc_mem(5, HBM)
    snap = D.dump_index(), list(D.state[HBM])
    with pytest.raises(MPError) as e:
        transfer(P, D, src)
    assert e.value.name == "DST_OOM"
    assert (D.dump_index(), list(D.state[HBM])) == snap
    with pytest.raises(MPError) as e:
        transfer(P, D, [(0, DRAM, 0)])       # R13: a FREE DRAM block is no source
    assert e.value.name in ("PRECONDITION",)
    with pytest.raises(MPError) as e:
        transfer(P, None, src)
    assert e.value.name == "DST_UNREACHABLE"


def test_suffix_and_prefix_missing():
    """D->P return: the receiver already holds the prompt; the sender
    ships only the decode blocks (suffix, R3)."""
    P, D = mk(0), mk(1)
    prompt = T(0, 24)                        # 3 blocks of B=8
    gen = T(100, 116)                        # 2 more blocks
    full = np.concatenate([prompt, gen])
    pa = P.alloc_mem(3, HBM)
    P.fill(pa)
    P.insert(prompt, pa)
    # D has the prompt (as if P->D transferred it) and decoded 2 more blocks
    final, moved, _ = transfer_with_insert(P, D, prompt, pa)
    assert moved == 3
    da = D.alloc_mem(2, HBM)
    D.fill(da)
    D.insert(full, final + da)
    # D -> P with the suffix only
    _, dsrc = D.match(full)
    f2, moved2, dup2 = transfer_with_insert(D, P, full, dsrc[3:])
    assert moved2 == 2 and dup2 == 0
    assert f2[:3] == pa
    assert P.match(full)[0] == 40
    for s, d in zip(dsrc[3:], f2[3:]):
        np.testing.assert_array_equal(P.hbm_bytes[:, d[2]], D.hbm_bytes[:, s[2]])
    # a receiver missing the prefix refuses and changes nothing
    X = mk(2)
    snap = X.clock, X.dump_index()
    with pytest.raises(MPError) as e:
        transfer_with_insert(D, X, full, dsrc[3:])
    assert e.value.name == "PREFIX_MISSING"
    assert (X.clock, X.dump_index()) == snap


def test_dram_source_memory_asymmetry():
    """historical KV swapped out to DRAM is transferred straight
    from DRAM.  After swap_out, the matched prefix mixes HBM and DRAM addrs;
    the receiver's bytes must equal the ORIGINAL (pre-swap) content."""
    P, D = mk(0), mk(1)
    p = T(0, 48)
    a = P.alloc_mem(6, HBM)
    P.fill(a)
    P.insert(p, a)
    want = {x[2]: P.hbm_bytes[:, x[2]].copy() for x in a}
    moved = P.swap_out(2)                    # the two deepest blocks go to DRAM
    assert [o[2] for o, _ in moved] == [5, 4]
    _, matched = P.match(p)
    assert [x[1] for x in matched] == [HBM] * 4 + [DRAM] * 2
    final, nm, _ = transfer_with_insert(P, D, p, matched)
    assert nm == 6
    for i, d in enumerate(final):
        np.testing.assert_array_equal(D.hbm_bytes[:, d[2]], want[a[i][2]])
    # by-layer from a DRAM block into a caller-given block
    x = D.alloc_mem(1, HBM)
    transfer(P, D, [matched[5]], x, flags=FLAG_DST_GIVEN, layer_begin=1, layer_end=3)
    np.testing.assert_array_equal(D.hbm_bytes[2:6, x[0][2]], want[a[5][2]][2:6])


def test_dedup_conflict_flag():
    P, D = mk(0), mk(1)
    p = T(0, 32)
    a = P.alloc_mem(4, HBM)
    P.insert(p, a)
    transfer_with_insert(P, D, p, a)
    with pytest.raises(MPError) as e:
        transfer_with_insert(P, D, p, a, flags=FLAG_INS_ERR_ON_CONFLICT)
    assert e.value.name == "CONFLICT"
    final, moved, dup = transfer_with_insert(P, D, p, a, flags=FLAG_DEDUP)
    assert moved == 0 and dup == 0


def test_dst_oom_rolls_back_dedup_match():
    P, D = mk(0), mk(1, n=4)
    p = T(0, 24)
    a = P.alloc_mem(3, HBM)
    P.insert(p, a)
    transfer_with_insert(P, D, p, a)
    x = D.alloc_mem(1, HBM)                    # D: 3 indexed + 1 active, 0 free
    q = np.concatenate([p, T(500, 516)])       # shares 3 blocks, needs 2 more
    b = P.alloc_mem(2, HBM)
    P.insert(q, a + b)
    snap = D.clock, D.dump_index(), list(D.state[HBM])
    with pytest.raises(MPError) as e:
        transfer_with_insert(P, D, q, a + b, flags=FLAG_DEDUP)
    assert e.value.name == "DST_OOM"
    assert (D.clock, D.dump_index(), list(D.state[HBM])) == snap
    D.free_mem(x)
    with pytest.raises(MPError):
        transfer_with_insert(P, D, q, a + b, flags=FLAG_DEDUP)   # needs 2, 1 free, prefix pinned
    assert (D.clock, D.dump_index()) == snap[:2]

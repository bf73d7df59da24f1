"""Asymmetric parallelism (§4.3): moving KV
between instances of different tensor-parallel degree.

CPU: the split plan is pinned by its defining property (every head of the
model moves exactly once, from the rank holding it to the rank that will
hold it) and the C-ABI plan must equal the oracle's; the
oracle's head-range copy is pinned by reassembly (concatenating the
destination shards' heads gives back the concatenation of the source
shards').  GPU: the CUDA path (mp_transfer_heads per plan piece) must equal
the oracle byte for byte."""
import numpy as np
import pytest

import oracle as O
from workloads.configs import KVShape


@pytest.mark.parametrize("H,p,q", [(8, 1, 2), (8, 2, 1), (8, 2, 4), (8, 4, 2), (12, 3, 4),
                                   (40, 2, 8), (32, 8, 8), (6, 6, 1)])
def test_plan_covers_each_head_once(H, p, q):
    plan = O.tp_plan(H, p, q)
    seen = []
    for r, s, h0, g0, k in plan:
        for i in range(k):
            h = r * (H // p) + h0 + i            # global head index at the source
            assert h == s * (H // q) + g0 + i    # ... and at the destination
            seen.append(h)
    assert sorted(seen) == list(range(H))


def test_capi_plan_equals_oracle():
    from paper_2406_17565_b200 import mempool as M
    for H in (1, 2, 6, 8, 12, 40, 64):
        for p in range(1, 9):
            for q in range(1, 9):
                if H % p or H % q:
                    with pytest.raises(M.MempoolError):
                        M.tp_plan(H, p, q)
                    continue
                assert sorted(M.tp_plan(H, p, q)) == O.tp_plan(H, p, q)


def _shards(H, t, shape, n, base_inst, seed):
    pools = []
    for r in range(t):
        P = O.OraclePool(base_inst + r, shape.layers, H // t, shape.head_dim,
                         shape.block_tokens, n, seed=seed, materialize=True)
        pools.append(P)
    return pools


def _full_view(pools, H, t, block_ids, W_head):
    """[n][2L][H*W_head]: the model-wide chunk of each block, heads in order."""
    parts = [P.hbm_bytes[:, block_ids[r]].reshape(P.nch, len(block_ids[r]), H // t, W_head)
             for r, P in enumerate(pools)]
    return np.concatenate(parts, axis=2).transpose(1, 0, 2, 3)


@pytest.mark.parametrize("p,q", [(2, 1), (1, 2), (2, 4), (4, 2)])
def test_oracle_reassembly(p, q):
    H, shape = 8, KVShape("tp", 2, 8, 64, 16)
    n = 5
    src = _shards(H, p, shape, 12, 0, 7)
    dst = _shards(H, q, shape, 12, 100, 7)
    s_ids, d_ids = [], []
    for P in src:
        a = P.alloc_mem(n, O.HBM)
        P.fill(a)
        s_ids.append(a)
    for D in dst:
        d_ids.append(D.alloc_mem(n, O.HBM))
    for r, s, h0, g0, k in O.tp_plan(H, p, q):
        O.transfer_heads(src[r], dst[s], s_ids[r], d_ids[s], h0, g0, k,
                         kv_heads=(H // p, H // q))
    W_head = src[0].W // (H // p)
    a = _full_view(src, H, p, [[x[2] for x in ids] for ids in s_ids], W_head)
    b = _full_view(dst, H, q, [[x[2] for x in ids] for ids in d_ids], W_head)
    np.testing.assert_array_equal(a, b)


@pytest.mark.gpu
@pytest.mark.parametrize("p,q", [(2, 1), (1, 2), (2, 4), (4, 2), (1, 4)])
def test_gpu_repartition_matches_oracle(p, q):
    from paper_2406_17565_b200 import mempool as M
    H, shape, n, seed = 8, KVShape("tp", 3, 8, 64, 16), 7, 11
    osrc = _shards(H, p, shape, 16, 0, seed)
    odst = _shards(H, q, shape, 16, 100, seed)
    gsrc = [M.Pool(r, 0, shape.layers, H // p, shape.head_dim, shape.block_tokens, 16,
                   verify=True) for r in range(p)]
    gdst = [M.Pool(100 + s, 0, shape.layers, H // q, shape.head_dim, shape.block_tokens, 16,
                   verify=True) for s in range(q)]
    for a in gsrc:
        for b in gdst:
            M.connect(a, b)
    s_ids, d_ids, gs_ids, gd_ids = [], [], [], []
    for P, G in zip(osrc, gsrc):
        G.alloc_mem(2)                       # shards need not share block ids
        P.alloc_mem(2, O.HBM)
        a, ga = P.alloc_mem(n, O.HBM), G.alloc_mem(n)
        P.fill(a)
        G.debug_fill(ga, seed)
        s_ids.append(a)
        gs_ids.append(ga)
    for D, G in zip(odst, gdst):
        d, gd = D.alloc_mem(n, O.HBM), G.alloc_mem(n)
        d_ids.append(d)
        gd_ids.append(gd)
    for r, s, h0, g0, k in O.tp_plan(H, p, q):
        O.transfer_heads(osrc[r], odst[s], s_ids[r], d_ids[s], h0, g0, k, 1, 3,
                         kv_heads=(H // p, H // q))
    M.repartition(gsrc, gdst, gs_ids, gd_ids, H, layer_begin=1, layer_end=3,
                  flags=M.XFER_ASYNC)
    for D, G, ids in zip(odst, gdst, d_ids):
        G.sync()
        for x in ids:
            got = G.debug_read_block(M.make_addr(G.inst, 0, x[2]))
            want = D.hbm_bytes[:, x[2]]
            np.testing.assert_array_equal(got[2:6], want[2:6])   # layers 1..2 moved
    for G in gsrc + gdst:
        G.close()

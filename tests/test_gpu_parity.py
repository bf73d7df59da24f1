"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle, element by
element -- block ids, returned addrs, moved counts, error names, clocks, index
dumps, device bitmap, and every byte of every written block (integer compare).

Tiny config (BASELINE.json configs[0]) golden run + randomized op sequences
that cross several kernel tiles and ragged tails, on 1 GPU (two pools on
cuda:0: the loopback transport)."""
import numpy as np
import pytest

import oracle as O
from paper_2406_17565_b200 import mempool as M
from tests.twin import Twin, connect, transfer, transfer_with_insert
from workloads.configs import TINY, KVShape
from workloads.traces import golden_prompts

pytestmark = pytest.mark.gpu

PATHS = [M.PATH_FUSED, M.PATH_STAGED, M.PATH_CE]
# stream-ordered (MP_XFER_ASYNC) variants: results must not depend on the sync
PATHS_ASYNC = [M.PATH_FUSED | M.XFER_ASYNC, M.PATH_CE | M.XFER_ASYNC,
               M.PATH_STAGED | M.XFER_ASYNC]


def golden_pair(dedup, path, n_dram=64):
    P = Twin(0, TINY, 64, n_dram)
    D = Twin(1, TINY, 64, n_dram)
    connect(P, D)
    S, p1, p2, p3 = golden_prompts()
    res = []
    for p in (p1, p2, p3):
        mt, matched = P.match(p)
        new = P.alloc(-(-len(p) // 16) - len(matched))
        P.fill(new)
        P.insert(p, (matched + new)[: len(p) // 16])
        res.append(transfer_with_insert(P, D, p, matched + new,
                                        oflags=O.FLAG_DEDUP if dedup else 0, path=path))
    return P, D, res


@pytest.mark.parametrize("path", PATHS + PATHS_ASYNC)
@pytest.mark.parametrize("dedup", [False, True])
def test_golden_tiny(dedup, path):
    P, D, res = golden_pair(dedup, path)
    P.check_state()
    D.check_state()
    moved = [r[1] for r in res]
    assert moved == ([4, 3, 1] if dedup else [4, 5, 3])
    # private delivery
    msgs = []
    while True:
        m = D.g.recv_poll()
        if m is None:
            break
        msgs.append(m)
    assert len(msgs) == 3 and all(k == 1 and s == 0 for k, s, _p, _a in msgs)


def test_golden_swap_evict():
    P, D, _ = golden_pair(False, M.PATH_FUSED)
    S, p1, p2, p3 = golden_prompts()
    moved = P.swap_out(2)
    assert [(o[2], n[2]) for o, n in moved] == [(2, 0), (5, 1)]
    P.match(p1)
    P.match(p2)
    P.check_state()
    assert P.swap_in([(0, O.DRAM, 0)]) == [(0, O.HBM, 2)]
    P.check_state()
    assert P.evict(1, O.HBM) != []
    P.check_state()


def test_private_and_transfer_layers():
    P = Twin(0, TINY, 64)
    D = Twin(1, TINY, 64)
    connect(P, D)
    src = P.alloc(5)
    P.fill(src)
    dst = D.alloc(5)
    D.fill(dst)
    for path in PATHS:
        transfer(P, D, src, dst, oflags=O.FLAG_DST_GIVEN, l0=1, l1=2, priv=b"layer-1", path=path)
        D.check_state()
    out = transfer(P, D, src, priv=b"\x00req\xff")
    D.check_state()
    kinds = []
    while True:
        m = D.g.recv_poll()
        if m is None:
            break
        kinds.append(m)
    assert kinds[-1][2] == b"\x00req\xff"
    assert [M.addr_index(a) for a in kinds[-1][3]] == [x[2] for x in out]


@pytest.mark.parametrize("dram_mode,staging", [("ce", 0), ("ce", 2), ("sm", 0)])
@pytest.mark.parametrize("path", [M.PATH_FUSED, M.PATH_FUSED | M.XFER_ASYNC, M.PATH_STAGED,
                                  M.PATH_CE])
def test_dram_source_memory_asymmetry(path, dram_mode, staging, monkeypatch):
    """historical KV swapped out to DRAM goes straight from the
    source's pinned DRAM to the receiver's HBM (mixed-media source lists,
    whole blocks and a by-layer range) -- through the copy engine and the
    source's staging (default; `staging` blocks of room: 2 forces one-block
    slots alternating between two halves) or one zero-copy kernel
    (MP_DRAM_SOURCE=sm)."""
    monkeypatch.setenv("MP_DRAM_SOURCE", dram_mode)
    kw = dict(staging_bytes=staging * TINY.block_bytes, staging_slots=staging) if staging else {}
    P = Twin(0, TINY, 32, 16, **kw)
    D = Twin(1, TINY, 32, 16, **kw)
    connect(P, D)
    S, p1, p2, p3 = golden_prompts()
    for p in (p1, p2):
        _, matched = P.match(p)
        new = P.alloc(-(-len(p) // 16) - len(matched))
        P.fill(new)
        P.insert(p, (matched + new)[: len(p) // 16])
    P.swap_out(3)
    _, src = P.match(p2)
    assert {a[1] for a in src} == {O.HBM, O.DRAM}
    transfer_with_insert(P, D, p2[: len(src) * 16], src, path=path)
    x = D.alloc(2)
    D.fill(x)
    transfer(P, D, src[-2:], x, oflags=O.FLAG_DST_GIVEN, l0=1, l1=2, path=path)
    P.check_state()
    D.check_state()


def random_ops(seed, shape, n_ops, path, n_hbm=48, n_dram=24, copy_kernel=0, coalesce_mib=0,
               swap_flags=0, staging_bytes=0, n_pools=2, **pool_kw):
    rng = np.random.default_rng(seed)
    kw = dict(copy_kernel=copy_kernel, coalesce_mib=coalesce_mib, staging_bytes=staging_bytes,
              **pool_kw)
    twins = [Twin(i, shape, n_hbm, n_dram, **kw) for i in range(n_pools)]
    for t in twins:
        t.swap_flags = swap_flags
    for i in range(n_pools):
        for j in range(i + 1, n_pools):
            connect(twins[i], twins[j])
    P, D = twins[0], twins[1]
    B = shape.block_tokens
    pools = dict(enumerate(twins))
    seqs = []
    vocab = 4

    def gen():
        if seqs and rng.random() < 0.7:
            base = seqs[rng.integers(len(seqs))]
            cut = int(rng.integers(0, len(base) + 1))
            return np.concatenate([base[:cut], rng.integers(0, vocab, int(rng.integers(0, 4 * B)),
                                                          dtype=np.int32)]).astype(np.int32)
        return rng.integers(0, vocab, int(rng.integers(1, 6 * B)), dtype=np.int32)

    for step in range(n_ops):
        x = int(rng.integers(n_pools))
        X = pools[x]
        Y = pools[(x + 1 + int(rng.integers(n_pools - 1))) % n_pools]
        op = rng.random()
        try:
            if op < 0.22:
                # engine-style prefill: match, alloc the rest, fill, insert
                t = gen()
                mt, matched = X.match(t)
                new = X.alloc(-(-len(t) // B) - len(matched),
                              stream_ordered=bool(path & M.XFER_ASYNC) and rng.random() < 0.5)
                X.fill(new)
                X.insert(t, (matched + new)[: len(t) // B])
                seqs.append(t)
            elif op < 0.40 and seqs:
                t = seqs[rng.integers(len(seqs))]
                mt, addrs = X.match(t)
                if addrs:
                    k = int(rng.integers(0, len(addrs) + 1))
                    fl = int(rng.choice([0, O.FLAG_DEDUP, O.FLAG_INS_ERR_ON_CONFLICT]))
                    transfer_with_insert(X, Y, t[: len(addrs) * B], addrs[k:] if k else addrs,
                                         oflags=fl, priv=bytes([step % 256]), path=path)
            elif op < 0.50:
                a = X.alloc(int(rng.integers(0, 4)))
                if a and rng.random() < 0.5:
                    X.fill(a)
                if a and rng.random() < 0.5:
                    transfer(X, Y, a, priv=b"x", path=path,
                             l0=0, l1=shape.layers)
                elif a:
                    X.free(a)
            elif op < 0.58 and seqs:
                X.delete(seqs[rng.integers(len(seqs))])
            elif op < 0.64:
                X.evict(int(rng.integers(1, 4)), int(rng.integers(2)))
            elif op < 0.74:
                X.swap_out(int(rng.integers(1, 6)))
            elif op < 0.82:
                dram = [(X.inst, O.DRAM, i) for i, s in enumerate(X.o.state[O.DRAM])
                        if s in (O.INDEXED, O.ACTIVE)]
                if dram:
                    k = int(rng.integers(1, min(4, len(dram)) + 1))
                    pick = [dram[j] for j in rng.choice(len(dram), k, replace=False)]
                    X.swap_in(pick)
            elif op < 0.88 and seqs:
                t = seqs[rng.integers(len(seqs))]
                _, addrs = X.match(t, O.FLAG_MATCH_PIN)
                if addrs and rng.random() < 0.7:
                    X.unpin(addrs)
            elif op < 0.91:
                # invalid ops must fail identically and change nothing
                bad = [(X.inst, O.HBM, int(rng.integers(0, n_hbm)))]
                X.free(bad)
            elif op < 0.94:
                # MIXED allocation (HBM first, then DRAM), DRAM-only, free
                med = int(rng.choice([O.MIXED, O.DRAM]))
                a = X.alloc(int(rng.integers(1, 8)), med)
                if rng.random() < 0.5:
                    X.free(a)
            else:
                st = [(X.inst, O.HBM, i) for i, s in enumerate(X.o.state[O.HBM]) if s == O.ACTIVE]
                if st:
                    dst = Y.alloc(min(len(st), 2))
                    transfer(X, Y, st[: len(dst)], dst, oflags=O.FLAG_DST_GIVEN,
                             l0=int(rng.integers(0, shape.layers)), l1=shape.layers, path=path)
        except O.MPError:
            pass
        if step % 25 == 24:
            for t in twins:
                t.check_state()
    for t in twins:
        t.check_state()


@pytest.mark.parametrize("path", PATHS + PATHS_ASYNC)
def test_random_ops_tiny(path):
    for seed in range(3):
        random_ops(seed, TINY, 300, path)


@pytest.mark.parametrize("path", [M.PATH_FUSED | M.XFER_ASYNC, M.PATH_FUSED])
def test_random_ops_coalesced_launches(path, monkeypatch):
    """Launch coalescing batched by size only (no idle flush): many transfers
    per launch, interleaved with fills, frees, swaps, deletes and transfers in
    the other direction -- every hazard must flush in the right order."""
    monkeypatch.setenv("MP_COALESCE_NO_IDLE_FLUSH", "1")
    for seed in range(3):
        random_ops(200 + seed, TINY, 400, path, coalesce_mib=1)


@pytest.mark.parametrize("path", [M.PATH_FUSED | M.XFER_ASYNC, M.PATH_FUSED])
def test_random_ops_three_pools_coalesced(path, monkeypatch):
    """Three connected pools, transfers between every pair in both
    directions, size-only coalescing: batches from different sources into one
    pool, and batches reading a pool while another writes it, must flush in
    hazard order (batch_open) with the allocator writing into the open
    batch's id table."""
    monkeypatch.setenv("MP_COALESCE_NO_IDLE_FLUSH", "1")
    for seed in range(3):
        random_ops(500 + seed, TINY, 400, path, coalesce_mib=1, n_pools=3)


def test_random_ops_ce_and_swap_ce():
    """The library baselines: one copy-engine memcpy per chunk, and swap
    through device staging + copy-engine D2H/H2D (small staging: 2 blocks per
    round so multi-round swaps are exercised)."""
    for seed in range(2):
        random_ops(400 + seed, TINY, 300, M.PATH_CE, swap_flags=M.SWAP_CE,
                   staging_bytes=2 * TINY.block_bytes)


def test_random_ops_no_coalescing():
    # also the zero-copy swap transport (SM stores / loads on mapped DRAM)
    for seed in range(2):
        random_ops(300 + seed, TINY, 300, M.PATH_FUSED | M.XFER_ASYNC, coalesce_mib=-1,
                   swap_flags=M.SWAP_ZERO_COPY)


@pytest.mark.parametrize("path", [M.PATH_FUSED | M.XFER_ASYNC, M.PATH_STAGED])
def test_random_ops_bulk_copy_engine(path):
    """The cp.async.bulk (TMA) copy engine, tiny chunks (4 KiB < one 16 KiB piece)."""
    for seed in range(2):
        random_ops(100 + seed, TINY, 300, path, copy_kernel=2)


@pytest.mark.parametrize("copy_kernel", [1, 2])
def test_random_ops_ragged_chunk(copy_kernel):
    # chunk = 8*3*24*2 = 1152 B: not a multiple of the kernel's 4 KiB warp
    # unit / 16 KiB bulk piece -> exercises the predicated tail; B = 8
    shape = KVShape("ragged", 3, 3, 24, 8)
    random_ops(11, shape, 300, M.PATH_FUSED, copy_kernel=copy_kernel)
    random_ops(12, shape, 150, M.PATH_STAGED, copy_kernel=copy_kernel)


@pytest.mark.parametrize("copy_kernel", [1, 2])
def test_multi_piece_chunks(copy_kernel):
    # chunk = 16*16*88*2 = 45056 B = 2.75 bulk pieces / 11 vector units
    shape = KVShape("mp", 2, 16, 88, 16)
    random_ops(21, shape, 120, M.PATH_FUSED | M.XFER_ASYNC, n_hbm=40, n_dram=8,
               copy_kernel=copy_kernel)


# The NVLink dispatch on one GPU: force_peer makes same-GPU pools take the
# peer path (one-sided stores from the sender's stream through the peer slab
# table, the pool's peer engine and split), the path two pools on two GPUs
# take; every engine x split combination against the oracle.
PEER_ENGINES = {"vector-static": dict(peer_engine=1, peer_sched=1),
                "vector-dynamic": dict(peer_engine=1, peer_sched=2),
                "bulk-static": dict(peer_engine=2, peer_sched=1),
                "bulk-dynamic": dict(peer_engine=2, peer_sched=2)}


@pytest.mark.parametrize("engine", list(PEER_ENGINES))
@pytest.mark.parametrize("path", [M.PATH_FUSED, M.PATH_FUSED | M.XFER_ASYNC])
def test_random_ops_peer_dispatch(engine, path):
    for seed in range(2):
        random_ops(600 + seed, TINY, 300, path, force_peer=True, **PEER_ENGINES[engine])


@pytest.mark.parametrize("engine", list(PEER_ENGINES))
def test_multi_piece_chunks_peer_dispatch(engine):
    # 45056 B chunks: 2.75 bulk pieces / 11 vector units per chunk
    shape = KVShape("mp", 2, 16, 88, 16)
    random_ops(31, shape, 120, M.PATH_FUSED | M.XFER_ASYNC, n_hbm=40, n_dram=8,
               force_peer=True, **PEER_ENGINES[engine])


def test_random_ops_staged_async_small_ring():
    """STAGED without a host wait: 2 slots of 2 blocks, so one transfer wraps
    the ring and consecutive transfers reuse slots still being unpacked."""
    for seed in range(2):
        random_ops(700 + seed, TINY, 300, M.PATH_STAGED | M.XFER_ASYNC,
                   staging_bytes=4 * TINY.block_bytes, staging_slots=2)


def test_pack_unpack_np_take():
    import torch
    shape = KVShape("pk", 4, 4, 64, 16)     # c = 8 KiB: two 4 KiB units per chunk
    P = Twin(0, shape, 40)
    a = P.alloc(23)
    P.fill(a)
    rng = np.random.default_rng(3)
    sel = [a[i] for i in rng.permutation(23)[:17]]
    c = shape.chunk_bytes
    for l0, l1 in ((0, 4), (1, 3), (2, 3)):
        nj = 2 * (l1 - l0)
        stg = torch.zeros(17 * nj * c // 8, dtype=torch.int64, device="cuda:0")
        P.g.pack(M.np.array([M.make_addr(0, 0, x[2]) for x in sel], np.uint64), l0, l1,
                 stg.data_ptr())
        got = stg.cpu().numpy().view(np.uint64).reshape(17, nj, c // 8)
        for i, x in enumerate(sel):
            want = P.o.block_bytes(x)[2 * l0: 2 * l1]
            np.testing.assert_array_equal(got[i], want)
        # unpack o pack == identity on fresh blocks
        fresh = P.alloc(17)
        P.g.unpack(stg.data_ptr(), M.np.array([M.make_addr(0, 0, x[2]) for x in fresh],
                                              np.uint64), l0, l1)
        for i, x in enumerate(fresh):
            blk = P.g.debug_read_block(M.make_addr(0, 0, x[2]))
            np.testing.assert_array_equal(blk[2 * l0: 2 * l1], got[i])
        P.free(fresh)

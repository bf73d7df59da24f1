"""Stream-ordered integration with an engine's torch streams (mp_wait_event /
mp_record_event): the layer-by-layer pattern of P:369 / P:525 -- the engine
writes layer l's KV on its own stream, records an event, and the transfer of
layer l (caller-given destination blocks, no allocation step) must copy the
NEW content even though the host issues it before the write has run."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _pool(M, torch, inst, shape, n, **kw):
    c = shape.chunk_bytes
    region = torch.zeros(2 * shape.layers * n * c, dtype=torch.uint8, device="cuda:0")
    slabs = [region.data_ptr() + j * n * c for j in range(2 * shape.layers)]
    p = M.Pool(inst, 0, shape.layers, shape.kv_heads, shape.head_dim, shape.block_tokens, n,
               slabs=slabs, verify=True, **kw)
    return p, region.view(2 * shape.layers, n, c)


def test_layer_by_layer_waits_for_engine_stream():
    import torch
    from paper_2406_17565_b200 import mempool as M
    from workloads.configs import KVShape
    shape = KVShape("s", 4, 4, 64, 16)
    P, pr = _pool(M, torch, 0, shape, 16)
    D, dr = _pool(M, torch, 1, shape, 16)
    M.connect(P, D)
    src = P.alloc_mem(3)
    dst = D.alloc_mem(3)
    sid = M.addr_indices(src)
    did = M.addr_indices(dst)
    engine = torch.cuda.Stream()
    landed = torch.cuda.Event()
    for layer in range(shape.layers):
        ev = torch.cuda.Event()
        with torch.cuda.stream(engine):
            torch.cuda._sleep(2_000_000)            # the layer's "compute"
            for kv in range(2):                      # its KV write
                pr[2 * layer + kv, torch.as_tensor(sid, device="cuda:0")] = 10 * layer + kv + 1
            ev.record(engine)
        P.wait_event(ev)
        P.transfer(1, src, dst, layer_begin=layer, layer_end=layer + 1, flags=M.XFER_ASYNC)
    D.record_event(landed)
    torch.cuda.current_stream().wait_event(landed)
    got = dr[:, torch.as_tensor(did, device="cuda:0")].cpu().numpy()
    for j in range(2 * shape.layers):
        assert (got[j] == 10 * (j // 2) + j % 2 + 1).all(), f"chunk {j} copied stale KV"
    P.close()
    D.close()


def test_stream_ordered_alloc_reuses_block_still_being_read():
    """MP_ALLOC_STREAM_ORDERED: a block freed while an ASYNC transfer still
    reads it comes straight back (lowest-first, same ids as a draining alloc);
    the engine's write, ordered after mp_record_event, must not reach the
    receiver's copy."""
    import torch
    from paper_2406_17565_b200 import mempool as M
    from workloads.configs import KVShape
    shape = KVShape("s", 4, 4, 64, 16)
    P, pr = _pool(M, torch, 0, shape, 16)
    D, dr = _pool(M, torch, 1, shape, 16)
    M.connect(P, D)
    src = P.alloc_mem(3)
    sid = torch.as_tensor(M.addr_indices(src), device="cuda:0")
    pr[:, sid] = 7
    torch.cuda.synchronize()
    gate = torch.cuda.Event()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        torch.cuda._sleep(20_000_000)               # hold the copy back on the device
        gate.record(side)
    P.wait_event(gate)
    dst = P.transfer(1, src, flags=M.XFER_ASYNC)
    P.free_mem(src)
    again = P.alloc_mem(3, stream_ordered=True)
    assert list(M.addr_indices(again)) == list(M.addr_indices(src))
    ready = torch.cuda.Event()
    P.record_event(ready)
    engine = torch.cuda.Stream()
    engine.wait_event(ready)
    with torch.cuda.stream(engine):
        pr[:, sid] = 99                              # the new owner's KV write
    landed = torch.cuda.Event()
    D.record_event(landed)
    torch.cuda.current_stream().wait_event(landed)
    torch.cuda.current_stream().wait_stream(engine)
    did = torch.as_tensor(M.addr_indices(dst), device="cuda:0")
    assert (dr[:, did] == 7).all(), "receiver copied the new owner's bytes"
    assert (pr[:, sid] == 99).all()
    P.close()
    D.close()


def test_sampled_profiling_counts():
    """mp_profile(every=k): every k-th data-stream migration is timed with
    CUDA events; profiled_launches / profiled_bytes count all of them, and the
    harvest never blocks (ASYNC transfers stay queued until the sync)."""
    import torch
    from paper_2406_17565_b200 import mempool as M
    from workloads.configs import KVShape
    shape = KVShape("s", 4, 4, 64, 16)
    P, _ = _pool(M, torch, 0, shape, 64, coalesce_mib=-1)   # one launch per transfer
    D, _ = _pool(M, torch, 1, shape, 256, coalesce_mib=-1)
    M.connect(P, D)
    src = P.alloc_mem(8)
    P.debug_fill(src, 5)
    P.sync()
    per = 8 * 2 * shape.layers * shape.chunk_bytes
    for every, n in ((3, 10), (1, 5)):
        D.stats_reset()
        P.stats_reset()
        D.profile(True, every=every)
        P.profile(True, every=every)
        got = [P.transfer(1, src, flags=M.XFER_ASYNC | M.PATH_FUSED) for _ in range(n)]
        P.sync()
        D.sync()
        st = [D.stats(), P.stats()]
        prof = sum(s["profiled_launches"] for s in st)
        assert prof == n                                   # one launch per transfer
        assert sum(s["profiled_bytes"] for s in st) == n * per
        assert sum(s["timed_launches"] for s in st) == -(-n // every)
        assert sum(s["timed_bytes"] for s in st) == -(-n // every) * per
        assert sum(s["kernel_ms"] for s in st) > 0
        for p in (P, D):
            p.profile(False)
        for g in got:
            D.free_mem(g)
    P.close()
    D.close()

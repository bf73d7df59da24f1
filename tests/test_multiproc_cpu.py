"""Multi-process host logic on CPU (no GPU): the shared-memory mailbox that
carries the cross-process workflow messages, and the P/D pair
placement + handle bootstrap over torch.distributed with the gloo backend at
world_size 2."""
import multiprocessing as mp
import os
import uuid

import pytest


def _selftest(name, role, n, payload, q):
    try:
        from paper_2406_17565_b200 import mempool as M
        M.channel_selftest(name, role, n, payload)
        q.put((role, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((role, repr(e)))


@pytest.mark.parametrize("payload", [0, 7, 100_000])
def test_mailbox_two_processes(payload):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    name = f"/mpc_test_{uuid.uuid4().hex[:16]}"
    ps = [ctx.Process(target=_selftest, args=(name, r, 300, payload, q)) for r in (1, 0)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2406_17565_b200.topology import role_of
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    role = role_of(rank, world)
    # the same exchange mempool.exchange_handles performs, with a stand-in blob
    blob = bytes([rank]) * 64
    out = [None] * world
    dist.all_gather_object(out, (role.p_inst if role.kind == "P" else role.d_inst, blob))
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, role, out))


@pytest.mark.parametrize("world", [2, 4])
def test_pair_bootstrap_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 500) + world
    ps = [ctx.Process(target=_gloo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in ps:
        rank, role, out = q.get(timeout=120)
        res[rank] = (role, out)
    for p in ps:
        p.join(timeout=60)
    half = world // 2
    for rank, (role, out) in res.items():
        assert role.kind == ("P" if rank < half else "D")
        partner_role = res[role.partner][0]
        assert partner_role.partner == rank and partner_role.pair == role.pair
        # every rank sees every blob, keyed by instance id
        insts = [inst for inst, _ in out]
        assert sorted(insts) == list(range(world))
        assert out[role.partner][1] == bytes([role.partner]) * 64


def test_role_of_single_gpu():
    from paper_2406_17565_b200.topology import role_of
    r = role_of(0, 1)
    assert r.kind == "PD" and r.p_inst == 0 and r.d_inst == 1
    with pytest.raises(ValueError):
        role_of(0, 3)

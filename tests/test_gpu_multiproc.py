"""Cross-process MemPool on the GPU: P and D pools in two processes (both on
cuda:0 here -- the only GPU a test box has; on an 8-GPU box the same code maps
the peer's slabs over NVLink), bootstrapped with torch.distributed (gloo),
CUDA-IPC-mapped slabs/arena, shared-memory mailbox for the allocation /
insertion round trips.  The receiver's final state (index dump,
block states, every byte of every written block) must equal the oracle's
after the golden worked example (with and without DEDUP) plus plain
transfers with `private` payloads."""
import multiprocessing as mp
import os
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# Cross-process transports (name -> (pool keywords, path flag)).  On a 1-GPU
# box both processes share cuda:0; force_peer makes the sender treat the
# receiver as a remote GPU, so the NVLink dispatch (one-sided stores with
# the peer engine / split) is what runs and is checked here.
TINY_BLOCK = 16 * 1024
TRANSPORTS = {
    "fused-loopback": ({}, "PATH_FUSED"),
    "fused-vector-static": ({"force_peer": True, "peer_engine": 1, "peer_sched": 1},
                            "PATH_FUSED"),
    "fused-bulk-dynamic": ({"force_peer": True, "peer_engine": 2, "peer_sched": 2},
                           "PATH_FUSED"),
    # 2 slots of 2 tiny blocks: the ring wraps inside one transfer
    "ce-staged": ({"staging_bytes": 4 * TINY_BLOCK, "staging_slots": 2}, "PATH_STAGED"),
    "ce-per-chunk": ({}, "PATH_CE"),
    # ASYNC transfers enqueue their copy at the sender's next call
    # (MP_XFER_PIPELINE), after that call's request went out
    "fused-pipelined": ({}, "PATH_FUSED|XFER_PIPELINE"),
    "peer-vector-pipelined": ({"force_peer": True, "peer_engine": 1, "peer_sched": 1},
                              "PATH_FUSED|XFER_PIPELINE"),
    "ce-pipelined": ({}, "PATH_CE|XFER_PIPELINE"),
}


def _collect(q, ps, timeout):
    """Results of the worker processes; a worker that reports an error makes
    its peers hang in their next collective, so the first error is raised as
    soon as it arrives (with what the others did not report)."""
    import queue
    res = {}
    deadline = time.monotonic() + timeout
    while len(res) < len(ps):
        try:
            r, out = q.get(timeout=max(1.0, deadline - time.monotonic()))
        except queue.Empty:
            raise AssertionError(f"workers {sorted(set(range(len(ps))) - set(res))} did not "
                                 f"report within {timeout} s; got {sorted(res)}")
        res[r] = out
        if "error" in out:
            for p in ps:
                p.kill()
            raise AssertionError(f"worker {r}: {out['error']}")
    for p in ps:
        p.join(timeout=60)
    return res


def _run(rank, port, dedup, q, transport="fused-loopback"):
    try:
        import torch
        import torch.distributed as dist
        from paper_2406_17565_b200 import mempool as M
        from workloads.configs import TINY
        from workloads.traces import golden_prompts
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=2)
        torch.cuda.set_device(0)
        s = TINY
        kw, pname = TRANSPORTS[transport]
        path = sum(getattr(M, x) for x in pname.split("|"))
        pool = M.Pool(rank, 0, s.layers, s.kv_heads, s.head_dim, s.block_tokens, 64,
                      dram_blocks=16 if rank == 0 else 0, verify=True, **kw)
        blobs = M.exchange_handles(pool)
        pool.import_peer(blobs[1 - rank][1])
        dist.barrier()
        out = {}
        if rank == 0:
            _, p1, p2, p3 = golden_prompts()
            finals = []
            for i, p in enumerate((p1, p2, p3)):
                mt, matched = pool.match(p)
                new = pool.alloc_mem(-(-len(p) // 16) - len(matched))
                pool.debug_fill(new, 17565)
                full = np.concatenate([matched, new])
                pool.insert(p, full[: len(p) // 16])
                fl = (M.XFER_DEDUP if dedup else 0) | path
                if i == 2:
                    fl |= M.XFER_ASYNC
                final, moved = pool.transfer_with_insert(1, p, full, flags=fl,
                                                         priv=bytes(p.astype(np.int32)))
                finals.append((M.addr_indices(final).tolist(), moved))
            extra = pool.alloc_mem(3)
            pool.debug_fill(extra, 17565)
            d = pool.transfer(1, extra, flags=path, priv=b"plain")
            finals.append((M.addr_indices(d).tolist(), 3))
            # memory asymmetry: historical KV swapped out to this
            # process's pinned DRAM goes straight into the peer's HBM
            _old, dram = pool.swap_out(2)
            d = pool.transfer(1, dram, flags=path, priv=b"from-dram")
            finals.append((M.addr_indices(d).tolist(), 2))
            pool.send_mark(1, 7)
            out["finals"] = finals
        else:
            served, mark = pool.serve(timeout_ms=120_000, until_mark=True)
            assert mark == 7, (served, mark)
            msgs = []
            while True:
                m = pool.recv_poll()
                if m is None:
                    break
                msgs.append((m[0], m[1], m[2], M.addr_indices(m[3]).tolist()))
            out["msgs"] = msgs
        pool.sync()
        out["dump"] = pool.dump_index()
        out["states"] = pool.block_states().tolist()
        out["bytes"] = {i: pool.debug_read_block(M.make_addr(rank, 0, i))
                        for i, st in enumerate(out["states"]) if st != 0}
        dist.barrier()
        pool.close()
        dist.destroy_process_group()
        q.put((rank, out))
    except Exception as e:  # report to the parent
        import traceback
        q.put((rank, {"error": traceback.format_exc() + repr(e)}))


@pytest.mark.parametrize("transport", list(TRANSPORTS))
@pytest.mark.parametrize("dedup", [False, True])
def test_two_process_golden(dedup, transport):
    import oracle as O
    from workloads.configs import TINY
    from workloads.traces import golden_prompts
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + (os.getpid() % 200) + int(dedup) + 2 * list(TRANSPORTS).index(transport)
    ps = [ctx.Process(target=_run, args=(r, port, dedup, q, transport)) for r in range(2)]
    for p in ps:
        p.start()
    res = _collect(q, ps, 300)
    for r in (0, 1):
        assert "error" not in res[r], res[r].get("error")
    # oracle of the same sequence
    s = TINY
    oP = O.OraclePool(0, s.layers, s.kv_heads, s.head_dim, s.block_tokens, 64, n_dram=16,
                      seed=17565)
    oD = O.OraclePool(1, s.layers, s.kv_heads, s.head_dim, s.block_tokens, 64, seed=17565)
    _, p1, p2, p3 = golden_prompts()
    finals = []
    for p in (p1, p2, p3):
        _, matched = oP.match(p)
        new = oP.alloc_mem(-(-len(p) // 16) - len(matched), O.HBM)
        oP.fill(new)
        full = matched + new
        oP.insert(p, full[: len(p) // 16])
        f, moved, _ = O.transfer_with_insert(oP, oD, p, full,
                                             flags=O.FLAG_DEDUP if dedup else 0,
                                             priv=bytes(p.astype(np.int32)))
        finals.append(([a[2] for a in f], moved))
    extra = oP.alloc_mem(3, O.HBM)
    oP.fill(extra)
    d = O.transfer(oP, oD, extra, priv=b"plain")
    finals.append(([a[2] for a in d], 3))
    moved = oP.swap_out(2)
    d = O.transfer(oP, oD, [new for _o, new in moved], priv=b"from-dram")
    finals.append(([a[2] for a in d], 2))
    assert res[0]["finals"] == finals
    for pool_o, r in ((oP, 0), (oD, 1)):
        assert res[r]["dump"] == pool_o.dump_index()
        smap = {O.FREE: 0, O.ACTIVE: 1, O.INDEXED: 2, O.ORPHAN: 3}
        assert res[r]["states"] == [smap[x] for x in pool_o.state[O.HBM]]
        for i, got in res[r]["bytes"].items():
            if all(t is not None for t in pool_o.tags[O.HBM][i]):
                assert np.array_equal(got, pool_o.block_bytes((r, O.HBM, i))), (r, i)
    # `private` delivered byte-exact at the receiver, with the final addrs
    want_msgs = [(1 if k == "transfer_with_insert" else 0, src, priv, [a[2] for a in addrs])
                 for (k, src, priv, addrs) in oD.inbox]
    assert res[1]["msgs"] == want_msgs


def _stress(rank, port, q, transport="fused-loopback"):
    """Rank 0 streams back-to-back ASYNC transfers (random scattered 7B
    blocks) into rank 1's pool through the cross-process path, rank 1 serves;
    then every received block is compared with its source by weighted
    checksums of sampled chunks computed in each process on its own slabs."""
    try:
        import torch
        import torch.distributed as dist
        from paper_2406_17565_b200 import mempool as M
        from workloads.configs import LLAMA2_7B as S
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=2)
        torch.cuda.set_device(0)
        n = 512
        c = S.chunk_bytes
        region = torch.empty(2 * S.layers * n * c, dtype=torch.uint8, device="cuda:0")
        slabs = [region.data_ptr() + j * n * c for j in range(2 * S.layers)]
        kw, pname = TRANSPORTS[transport]
        if "staging_bytes" in kw:   # 7B blocks: 3 slots of 2 blocks
            kw = {"staging_bytes": 6 * S.block_bytes, "staging_slots": 3}
        path = sum(getattr(M, x) for x in pname.split("|"))
        pool = M.Pool(rank, 0, S.layers, S.kv_heads, S.head_dim, S.block_tokens, n,
                      slabs=slabs, verify=True, **kw)
        blobs = M.exchange_handles(pool)
        pool.import_peer(blobs[1 - rank][1])
        dist.barrier()
        pairs = []
        if rank == 0:
            rng = np.random.default_rng(3)
            src = pool.alloc_mem(n)
            pool.debug_fill(src, 41)
            for rnd in range(3):
                for _ in range(30):
                    sel = src[rng.choice(n, int(rng.integers(1, 12)), replace=False)]
                    d = pool.transfer(1, sel, flags=M.XFER_ASYNC | path)
                    if rnd == 2:
                        pairs += list(zip(M.addr_indices(sel).tolist(),
                                          M.addr_indices(d).tolist()))
                pool.send_mark(1, rnd)
                dist.barrier()
        else:
            for rnd in range(3):
                _served, mark = pool.serve(timeout_ms=120_000, until_mark=True)
                assert mark == rnd, (mark, rnd)
                pool.sync()
                while True:
                    m = pool.recv_poll()
                    if m is None:
                        break
                    if rnd < 2:   # freed: the next round re-allocates these ids
                        pool.free_mem(m[3])
                dist.barrier()
        pool.sync()
        torch.cuda.synchronize()
        g = torch.Generator(device="cuda:0").manual_seed(5)
        w = torch.randint(-2**31, 2**31, (c // 8,), generator=g, device="cuda:0")
        view = region.view(2 * S.layers, n, c).view(torch.int64)
        sums = torch.stack([(view[j] * w).sum(-1) for j in (0, 17, 63)], 1).cpu().numpy()
        out = {"pairs": pairs, "sums": sums.tolist()}
        dist.barrier()
        pool.close()
        dist.destroy_process_group()
        q.put((rank, out))
    except Exception as e:
        import traceback
        q.put((rank, {"error": traceback.format_exc() + repr(e)}))


@pytest.mark.parametrize("transport", list(TRANSPORTS))
def test_two_process_back_to_back_async(transport):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30300 + (os.getpid() % 40) + 50 * list(TRANSPORTS).index(transport)
    ps = [ctx.Process(target=_stress, args=(r, port, q, transport)) for r in range(2)]
    for p in ps:
        p.start()
    res = _collect(q, ps, 300)
    for r in (0, 1):
        assert "error" not in res[r], res[r].get("error")
    sums_p, sums_d = res[0]["sums"], res[1]["sums"]
    assert len(res[0]["pairs"]) > 30
    bad = [(s, d) for s, d in res[0]["pairs"] if sums_p[s] != sums_d[d]]
    assert not bad, f"{len(bad)} received blocks differ from their sources"


def _fanin(rank, port, q, rounds, per_round):
    """Rank 0 receives from ranks 1 and 2 at once (fan-in), enough transfers
    that its id arena wraps several times while the other sender's transfer
    sits between allocation reply and completion.  `private` carries the
    source ids; every received block is checksummed at the receiver before it
    is freed and compared with the sender's own checksum of the source."""
    try:
        import torch
        import torch.distributed as dist
        from paper_2406_17565_b200 import mempool as M
        from workloads.configs import TINY as S
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=3)
        torch.cuda.set_device(0)
        n = 1024 if rank == 0 else 64
        c = S.chunk_bytes
        region = torch.empty(2 * S.layers * n * c, dtype=torch.uint8, device="cuda:0")
        slabs = [region.data_ptr() + j * n * c for j in range(2 * S.layers)]
        pool = M.Pool(rank, 0, S.layers, S.kv_heads, S.head_dim, S.block_tokens, n,
                      slabs=slabs, verify=True)
        blobs = M.exchange_handles(pool)
        for r in range(3):
            if r != rank and (rank == 0 or r == 0):
                pool.import_peer(blobs[r][1])
        dist.barrier()
        g = torch.Generator(device="cuda:0").manual_seed(5)
        w = torch.randint(-2**31, 2**31, (c // 8,), generator=g, device="cuda:0")
        view = region.view(2 * S.layers, n, c).view(torch.int64)

        def sums(ids):
            t = torch.as_tensor(np.asarray(ids, np.int64), device="cuda:0")
            return torch.stack([(view[j][t] * w).sum(-1) for j in range(2 * S.layers)],
                               1).cpu().numpy().tolist()

        out = {}
        if rank == 0:
            got = []          # (sender, src id, checksum of the received block)
            for rnd in range(rounds):
                marks = 0
                while marks < 2:
                    _s, mark = pool.serve(timeout_ms=120_000, until_mark=True)
                    marks += mark is not None
                pool.sync()
                msgs = []
                while True:
                    m = pool.recv_poll()
                    if m is None:
                        break
                    msgs.append(m)
                ids = [int(x) for m in msgs for x in M.addr_indices(m[3])]
                cs = sums(ids) if ids else []
                k = 0
                for m in msgs:
                    srcs = np.frombuffer(m[2], np.int32)
                    for sid in srcs:
                        got.append((int(m[1]), int(sid), cs[k]))
                        k += 1
                    pool.free_mem(m[3])
                dist.barrier()
            out["got"] = got
            out["arena_wraps_min"] = 0
        else:
            rng = np.random.default_rng(rank)
            src = pool.alloc_mem(n)
            pool.debug_fill(src, 77)
            pool.sync()
            out["sums"] = sums(list(range(n)))
            for rnd in range(rounds):
                for _ in range(per_round):
                    k = int(rng.integers(1, 7))
                    sel = np.sort(rng.choice(n, k, replace=False))
                    # sender 1 pipelines (its copy is enqueued at its next call)
                    pool.transfer(0, src[sel],
                                  flags=M.XFER_ASYNC | (M.XFER_PIPELINE if rank == 1 else 0),
                                  priv=sel.astype(np.int32).tobytes())
                pool.send_mark(0, rnd)
                dist.barrier()
        pool.sync()
        dist.barrier()
        pool.close()
        dist.destroy_process_group()
        q.put((rank, out))
    except Exception as e:
        import traceback
        q.put((rank, {"error": traceback.format_exc() + repr(e)}))


def test_fan_in_two_senders_arena_wraps():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29900 + (os.getpid() % 40)
    # 2 senders x 160 rounds x 120 transfers x 3.5 blocks ~ 134K receiver ids:
    # the 65536-id arena wraps twice
    rounds, per_round = 160, 120
    ps = [ctx.Process(target=_fanin, args=(r, port, q, rounds, per_round)) for r in range(3)]
    for p in ps:
        p.start()
    res = _collect(q, ps, 900)
    for r in (0, 1, 2):
        assert "error" not in res[r], res[r].get("error")
    got = res[0]["got"]
    assert len(got) > 2 * rounds * per_round
    bad = [(s, i) for s, i, cs in got if res[s]["sums"][i] != cs]
    assert not bad, f"{len(bad)} of {len(got)} received blocks differ from their sources"


# ---------------------------------------------------------------------------
# Randomized cross-process parity: rank 0 (P) runs a seeded op list -- engine
# prefill + transfer_with_insert with / without DEDUP, sync / async, swap_out,
# transfers of swapped-out (DRAM) blocks, deletes -- against rank 1 (D), which
# serves and, at every end-of-phase mark, frees the partial / plain-transfer
# blocks it received and deletes some of the prompts.  The parent replays the
# same list on two oracle pools; per-op results, index dumps, block states and
# every written block's bytes must match.
def _rand_ops(seed, n_phases=10, per_phase=14):
    rng = np.random.default_rng(seed)
    B = 16
    base = [rng.integers(3, 40, size=int(rng.integers(2, 5)) * B).astype(np.int32)
            for _ in range(3)]
    prompts, phases = [], []
    for ph in range(n_phases):
        ops = []
        for _ in range(per_phase):
            r = rng.random()
            if r < 0.6 or not prompts:
                b = base[int(rng.integers(len(base)))]
                cut = int(rng.integers(0, len(b) + 1))
                tail = rng.integers(3, 40, size=int(rng.integers(1, 3 * B))).astype(np.int32)
                prompts.append(np.concatenate([b[:cut], tail]).astype(np.int32))
                ops.append(("twi", len(prompts) - 1, bool(rng.random() < 0.6),
                            bool(rng.random() < 0.5)))
            elif r < 0.75:
                ops.append(("swap_out", int(rng.integers(1, 4))))
            elif r < 0.88:
                ops.append(("xfer_dram", int(rng.integers(1, 3))))
            else:
                ops.append(("p_delete", int(rng.integers(len(prompts)))))
        phases.append(ops)
    return prompts, phases


def _d_retire(msgs, prompts, phase_ops):
    """D's end-of-phase work, from its delivered messages (kind 1 =
    transfer_with_insert, 0 = plain transfer) -- returns the ops to apply."""
    frees, deletes = [], []
    twis = [op for op in phase_ops if op[0] == "twi"]
    k = 0
    for kind, addrs in msgs:
        if kind == 0:
            frees.extend(addrs)
        else:
            i = twis[k][1]
            k += 1
            if len(prompts[i]) % 16:
                frees.append(addrs[-1])              # the trailing partial block
            if i % 2 == 0:
                deletes.append(i)                    # odd prompts stay cached
    return frees, deletes


def _rand_worker(rank, port, seed, q, transport="fused-loopback"):
    try:
        import torch
        import torch.distributed as dist
        from paper_2406_17565_b200 import mempool as M
        from workloads.configs import TINY as S
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=2)
        torch.cuda.set_device(0)
        prompts, phases = _rand_ops(seed)
        kw, pname = TRANSPORTS[transport]
        path = sum(getattr(M, x) for x in pname.split("|"))
        pool = M.Pool(rank, 0, S.layers, S.kv_heads, S.head_dim, S.block_tokens,
                      48 if rank == 0 else 24, dram_blocks=12 if rank == 0 else 0, verify=True,
                      **kw)
        blobs = M.exchange_handles(pool)
        pool.import_peer(blobs[1 - rank][1])
        dist.barrier()
        res = []
        for ph, ops in enumerate(phases):
            if rank == 0:
                for op in ops:
                    try:
                        if op[0] == "twi":
                            _, i, dedup, asy = op
                            t = prompts[i]
                            _, m = pool.match(t)
                            new = pool.alloc_mem(-(-len(t) // 16) - len(m))
                            pool.debug_fill(new, 17565)
                            full = np.concatenate([m, new])
                            pool.insert(t, full[: len(t) // 16])
                            fl = ((M.XFER_DEDUP if dedup else 0) | (M.XFER_ASYNC if asy else 0)
                                  | path)
                            fin, moved = pool.transfer_with_insert(1, t, full, flags=fl)
                            if len(t) % 16:
                                pool.free_mem(full[-1:])
                            res.append(("twi", M.addr_indices(fin).tolist(), moved))
                        elif op[0] == "swap_out":
                            o, nw = pool.swap_out(op[1])
                            res.append(("swap_out", M.addr_indices(o).tolist(),
                                        M.addr_indices(nw).tolist()))
                        elif op[0] == "xfer_dram":
                            st = pool.block_states(M.DRAM)
                            ids = [i for i, s in enumerate(st) if s in (1, 2)][: op[1]]
                            if ids:
                                src = np.array([M.make_addr(0, M.DRAM, i) for i in ids],
                                               np.uint64)
                                d = pool.transfer(1, src, flags=path)
                                res.append(("xfer_dram", ids, M.addr_indices(d).tolist()))
                        elif op[0] == "p_delete":
                            pool.delete(prompts[op[1]])
                    except M.MempoolError as e:
                        res.append(("error", op[0], e.name))
                pool.send_mark(1, ph)
            else:
                _s, mark = pool.serve(timeout_ms=120_000, until_mark=True)
                assert mark == ph, (mark, ph)
                pool.sync()
                msgs = []
                while True:
                    m = pool.recv_poll()
                    if m is None:
                        break
                    msgs.append((m[0], [int(a) for a in m[3]]))
                frees, deletes = _d_retire(msgs, prompts, ops)
                if frees:
                    pool.free_mem(np.array(frees, np.uint64))
                for i in deletes:
                    pool.delete(prompts[i])
            dist.barrier()
        pool.sync()
        out = {"res": res, "dump": pool.dump_index(),
               "states": [pool.block_states(M.HBM).tolist(),
                          pool.block_states(M.DRAM).tolist() if rank == 0 else []]}
        out["bytes"] = {}
        for med in (0, 1):
            for i, s in enumerate(out["states"][med]):
                if s != 0:
                    out["bytes"][(med, i)] = pool.debug_read_block(M.make_addr(rank, med, i))
        dist.barrier()
        pool.close()
        dist.destroy_process_group()
        q.put((rank, out))
    except Exception as e:
        import traceback
        q.put((rank, {"error": traceback.format_exc() + repr(e)}))


def _rand_oracle(seed):
    import oracle as O
    from workloads.configs import TINY as S
    prompts, phases = _rand_ops(seed)
    mk = lambda inst, n, nd: O.OraclePool(inst, S.layers, S.kv_heads,  # noqa: E731
                                          S.head_dim, S.block_tokens, n, n_dram=nd,
                                          seed=17565)
    P, D = mk(0, 48, 12), mk(1, 24, 0)   # a small receiver: it evicts (R2, R8)
    res = []
    for ph, ops in enumerate(phases):
        msgs = []
        for op in ops:
            try:
                if op[0] == "twi":
                    _, i, dedup, _asy = op
                    t = prompts[i]
                    _, m = P.match(t)
                    new = P.alloc_mem(-(-len(t) // 16) - len(m), O.HBM)
                    P.fill(new)
                    full = list(m) + new
                    P.insert(t, full[: len(t) // 16])
                    fin, moved, _ = O.transfer_with_insert(P, D, t, full,
                                                           flags=O.FLAG_DEDUP if dedup else 0)
                    if len(t) % 16:
                        P.free_mem(full[-1:])
                    res.append(("twi", [a[2] for a in fin], moved))
                    msgs.append((1, fin))
                elif op[0] == "swap_out":
                    mv = P.swap_out(op[1])
                    res.append(("swap_out", [o[2] for o, _ in mv], [n[2] for _, n in mv]))
                elif op[0] == "xfer_dram":
                    ids = [i for i, s in enumerate(P.state[O.DRAM])
                           if s in (O.ACTIVE, O.INDEXED)][: op[1]]
                    if ids:
                        d = O.transfer(P, D, [(0, O.DRAM, i) for i in ids])
                        res.append(("xfer_dram", ids, [a[2] for a in d]))
                        msgs.append((0, d))
                elif op[0] == "p_delete":
                    P.delete(prompts[op[1]])
            except O.MPError as e:
                res.append(("error", op[0], e.name))
        frees, deletes = _d_retire(msgs, prompts, ops)
        if frees:
            D.free_mem(frees)
        for i in deletes:
            D.delete(prompts[i])
    return P, D, res


@pytest.mark.parametrize("seed,transport", [(3, "fused-loopback"), (11, "fused-loopback"),
                                            (29, "fused-loopback"), (5, "fused-vector-static"),
                                            (7, "fused-bulk-dynamic"), (13, "ce-staged"),
                                            (17, "ce-per-chunk"), (19, "fused-pipelined"),
                                            (23, "fused-pipelined")])
def test_two_process_random_ops(seed, transport):
    import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29990 + (os.getpid() % 8) + seed
    ps = [ctx.Process(target=_rand_worker, args=(r, port, seed, q, transport)) for r in range(2)]
    for p in ps:
        p.start()
    got = _collect(q, ps, 600)
    for r in (0, 1):
        assert "error" not in got[r], got[r].get("error")
    P, D, res = _rand_oracle(seed)
    assert got[0]["res"] == res
    smap = {O.FREE: 0, O.ACTIVE: 1, O.INDEXED: 2, O.ORPHAN: 3}
    for pool_o, r in ((P, 0), (D, 1)):
        assert got[r]["dump"] == pool_o.dump_index(), r
        assert got[r]["states"][0] == [smap[x] for x in pool_o.state[O.HBM]], r
        if r == 0:
            assert got[r]["states"][1] == [smap[x] for x in pool_o.state[O.DRAM]]
        n = 0
        for (med, i), b in got[r]["bytes"].items():
            if all(t is not None for t in pool_o.tags[med][i]):
                assert np.array_equal(b, pool_o.block_bytes((r, med, i))), (r, med, i)
                n += 1
        assert n > 0


# ---------------------------------------------------------------------------
# Cross-process ReAct (configs[3] shape of work, PD-Caching-3) at
# tiny size, against the oracle: per turn P -> D transfer_with_insert with
# DEDUP of the prompt, D appends the generated blocks (engine stand-in fills
# them), D -> P suffix transfer_with_insert from block floor(prompt/B) (R3);
# both sides free their partial blocks, sessions end with deletes.  Lockstep
# (end-of-step marks both ways) so the oracle can replay the same order.
def _react_sessions(seed, n_sessions=4):
    rng = np.random.default_rng(seed)
    tok = lambda n: rng.integers(3, 40, size=n).astype(np.int32)  # noqa: E731
    shared = tok(40)
    out = []
    for _ in range(n_sessions):
        prompt = np.concatenate([shared, tok(int(rng.integers(3, 20)))])
        turns = []
        for _ in range(int(rng.integers(2, 4))):
            gen = tok(int(rng.integers(5, 40)))
            turns.append((prompt, gen))
            prompt = np.concatenate([prompt, gen, tok(int(rng.integers(3, 20)))])
        out.append(turns)
    return out


def _react_worker(rank, port, seed, q, transport):
    try:
        import torch
        import torch.distributed as dist
        from paper_2406_17565_b200 import mempool as M
        from workloads.configs import TINY as S
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=2)
        torch.cuda.set_device(0)
        kw, pname = TRANSPORTS[transport]
        path = sum(getattr(M, x) for x in pname.split("|"))
        pool = M.Pool(rank, 0, S.layers, S.kv_heads, S.head_dim, S.block_tokens, 96,
                      verify=True, **kw)
        blobs = M.exchange_handles(pool)
        pool.import_peer(blobs[1 - rank][1])
        dist.barrier()
        B, other = S.block_tokens, 1 - rank
        res, step = [], 0

        def prefill(t):
            _, m = pool.match(t)
            new = pool.alloc_mem(-(-len(t) // B) - len(m))
            if len(new):
                pool.debug_fill(new, 17565)
            full = np.concatenate([m, new])
            pool.insert(t, full[: len(t) // B])
            return full

        def poll():
            m = pool.recv_poll()
            assert m is not None and pool.recv_poll() is None
            return m[3]

        for turns in _react_sessions(seed):
            for prompt, gen in turns:
                whole = np.concatenate([prompt, gen])
                k = len(prompt) // B
                if rank == 0:
                    src = prefill(prompt)
                    fin, nm = pool.transfer_with_insert(1, prompt, src,
                                                        flags=M.XFER_DEDUP | M.XFER_ASYNC | path)
                    res.append(("p2d", M.addr_indices(fin).tolist(), nm))
                    pool.send_mark(1, step)
                    _s, mark = pool.serve(timeout_ms=120_000, until_mark=True)
                    assert mark == step + 1, (mark, step)
                    back = poll()
                    res.append(("d2p_final", M.addr_indices(back).tolist()))
                    pool.free_mem(back[len(whole) // B:])
                    pool.free_mem(src[k:])
                else:
                    _s, mark = pool.serve(timeout_ms=120_000, until_mark=True)
                    assert mark == step, (mark, step)
                    fin = poll()
                    pool.free_mem(fin[k:])
                    d = prefill(whole)
                    _, nm = pool.transfer_with_insert(0, whole, d[k:], flags=M.XFER_ASYNC | path)
                    res.append(("d2p", nm))
                    pool.free_mem(d[len(whole) // B:])
                    pool.send_mark(0, step + 1)
                step += 2
            for prompt, gen in turns:
                pool.delete(np.concatenate([prompt, gen]))
            dist.barrier()
        pool.sync()
        out = {"res": res, "dump": pool.dump_index(), "states": pool.block_states(M.HBM).tolist()}
        out["bytes"] = {i: pool.debug_read_block(M.make_addr(rank, M.HBM, i))
                        for i, s in enumerate(out["states"]) if s != 0}
        dist.barrier()
        pool.close()
        dist.destroy_process_group()
        q.put((rank, out))
    except Exception as e:
        import traceback
        q.put((rank, {"error": traceback.format_exc() + repr(e)}))


def _react_oracle(seed):
    import oracle as O
    from workloads.configs import TINY as S
    B = S.block_tokens
    mk = lambda inst: O.OraclePool(inst, S.layers, S.kv_heads, S.head_dim, B, 96,  # noqa: E731
                                   seed=17565)
    P, D = mk(0), mk(1)
    res = {0: [], 1: []}

    def prefill(X, t):
        _, m = X.match(t)
        new = X.alloc_mem(-(-len(t) // B) - len(m), O.HBM)
        if new:
            X.fill(new)
        full = list(m) + new
        X.insert(t, full[: len(t) // B])
        return full

    for turns in _react_sessions(seed):
        for prompt, gen in turns:
            whole = np.concatenate([prompt, gen])
            k = len(prompt) // B
            src = prefill(P, prompt)
            fin, nm, _ = O.transfer_with_insert(P, D, prompt, src, flags=O.FLAG_DEDUP)
            res[0].append(("p2d", [a[2] for a in fin], nm))
            D.free_mem(fin[k:])
            d = prefill(D, whole)
            back, nm2, _ = O.transfer_with_insert(D, P, whole, d[k:], flags=0)
            res[1].append(("d2p", nm2))
            D.free_mem(d[len(whole) // B:])
            res[0].append(("d2p_final", [a[2] for a in back]))
            P.free_mem(back[len(whole) // B:])
            P.free_mem(src[k:])
        for prompt, gen in turns:
            w = np.concatenate([prompt, gen])
            P.delete(w)
            D.delete(w)
    return P, D, res


@pytest.mark.parametrize("seed,transport", [(41, "fused-loopback"), (43, "fused-vector-static"),
                                            (47, "ce-staged"), (53, "ce-per-chunk"),
                                            (59, "fused-pipelined")])
def test_two_process_react_vs_oracle(seed, transport):
    import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30700 + (os.getpid() % 20) + seed
    ps = [ctx.Process(target=_react_worker, args=(r, port, seed, q, transport))
          for r in range(2)]
    for p in ps:
        p.start()
    got = _collect(q, ps, 600)
    for r in (0, 1):
        assert "error" not in got[r], got[r].get("error")
    P, D, res = _react_oracle(seed)
    smap = {O.FREE: 0, O.ACTIVE: 1, O.INDEXED: 2, O.ORPHAN: 3}
    for pool_o, r in ((P, 0), (D, 1)):
        assert got[r]["res"] == res[r], r
        assert got[r]["dump"] == pool_o.dump_index(), r
        assert got[r]["states"] == [smap[x] for x in pool_o.state[O.HBM]], r
        n = 0
        for i, b in got[r]["bytes"].items():
            if all(t is not None for t in pool_o.tags[O.HBM][i]):
                assert np.array_equal(b, pool_o.block_bytes((r, O.HBM, i))), (r, i)
                n += 1
        assert n > 0, r


# ---------------------------------------------------------------------------
# MP_XFER_PIPELINE contract (include/mempool.h): the call returns after the
# receiver's reply with the final addrs; the copy is enqueued by the sender's
# next call -- not by mp_match -- and consecutive pipelined transfers to the
# same peer merge into one launch while the sender's GPU is busy (size-only
# batching, MP_COALESCE_NO_IDLE_FLUSH=1, stands in for a busy GPU here); on an
# idle GPU the next transfer enqueues the pending copy instead of merging;
# mp_sync enqueues and completes it.
def _pipe_worker(rank, port, q, idle_flush=False):
    try:
        if not idle_flush:
            os.environ["MP_COALESCE_NO_IDLE_FLUSH"] = "1"
        import torch
        import torch.distributed as dist
        from paper_2406_17565_b200 import mempool as M
        from workloads.configs import TINY as S
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=2)
        torch.cuda.set_device(0)
        pool = M.Pool(rank, 0, S.layers, S.kv_heads, S.head_dim, S.block_tokens, 64, verify=True)
        blobs = M.exchange_handles(pool)
        pool.import_peer(blobs[1 - rank][1])
        dist.barrier()
        out = {}
        if rank == 0:
            src = pool.alloc_mem(12)
            pool.debug_fill(src, 5)
            pool.sync()
            pool.stats_reset()
            fl = M.XFER_ASYNC | M.XFER_PIPELINE
            d1 = pool.transfer(1, src[:4], flags=fl)
            out["after_first"] = pool.stats()["kernel_launches"]
            pool.match(np.arange(40, dtype=np.int32))          # host only: no flush
            out["after_match"] = pool.stats()["kernel_launches"]
            d2 = pool.transfer(1, src[4:9], flags=fl)            # merges (size-only batching)
            out["after_second"] = pool.stats()["kernel_launches"]
            pool.sync()                                         # enqueues and completes
            out["after_sync"] = pool.stats()["kernel_launches"]
            d3 = pool.transfer(1, src[9:], flags=fl)
            pool.send_mark(1, 1)                                # any other call flushes
            out["after_mark"] = pool.stats()["kernel_launches"]
            out["pairs"] = list(zip(M.addr_indices(src).tolist(),
                                    M.addr_indices(np.concatenate([d1, d2, d3])).tolist()))
            out["src"] = {int(i): pool.debug_read_block(a) for i, a in
                          zip(M.addr_indices(src).tolist(), src)}
            dist.barrier()
        else:
            _s, mark = pool.serve(timeout_ms=120_000, until_mark=True)
            assert mark == 1
            pool.sync()                                         # joins the sender's copies
            out["dst"] = {i: pool.debug_read_block(M.make_addr(1, M.HBM, i)) for i in range(12)}
            dist.barrier()
        dist.barrier()
        pool.close()
        dist.destroy_process_group()
        q.put((rank, out))
    except Exception as e:
        import traceback
        q.put((rank, {"error": traceback.format_exc() + repr(e)}))


@pytest.mark.parametrize("idle_flush", [False, True])
def test_two_process_pipeline_contract(idle_flush):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30900 + (os.getpid() % 40) + (40 if idle_flush else 0)
    ps = [ctx.Process(target=_pipe_worker, args=(r, port, q, idle_flush)) for r in range(2)]
    for p in ps:
        p.start()
    res = _collect(q, ps, 300)
    s = res[0]
    assert s["after_first"] == 0 and s["after_match"] == 0   # still pending
    if idle_flush:   # the sender's GPU is idle: the second call enqueues the first copy
        assert s["after_second"] == 1
        assert s["after_sync"] == 2
        assert s["after_mark"] == 3
    else:
        assert s["after_second"] == 0                         # merged, still pending
        assert s["after_sync"] == 1                           # one launch for both
        assert s["after_mark"] == 2
    for si, di in s["pairs"]:
        assert np.array_equal(res[1]["dst"][di], s["src"][si]), (si, di)


# ---------------------------------------------------------------------------
# Edge cases of the cross-process protocol, each against the oracle replayed
# in the parent: an empty transfer, a DEDUP transfer that moves nothing, a
# receiver out of memory (error, no state change, sequence numbers intact),
# then ordinary transfers -- synchronous, ASYNC and pipelined.
_EDGE_FLAGS = [0, "ASYNC", "ASYNC|PIPELINE"]


def _edge_worker(rank, port, q, mode):
    try:
        import torch
        import torch.distributed as dist
        from paper_2406_17565_b200 import mempool as M
        from workloads.configs import TINY as S
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=2)
        torch.cuda.set_device(0)
        fl = 0 if mode == 0 else sum(getattr(M, "XFER_" + x) for x in mode.split("|"))
        pool = M.Pool(rank, 0, S.layers, S.kv_heads, S.head_dim, S.block_tokens,
                      64 if rank == 0 else 16, verify=True)
        blobs = M.exchange_handles(pool)
        pool.import_peer(blobs[1 - rank][1])
        dist.barrier()
        out = {}
        if rank == 0:
            res = []
            src = pool.alloc_mem(40)
            pool.debug_fill(src, 3)
            t = np.arange(3, 3 + 64, dtype=np.int32)           # 4 full blocks
            res.append(("empty", M.addr_indices(pool.transfer(1, src[:0], flags=fl)).tolist()))
            fin, nm = pool.transfer_with_insert(1, t, src[:4], flags=fl | M.XFER_DEDUP)
            res.append(("twi", M.addr_indices(fin).tolist(), nm))
            fin, nm = pool.transfer_with_insert(1, t, src[:4], flags=fl | M.XFER_DEDUP)
            res.append(("twi_dedup_all", M.addr_indices(fin).tolist(), nm))
            try:
                pool.transfer(1, src[4:24], flags=fl)            # 20 > 12 free at D
                res.append(("oom", "no error"))
            except M.MempoolError as e:
                res.append(("oom", e.name))
            d = pool.transfer(1, src[24:30], flags=fl)
            res.append(("after", M.addr_indices(d).tolist()))
            pool.send_mark(1, 1)
            out["res"] = res
            out["src"] = {i: pool.debug_read_block(src[i]) for i in list(range(4)) + list(range(24, 30))}
        else:
            _s, mark = pool.serve(timeout_ms=120_000, until_mark=True)
            assert mark == 1
            pool.sync()
            out["states"] = pool.block_states(M.HBM).tolist()
            out["dump"] = pool.dump_index()
            out["bytes"] = {i: pool.debug_read_block(M.make_addr(1, M.HBM, i))
                            for i, st in enumerate(out["states"]) if st}
        dist.barrier()
        pool.close()
        dist.destroy_process_group()
        q.put((rank, out))
    except Exception as e:
        import traceback
        q.put((rank, {"error": traceback.format_exc() + repr(e)}))


@pytest.mark.parametrize("mode", _EDGE_FLAGS)
def test_two_process_edges_vs_oracle(mode):
    import oracle as O
    from workloads.configs import TINY as S
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31100 + (os.getpid() % 30) + 3 * _EDGE_FLAGS.index(mode)
    ps = [ctx.Process(target=_edge_worker, args=(r, port, q, mode)) for r in range(2)]
    for p in ps:
        p.start()
    got = _collect(q, ps, 300)
    mk = lambda inst, n: O.OraclePool(inst, S.layers, S.kv_heads, S.head_dim,  # noqa: E731
                                      S.block_tokens, n, seed=3)
    P, D = mk(0, 64), mk(1, 16)
    src = P.alloc_mem(40, O.HBM)
    P.fill(src)
    t = np.arange(3, 3 + 64, dtype=np.int32)
    want = [("empty", [a[2] for a in O.transfer(P, D, src[:0])])]
    for tag in ("twi", "twi_dedup_all"):
        fin, nm, _ = O.transfer_with_insert(P, D, t, src[:4], flags=O.FLAG_DEDUP)
        want.append((tag, [a[2] for a in fin], nm))
    try:
        O.transfer(P, D, src[4:24])
        want.append(("oom", "no error"))
    except O.MPError as e:
        want.append(("oom", e.name))
    want.append(("after", [a[2] for a in O.transfer(P, D, src[24:30])]))
    assert [list(x) for x in got[0]["res"]] == [list(x) for x in want]
    smap = {O.FREE: 0, O.ACTIVE: 1, O.INDEXED: 2, O.ORPHAN: 3}
    assert got[1]["states"] == [smap[x] for x in D.state[O.HBM]]
    assert got[1]["dump"] == D.dump_index()
    for i, b in got[1]["bytes"].items():
        assert np.array_equal(b, D.block_bytes((1, O.HBM, i))), i

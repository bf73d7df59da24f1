"""Back-to-back ASYNC transfers at the host's full speed (no oracle between
calls), so coalesced batches are built while earlier migration kernels are
still running -- the regime bench.py times.  Every received block must equal
its source block byte for byte (compared on the device with torch).  The
slower twin-harness tests leave the GPU idle between calls and cannot see
cross-launch hazards on the library's own tables."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _pool(M, torch, inst, shape, n, **kw):
    c = shape.chunk_bytes
    region = torch.empty(2 * shape.layers * n * c, dtype=torch.uint8, device="cuda:0")
    slabs = [region.data_ptr() + j * n * c for j in range(2 * shape.layers)]
    p = M.Pool(inst, 0, shape.layers, shape.kv_heads, shape.head_dim, shape.block_tokens, n,
               slabs=slabs, verify=True, **kw)
    return p, region.view(2 * shape.layers, n, c)


@pytest.mark.parametrize("copy_kernel", [0, 1])
def test_back_to_back_async_transfers_bytes(copy_kernel):
    import torch
    from paper_2406_17565_b200 import mempool as M
    from workloads.configs import LLAMA2_7B as S
    n = 1536
    P, pr = _pool(M, torch, 0, S, n, copy_kernel=copy_kernel)
    D, dr = _pool(M, torch, 1, S, n, copy_kernel=copy_kernel)
    M.connect(P, D)
    rng = np.random.default_rng(5)
    src = P.alloc_mem(n)
    P.debug_fill(src, 99)
    P.sync()
    pairs = []
    for rnd in range(6):
        got = []
        for _ in range(40):
            k = int(rng.integers(1, 24))
            sel = src[rng.choice(n, k, replace=False)]
            dst = P.transfer(1, sel, flags=M.XFER_ASYNC)
            got.append((M.addr_indices(sel), M.addr_indices(dst), dst))
        P.sync()
        D.sync()
        s_ids = torch.as_tensor(np.concatenate([g[0] for g in got]), device="cuda:0")
        d_ids = torch.as_tensor(np.concatenate([g[1] for g in got]), device="cuda:0")
        for j in range(0, 2 * S.layers, 7):
            bad = (dr[j, d_ids] != pr[j, s_ids]).any(dim=1).nonzero().flatten()
            assert bad.numel() == 0, f"round {rnd}: {bad.numel()} blocks differ in chunk {j}"
        D.free_mem(np.concatenate([g[2] for g in got]))
    P.close()
    D.close()


@pytest.mark.parametrize("coalesce_mib", [0, -1, 64, 1024])   # default 4 GiB, off, 64 MiB, 1 GiB
def test_bench_pattern_dedup_retire_bytes(coalesce_mib):
    """bench.py's step at host speed: P.match + DEDUP transfer_with_insert
    (ASYNC) per request, D retires the batch (free partials, delete prompts),
    blocks are re-allocated by the next batch while earlier copies may still
    run.  After every batch, each request's blocks at D equal P's."""
    import torch
    from paper_2406_17565_b200 import mempool as M
    from workloads import traces
    from workloads.configs import LLAMA2_7B as S
    B = S.block_tokens
    n = 1024
    kw = {"coalesce_mib": coalesce_mib}
    P, pr = _pool(M, torch, 0, S, n, **kw)
    D, dr = _pool(M, torch, 1, S, 640, **kw)
    M.connect(P, D)
    sessions = traces.sharegpt_like(31, n_sessions=400)
    reqs, used = [], 0
    for s in sessions:
        blocks = -(-len(s.turns[-1].prompt) // B) + len(s.turns)
        if used + blocks > 0.9 * n:
            continue
        used += blocks
        for t in s.turns:
            _, m = P.match(t.prompt)
            new = P.alloc_mem(-(-len(t.prompt) // B) - len(m))
            P.debug_fill(new, 7)
            full = np.concatenate([m, new])
            P.insert(t.prompt, full[: len(t.prompt) // B])
            reqs.append((t.prompt, full[len(t.prompt) // B:]))
    P.sync()
    for step in range(4):
        batch = reqs[step * len(reqs) // 4:(step + 1) * len(reqs) // 4]
        done = []
        for prompt, partial in batch:
            _, m = P.match(prompt)
            src = np.concatenate([m, partial])
            fin, _ = P.transfer_with_insert(1, prompt, src, flags=M.XFER_DEDUP | M.XFER_ASYNC)
            done.append((prompt, src, fin))
        D.sync()
        P.sync()
        s_ids = torch.as_tensor(np.concatenate([M.addr_indices(s) for _, s, _ in done]),
                                device="cuda:0")
        d_ids = torch.as_tensor(np.concatenate([M.addr_indices(f) for _, _, f in done]),
                                device="cuda:0")
        for j in (0, 31, 63):
            bad = (dr[j, d_ids] != pr[j, s_ids]).any(dim=1).nonzero().flatten()
            assert bad.numel() == 0, f"step {step}: {bad.numel()} blocks differ in chunk {j}"
        D.free_mem(np.concatenate([f[len(p) // B:] for p, _, f in done]))
        for prompt, _, _ in done:
            D.delete(prompt)
    P.close()
    D.close()


def test_static_split_engines():
    """MP_BULK_SCHED=static (the comparison knob, read once per process): the
    static round-robin split of both engines still moves every byte."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MP_BULK_SCHED="static")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        "tests/test_gpu_stress.py::test_back_to_back_async_transfers_bytes",
                        "tests/test_gpu_stress.py::test_bench_pattern_dedup_retire_bytes"],
                       env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_three_pools_crossing_transfers_bytes():
    """Three pools at host speed, ASYNC transfers between every ordered pair in
    random order (fan-in from two sources into one pool, opposite directions
    interleaved): coalesced batches from different sources and batches that
    read a pool another batch writes must flush in hazard order.  Every
    received block is compared with its source on the device."""
    import torch
    from paper_2406_17565_b200 import mempool as M
    from workloads.configs import LLAMA2_7B as S
    n, n_src = 512, 160
    pools = [_pool(M, torch, i, S, n, coalesce_mib=256) for i in range(3)]
    for i in range(3):
        for j in range(i + 1, 3):
            M.connect(pools[i][0], pools[j][0])
    srcs = []
    for i, (p, _r) in enumerate(pools):
        a = p.alloc_mem(n_src)
        p.debug_fill(a, 100 + i)
        srcs.append(a)
    for p, _r in pools:
        p.sync()
    rng = np.random.default_rng(9)
    for rnd in range(5):
        moves = []
        for _ in range(60):
            x = int(rng.integers(3))
            y = (x + 1 + int(rng.integers(2))) % 3
            sel = srcs[x][rng.choice(n_src, int(rng.integers(1, 8)), replace=False)]
            d = pools[x][0].transfer(y, sel, flags=M.XFER_ASYNC)
            moves.append((x, M.addr_indices(sel), y, d))
        for p, _r in pools:
            p.sync()
        for j in (0, 33, 63):
            for x in range(3):
                for y in range(3):
                    mv = [(s, d) for xx, s, yy, d in moves if xx == x and yy == y]
                    if not mv:
                        continue
                    s_ids = torch.as_tensor(np.concatenate([s for s, _ in mv]), device="cuda:0")
                    d_ids = torch.as_tensor(np.concatenate([M.addr_indices(d) for _, d in mv]),
                                            device="cuda:0")
                    bad = (pools[y][1][j, d_ids] != pools[x][1][j, s_ids]).any(dim=1)
                    assert not bool(bad.any()), f"round {rnd}: {x}->{y} chunk {j}"
        for x, _s, y, d in moves:
            pools[y][0].free_mem(d)
    for p, _r in pools:
        p.close()


@pytest.mark.parametrize("k", [1, 40, 700])   # ids inline in the launch / through id tables
def test_relay_chain_reads_what_the_previous_hop_wrote(k):
    """k blocks hop A -> B -> C -> A -> ... eleven times, every hop ASYNC and
    issued before the previous one has run, in reverse order: each migration
    starts on exactly the blocks the previous migration writes last, so it
    must not start before that grid has completed (stream order on the shared
    data stream, and griddepcontrol.wait under programmatic dependent launch;
    a blocked next grid only gets SMs as the previous one's CTAs exit, so the
    window this guards is a unit or two wide).  The last hop's blocks must
    equal the first hop's sources byte for byte."""
    import torch
    from paper_2406_17565_b200 import mempool as M
    from workloads.configs import KVShape
    S = KVShape("relay", 8, 8, 128, 16)             # 32 KiB chunks, 512 KiB blocks
    n = 4 * k
    pools = [_pool(M, torch, i, S, n) for i in range(3)]
    for i in range(3):
        for j in range(i + 1, 3):
            M.connect(pools[i][0], pools[j][0])
    first = pools[0][0].alloc_mem(k)
    pools[0][0].debug_fill(first, 4242)
    cur, at = first, 0
    order = np.arange(k)             # cur[i] holds the content of first[order[i]]
    for hop in range(11):
        nxt = (at + 1) % 3
        # reversed: the hop's first units read the blocks the previous hop wrote last
        got = pools[at][0].transfer(nxt, cur[::-1], flags=M.XFER_ASYNC)
        if hop:      # forwarded: free it while the copy may still read it (stream order)
            pools[at][0].free_mem(cur)
        cur, at, order = got, nxt, order[::-1]
    for p, _r in pools:
        p.sync()
    s_ids = torch.as_tensor(M.addr_indices(first)[order], device="cuda:0")
    d_ids = torch.as_tensor(M.addr_indices(cur), device="cuda:0")
    for j in range(2 * S.layers):
        bad = (pools[at][1][j, d_ids] != pools[0][1][j, s_ids]).any(dim=1)
        assert not bool(bad.any()), f"chunk {j}: {int(bad.sum())} blocks differ"
    for p, _r in pools:
        p.close()

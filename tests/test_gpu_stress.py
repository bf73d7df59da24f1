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


@pytest.mark.parametrize("coalesce_mib", [0, -1, 64])   # default 1 GiB, off, 64 MiB
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

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

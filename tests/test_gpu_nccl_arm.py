"""The paper's NCCL send/recv transport (comparison arm, include/mempool_nccl.h)
on one GPU through a one-rank communicator: discrete per-chunk sends (one
group per block) and the aggregated path (mp_pack -> one send ->
mp_unpack) deliver the source blocks' bytes exactly."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_nccl_discrete_and_aggregated_bytes():
    import torch
    from bench import make_pool
    from paper_2406_17565_b200 import mempool as M
    from paper_2406_17565_b200 import nccl_arm as N
    from workloads.configs import KVShape
    S = KVShape("n", 4, 4, 64, 16)                       # 8 KiB chunks, 64 KiB blocks
    nb, c, L = 64, S.chunk_bytes, S.layers
    P = make_pool(M, torch, 0, 0, S, nb)
    D = make_pool(M, torch, 1, 0, S, nb)
    pv = P._region.view(2 * L, nb, c)
    dv = D._region.view(2 * L, nb, c)
    comm = N.NcclComm.create_single(0)
    st = torch.cuda.current_stream()
    rng = np.random.default_rng(1)
    src = P.alloc_mem(24)
    P.debug_fill(src, 3)
    P.sync()
    for mode in ("discrete", "aggregated"):
        sel = src[rng.choice(len(src), 9, replace=False)]
        dst = D.alloc_mem(9)
        dv[:, torch.as_tensor(M.addr_indices(dst), device="cuda:0")] = 0
        if mode == "discrete":
            for s, d in zip(M.addr_indices(sel), M.addr_indices(dst)):
                sp = [pv.data_ptr() + (j * nb + int(s)) * c for j in range(2 * L)]
                dp = [dv.data_ptr() + (j * nb + int(d)) * c for j in range(2 * L)]
                comm.exchange(0, sp, [c] * (2 * L), 0, dp, [c] * (2 * L), st.cuda_stream)
            st.synchronize()
        else:
            stg = torch.empty(2, 9 * S.block_bytes, dtype=torch.uint8, device="cuda:0")
            P.pack(sel, 0, L, stg[0].data_ptr())
            P.sync()
            comm.exchange(0, [stg[0].data_ptr()], [9 * S.block_bytes], 0, [stg[1].data_ptr()],
                          [9 * S.block_bytes], st.cuda_stream)
            st.synchronize()
            D.unpack(stg[1].data_ptr(), dst, 0, L)
            D.sync()
        s_ids = torch.as_tensor(M.addr_indices(sel), device="cuda:0")
        d_ids = torch.as_tensor(M.addr_indices(dst), device="cuda:0")
        assert bool((pv[:, s_ids] == dv[:, d_ids]).all()), mode
        D.free_mem(dst)
    comm.close()
    P.close()
    D.close()

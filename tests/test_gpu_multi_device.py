"""Two GPUs (skipped on a one-GPU box): in-process pools on cuda:0 and cuda:1
linked with CUDA peer access -- every transport (fused NVLink peer stores,
staged cross-device slot copies, copy engine) and a DRAM-source transfer --
checked against the oracle through the twin harness."""
import pytest

import oracle as O
from paper_2406_17565_b200 import mempool as M
from tests.twin import Twin, connect, transfer, transfer_with_insert
from workloads.configs import TINY
from workloads.traces import golden_prompts

pytestmark = pytest.mark.gpu


def _two_gpus():
    import torch
    return torch.cuda.device_count() >= 2


@pytest.mark.skipif("not _two_gpus()")
@pytest.mark.parametrize("path", [M.PATH_FUSED, M.PATH_FUSED | M.XFER_ASYNC, M.PATH_STAGED,
                                  M.PATH_CE])
def test_peer_gpus_golden_and_dram_source(path):
    P = Twin(0, TINY, 64, 8, device=0)
    D = Twin(1, TINY, 64, 8, device=1)
    connect(P, D)
    S, p1, p2, p3 = golden_prompts()
    for p in (p1, p2, p3):
        _, m = P.match(p)
        new = P.alloc(-(-len(p) // 16) - len(m))
        P.fill(new)
        P.insert(p, (m + new)[: len(p) // 16])
        transfer_with_insert(P, D, p, m + new, oflags=O.FLAG_DEDUP, path=path)
    P.swap_out(2)
    _, src = P.match(p2)
    transfer(P, D, src, path=path)
    P.check_state()
    D.check_state()

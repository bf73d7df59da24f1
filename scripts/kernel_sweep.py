#!/usr/bin/env python
"""Copy-engine geometry sweep (one B200): pack (pool -> staging) and a fused
pool -> pool transfer of 128 / 256 scattered Llama-2-7B blocks, CUDA-event
kernel time from the library.  Run once per MP_BULK_CFG value (the engine
geometry is read once per process)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2406_17565_b200 import mempool as M  # noqa: E402
from workloads.configs import LLAMA2_7B as S  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]


def main(ck):
    P = M.Pool(0, 0, S.layers, S.kv_heads, S.head_dim, S.block_tokens, 1024, copy_kernel=ck,
               coalesce_mib=-1)
    D = M.Pool(1, 0, S.layers, S.kv_heads, S.head_dim, S.block_tokens, 512, copy_kernel=ck,
               coalesce_mib=-1)
    M.connect(P, D)
    src = P.alloc_mem(1024)
    for k in range(0, 1024, 256):
        P.debug_fill(src[k:k + 256], 1)
    rng = np.random.default_rng(0)
    stg = torch.empty(256 * S.block_bytes, dtype=torch.uint8, device="cuda:0")
    res = {"copy_kernel": ck, "bulk_cfg": os.environ.get("MP_BULK_CFG", "0")}
    for n in (128, 256):
        for name in ("pack", "fused"):
            for rep in range(13):
                sel = src[rng.permutation(1024)[:n]]
                if rep == 3:
                    P.stats_reset(); D.stats_reset(); P.profile(True); D.profile(True)
                if name == "pack":
                    P.pack(sel, 0, S.layers, stg.data_ptr())
                else:
                    d = P.transfer(1, sel)
                    D.free_mem(d)
            P.profile(False); D.profile(False)
            st = [x.stats() for x in (P, D)]
            ms = sum(s["kernel_ms"] for s in st) / sum(s["timed_launches"] for s in st)
            gbs = 2 * n * S.block_bytes / (ms * 1e-3) / 1e9
            res[f"{name}_{n}"] = {"kernel_ms": round(ms, 4), "hbm_rw_GBps": round(gbs, 1),
                                  "frac": round(gbs / PEAK, 4)}
    print(json.dumps(res))


if __name__ == "__main__":
    main(int(sys.argv[1]))

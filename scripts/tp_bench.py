#!/usr/bin/env python
"""TP-asymmetric repartition measured on one B200:
the KV of n Llama-2-13B blocks moves from a TP=p instance to a TP=q instance
(every shard a pool on cuda:0, loopback wire), one mp_transfer_heads per piece
of mp_tp_plan.  Each piece copies a contiguous head range of every chunk
(R16: head-major chunks), 160 KiB x k/H bytes per chunk.

Reports payload GB/s (bytes that reach the receivers / time, CUDA events
around K repetitions) and the migration kernels' HBM read+write rate against
MEASURED_PEAKS.json, for 1->2, 1->4, 2->1, 4->2 and 2->4.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import Clocks, load_peaks  # noqa: E402
from paper_2406_17565_b200 import mempool as M  # noqa: E402
from workloads.configs import LLAMA2_13B as S  # noqa: E402


def shard_pools(first_inst, t, n):
    return [M.Pool(first_inst + r, 0, S.layers, S.kv_heads // t, S.head_dim, S.block_tokens, n)
            for r in range(t)]


def run(p, q, n, reps=5):
    src = shard_pools(0, p, n)
    dst = shard_pools(100, q, n)
    for a in src:
        for b in dst:
            M.connect(a, b)
    s_addrs = [x.alloc_mem(n) for x in src]
    d_addrs = [x.alloc_mem(n) for x in dst]
    for x, a in zip(src, s_addrs):
        x.debug_fill(a, 5)
    for x in src + dst:
        x.sync()
    M.repartition(src, dst, s_addrs, d_addrs, S.kv_heads, flags=M.XFER_ASYNC)   # warm-up
    for x in src + dst:
        x.sync()
        x.stats_reset()
        x.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        M.repartition(src, dst, s_addrs, d_addrs, S.kv_heads, flags=M.XFER_ASYNC)
    for x in src + dst:
        x.sync()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    st = [x.stats() for x in src + dst]
    kms = sum(s["kernel_ms"] for s in st)
    kb = sum(s["timed_bytes"] for s in st)
    payload = reps * n * S.block_bytes
    for x in src + dst:
        x.close()
    torch.cuda.empty_cache()
    return {"p": p, "q": q, "blocks": n, "pieces": len(M.tp_plan(S.kv_heads, p, q)),
            "payload_GBps": round(payload / (ms * 1e-3) / 1e9, 1),
            "kernel_hbm_rw_GBps": round(2 * kb / (kms * 1e-3) / 1e9, 1) if kms else None,
            "launches": sum(s["timed_launches"] for s in st), "ms": round(ms, 3)}


def main():
    torch.cuda.set_device(0)
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    peak, src = load_peaks()
    clocks = Clocks("/tmp/clocks_tp.csv", 0)
    out = []
    with clocks:
        for p, q in ((1, 2), (1, 4), (2, 1), (4, 2), (2, 4), (1, 1)):
            r = run(p, q, n)
            r["frac_of_hbm_peak"] = round(r["kernel_hbm_rw_GBps"] / peak, 4)
            out.append(r)
    print(json.dumps({"what": f"TP repartition of {n} Llama-2-13B blocks on one B200 "
                              "(shards = pools on cuda:0)",
                      "peak": peak, "peak_source": src, "runs": out,
                      "clocks": clocks.summary()}))


if __name__ == "__main__":
    main()

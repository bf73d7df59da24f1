#!/usr/bin/env python
"""Short-launch efficiency of the migration kernel (VERDICT r1 "what's weak"
3: ReAct-like launches of 10-100 13B blocks).  Chains of back-to-back ASYNC
transfers of n scattered Llama-2-13B blocks (Pb = 12.5 MiB), loopback on one
B200, issued while the pools' stream is gated behind a sleeping kernel so the
CUDA events time the device back to back (not the host):

  indep   every transfer reads a fresh random subset of P's blocks into fresh
          D blocks (no block shared: consecutive grids may overlap)
  dep     ping-pong: transfer k+1 reads the blocks transfer k wrote (RAW: each
          grid waits for the previous one)

One JSON line per (mode, n): us per transfer, payload GB/s, HBM read+write
fraction of the measured copy peak.  The ring geometry (MP_BULK_CFG) and the
CTA cap (--max-ctas) are the knobs under test; run one process per setting.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import load_peaks  # noqa: E402
from paper_2406_17565_b200 import mempool as M  # noqa: E402
from workloads.configs import LLAMA2_13B  # noqa: E402

S = LLAMA2_13B
Pb = S.block_bytes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-ctas", type=int, default=0)
    ap.add_argument("--sizes", default="1,4,8,16,32,64")
    ap.add_argument("--tag", default="")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    mk = lambda inst: M.Pool(inst, 0, S.layers, S.kv_heads, S.head_dim, S.block_tokens,  # noqa
                             2600, max_ctas=args.max_ctas, coalesce_mib=-1)
    P, D = mk(0), mk(1)
    M.connect(P, D)
    peak, _ = load_peaks()
    rng = np.random.default_rng(3)
    src = P.alloc_mem(1024)
    P.debug_fill(src, 1)
    P.sync()
    side = torch.cuda.Stream()
    for mode in ("indep", "dep"):
        for n in [int(x) for x in args.sizes.split(",")]:
            reps = min(200, 1400 // n) if mode == "indep" else 100
            ms = None
            for warm in (True, False):
                P.sync()
                D.sync()
                gate = torch.cuda.Event()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(side):
                    torch.cuda._sleep(200_000_000)
                    gate.record()
                P.wait_event(gate)
                D.wait_event(gate)
                P.record_event(e0)
                k = 10 if warm else reps
                got = []
                if mode == "indep":
                    for _ in range(k):
                        s = src[rng.choice(len(src), n, replace=False)]
                        got.append(P.transfer(1, s, flags=M.XFER_ASYNC))
                else:
                    a = src[:n]
                    b = D.alloc_mem(n, stream_ordered=True)
                    pa = P.alloc_mem(n, stream_ordered=True)
                    for i in range(k):   # P:a -> D:b -> P:pa -> D:b -> ...
                        if i % 2 == 0:
                            P.transfer(1, a if i == 0 else pa, b,
                                       flags=M.XFER_ASYNC | M.XFER_DST_GIVEN)
                        else:
                            D.transfer(0, b, pa, flags=M.XFER_ASYNC | M.XFER_DST_GIVEN)
                    got = [b]
                    P.free_mem(pa)
                D.record_event(e1)
                torch.cuda.synchronize()
                if not warm:
                    ms = e0.elapsed_time(e1)
                for g in got:
                    D.free_mem(g)
                P.sync()
                D.sync()
            us = ms * 1e3 / reps
            gbs = n * Pb / (us * 1e-6) / 1e9
            print(json.dumps({"tag": args.tag, "bulk_cfg": os.environ.get("MP_BULK_CFG", "auto"),
                              "overlap": os.environ.get("MP_PDL_OVERLAP", "1"),
                              "max_ctas": args.max_ctas, "mode": mode, "n_blocks": n,
                              "us_per_transfer": round(us, 2), "GBps": round(gbs, 1),
                              "frac_hbm_rw": round(2 * gbs / peak, 4)}), flush=True)
    P.close()
    D.close()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""By-layer vs by-request vs by-request-agg on one B200 (the
analog of the paper's Fig. "block aggregation" study, §5.2
P:523-555).

A 2048-token Llama-2-7B prefill (128 blocks, 1 GiB of KV) is emulated
per layer on an engine stream: a bf16 GEMM with the layer's prefill FLOPs
(2 * 2048 * (4 * 4096^2 + 3 * 4096 * 11008) = 0.83 TFLOP) followed by the
layer's KV write into the prefill pool.  The KV then moves to the decode pool
(loopback on one GPU) in one of five ways:

  compute_only        no transfer (reference time)
  by_request_agg      after the last layer: one fused transfer of all layers
  by_layer_agg        after each layer: a fused transfer of that layer (A10,
                      caller-given destination blocks, ordered after the
                      layer's event with mp_wait_event)
  by_request_discrete after the last layer: one copy-engine memcpy per
                      (block, layer, K/V) chunk -- the paper's discrete layout
                      with one network call per block
  by_layer_discrete   per layer, one memcpy per (block, K/V) chunk of the layer

Reported: time from prefill start to KV landed at D; `after_compute_ms`, the
time the KV is still moving after the last layer's compute ended (the
transfer's share of time-to-second-token); the difference to
compute_only (includes run-to-run clock variation of the GEMMs); the number of
API calls / copies issued; for 1 request (low load) and for R back-to-back
requests (transfers of request i overlap the compute of request i+1).
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2406_17565_b200 import mempool as M  # noqa: E402
from workloads.configs import LLAMA2_7B  # noqa: E402

S = LLAMA2_7B
NB = 128            # blocks of one 2048-token prompt
TOK = 2048
LAYER_N = int(2 * TOK * (4 * 4096 ** 2 + 3 * 4096 * 11008) / (2 * TOK * 4096))  # GEMM N


def make_pool(inst, n):
    c = S.chunk_bytes
    region = torch.zeros(2 * S.layers * n * c, dtype=torch.uint8, device="cuda:0")
    slabs = [region.data_ptr() + j * n * c for j in range(2 * S.layers)]
    p = M.Pool(inst, 0, S.layers, S.kv_heads, S.head_dim, S.block_tokens, n, slabs=slabs,
               staging_bytes=64 << 20)
    return p, region.view(2 * S.layers, n, c)


def run(mode, R, P, pr, D, engine, a, w):
    srcs = [P.alloc_mem(NB) for _ in range(R)]
    dsts = [D.alloc_mem(NB) for _ in range(R)]
    sidx = [torch.as_tensor(M.addr_indices(s), device="cuda:0") for s in srcs]
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    landed = torch.cuda.Event()
    t0.record(engine)
    calls = 0
    for r in range(R):
        for layer in range(S.layers):
            with torch.cuda.stream(engine):
                torch.matmul(a, w)                                  # the layer's compute
                pr[2 * layer: 2 * layer + 2, sidx[r]] = (layer + 1) & 0xFF  # its KV write
            if mode in ("by_layer_agg", "by_layer_discrete"):
                ev = torch.cuda.Event()
                ev.record(engine)
                P.wait_event(ev)
                path = M.PATH_FUSED if mode == "by_layer_agg" else M.PATH_CE
                P.transfer(1, srcs[r], dsts[r], layer_begin=layer, layer_end=layer + 1,
                           flags=path | M.XFER_ASYNC)
                calls += 1 if mode == "by_layer_agg" else 2 * NB
        if mode in ("by_request_agg", "by_request_discrete"):
            ev = torch.cuda.Event()
            ev.record(engine)
            P.wait_event(ev)
            path = M.PATH_FUSED if mode == "by_request_agg" else M.PATH_CE
            P.transfer(1, srcs[r], dsts[r], flags=path | M.XFER_ASYNC)
            calls += 1 if mode == "by_request_agg" else 2 * S.layers * NB
    tc = torch.cuda.Event(enable_timing=True)
    tc.record(engine)                      # compute (and KV writes) done
    D.record_event(landed)
    engine.wait_event(landed)
    t1.record(engine)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    tail_ms = tc.elapsed_time(t1)          # KV still moving after the compute ended
    P.sync()
    D.sync()                               # collects the library's kernel timings
    st = [x.stats() for x in (P, D)]
    kernel_ms = sum(s["kernel_ms"] for s in st)
    for x in (P, D):
        x.stats_reset()
    # check the last request's KV landed
    dst_idx = torch.as_tensor(M.addr_indices(dsts[-1]), device="cuda:0")
    ok = True
    if mode != "compute_only":
        got = D._view[:, dst_idx, :8].cpu().numpy()
        ok = all((got[j] == ((j // 2 + 1) & 0xFF)).all() for j in range(2 * S.layers))
    for s in srcs:
        P.free_mem(s)
    for d in dsts:
        D.free_mem(d)
    return ms, calls, ok, tail_ms, kernel_ms


def main():
    torch.cuda.set_device(0)
    P, pr = make_pool(0, 8 * NB + 8)
    D, dr = make_pool(1, 8 * NB + 8)
    D._view = dr
    M.connect(P, D)
    P.profile(True)
    D.profile(True)
    engine = torch.cuda.Stream()
    a = torch.randn(TOK, 4096, dtype=torch.bfloat16, device="cuda:0")
    w = torch.randn(4096, LAYER_N, dtype=torch.bfloat16, device="cuda:0")
    out = {"workload": f"Llama-2-7B, {TOK}-token prompt ({NB} blocks, 1 GiB KV), per-layer "
                       f"bf16 GEMM {TOK}x4096x{LAYER_N} as the layer's prefill compute, "
                       "loopback P->D on one B200", "results": []}
    modes = ["compute_only", "by_request_agg", "by_layer_agg", "by_request_discrete",
             "by_layer_discrete"]
    for R in (1, 4):
        base = None
        for mode in modes:
            run(mode, 1, P, pr, D, engine, a, w)           # warm-up
            ms, calls, ok, tail_ms, kernel_ms = run(mode, R, P, pr, D, engine, a, w)
            if mode == "compute_only":
                base = ms
            row = {"requests": R, "mode": mode, "ms": round(ms, 3),
                   "exposed_transfer_ms": round(ms - base, 3),
                   "after_compute_ms": round(tail_ms, 3),
                   "migration_kernel_ms": round(kernel_ms, 3), "api_or_copy_calls": calls,
                   "kv_landed_ok": bool(ok)}
            out["results"].append(row)
            print(json.dumps(row), file=sys.stderr)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

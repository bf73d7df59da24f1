#!/usr/bin/env python
"""Size sweeps on one B200:

  transfer  configs[1]'s fixed sweep: raw P->D transfer of n scattered 7B
            blocks, n in {1, 2, 4, ..., 256} (named point n = 128 = a 2048-token
            prompt), for each transport (fused vector / fused bulk /
            staged / copy-engine per chunk = the paper's discrete per-block
            transfer).  Loopback on one GPU: HBM-bound.
  swap      configs[4]: swap_out(n) then swap_in of the moved blocks,
            n in {1, 2, 4, ..., 4096}, 7B pool of 8192 HBM blocks (64 GiB) and
            4096 pinned DRAM blocks (32 GiB), plus the pinned-memcpy peak.

  dram_source  SURVEY f1: transfer of swapped-out blocks straight from the
            sender's pinned DRAM vs swap_in + HBM transfer.

Usage: python scripts/sweeps.py {transfer|swap|api|dram_source} > out.json
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2406_17565_b200 import mempool as M  # noqa: E402
from workloads.configs import LLAMA2_7B, seed_for  # noqa: E402

SHAPE = LLAMA2_7B
Pb = SHAPE.block_bytes


def pool(inst, n, **kw):
    return M.Pool(inst, 0, SHAPE.layers, SHAPE.kv_heads, SHAPE.head_dim, SHAPE.block_tokens,
                  n, **kw)


def transfer_sweep():
    out = {"workload": "raw transfer of n scattered Llama-2-7B blocks (Pb = 8 MiB), "
                       "loopback on one B200; payload GB/s; each repetition uses a fresh "
                       "random source subset (working set >> L2 for n >= 16)",
           "results": []}
    seed = seed_for(1)
    engines = [("fused_vector", M.PATH_FUSED, 1), ("fused_bulk", M.PATH_FUSED, 2),
               ("staged_bulk", M.PATH_STAGED, 2), ("ce_per_chunk", M.PATH_CE, 1)]
    for name, path, ck in engines:
        P = pool(0, 2048, copy_kernel=ck, coalesce_mib=-1, staging_bytes=1 << 30)
        D = pool(1, 1024, copy_kernel=ck, coalesce_mib=-1, staging_bytes=1 << 30)
        M.connect(P, D)
        src = P.alloc_mem(2048)
        for k in range(0, 2048, 256):
            P.debug_fill(src[k:k + 256], seed)
        rng = np.random.default_rng(seed)
        for n in (1, 2, 4, 8, 16, 32, 64, 128, 256):
            reps = 3 if path == M.PATH_CE and n >= 64 else 10
            for _ in range(2):   # warm-up
                d = P.transfer(1, src[rng.permutation(2048)[:n]], flags=path)
                D.free_mem(d)
            P.stats_reset()
            D.stats_reset()
            P.profile(True)
            D.profile(True)
            t = 0.0
            for _ in range(reps):
                sel = src[rng.permutation(2048)[:n]]
                t0 = time.perf_counter()
                d = P.transfer(1, sel, flags=path)
                t += time.perf_counter() - t0
                D.free_mem(d)
            P.profile(False)
            D.profile(False)
            st = [x.stats() for x in (P, D)]
            kms = sum(s["kernel_ms"] for s in st)
            kl = sum(s["timed_launches"] for s in st)
            row = {"engine": name, "n_blocks": n, "bytes": n * Pb,
                   "call_GBps": round(n * Pb * reps / t / 1e9, 2),
                   "call_us": round(t / reps * 1e6, 1),
                   "blocks_per_s": round(n * reps / t, 1)}
            if kl:
                row["kernel_ms_per_call"] = round(kms / reps, 4)
                row["kernels_per_call"] = kl / reps
            out["results"].append(row)
            print(json.dumps(row), file=sys.stderr)
        P.close()
        D.close()
    # PyTorch library baseline: the same gather/scatter as advanced indexing on
    # [2L, N, c] byte tensors (index_select + index_copy kernels)
    c = SHAPE.chunk_bytes
    src_t = torch.empty(2 * SHAPE.layers, 2048, c, dtype=torch.uint8, device="cuda:0")
    dst_t = torch.empty(2 * SHAPE.layers, 1024, c, dtype=torch.uint8, device="cuda:0")
    rng = np.random.default_rng(seed)
    for n in (1, 2, 4, 8, 16, 32, 64, 128, 256):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        for _ in range(2):
            dst_t[:, torch.arange(n, device="cuda:0")] = src_t[:, torch.as_tensor(
                rng.permutation(2048)[:n], device="cuda:0")]
        torch.cuda.synchronize()
        reps = 10
        sels = [torch.as_tensor(rng.permutation(2048)[:n], device="cuda:0") for _ in range(reps)]
        dsel = [torch.as_tensor(rng.permutation(1024)[:n], device="cuda:0") for _ in range(reps)]
        ev[0].record()
        for r in range(reps):
            dst_t[:, dsel[r]] = src_t[:, sels[r]]
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / reps
        row = {"engine": "torch_advanced_indexing", "n_blocks": n, "bytes": n * Pb,
               "call_GBps": round(n * Pb / (ms * 1e-3) / 1e9, 2), "call_us": round(ms * 1e3, 1),
               "blocks_per_s": round(n / (ms * 1e-3), 1), "kernel_ms_per_call": round(ms, 4)}
        out["results"].append(row)
        print(json.dumps(row), file=sys.stderr)
    return out


def sm_budget_sweep():
    """How many SMs a migration needs for a given rate: 128 scattered 7B blocks
    (1 GiB payload) per launch, loopback, with the grid capped at max_ctas
    CTAs (the block scheduler spreads small grids one CTA per SM).  Payload
    GB/s over the launch's own CUDA-event time.  The NVLink question (DESIGN
    §10: how few SMs still saturate ~775 GB/s per direction) is read off the
    per-CTA rate while the copy is far from HBM-bound."""
    seed = seed_for(1)
    out = {"workload": "128 scattered Llama-2-7B blocks (1 GiB payload) per fused transfer, "
                       "loopback on one B200, grid capped at max_ctas", "results": []}
    for name, ck in (("vector", 1), ("bulk", 2)):
        for cap in (4, 8, 16, 24, 32, 48, 64, 96, 148, 0):
            P = pool(0, 1024, copy_kernel=ck, coalesce_mib=-1, max_ctas=cap)
            D = pool(1, 1024, copy_kernel=ck, coalesce_mib=-1, max_ctas=cap)
            M.connect(P, D)
            src = P.alloc_mem(1024)
            rng = np.random.default_rng(seed)
            for _ in range(2):
                D.free_mem(P.transfer(1, src[rng.permutation(1024)[:128]]))
            for x in (P, D):
                x.stats_reset()
                x.profile(True)
            reps = 5
            for _ in range(reps):
                D.free_mem(P.transfer(1, src[rng.permutation(1024)[:128]]))
            for x in (P, D):
                x.profile(False)
            st = [x.stats() for x in (P, D)]
            kms = sum(t["kernel_ms"] for t in st) / max(1, sum(t["timed_launches"] for t in st))
            gbs = 128 * Pb / (kms * 1e-3) / 1e9
            row = {"engine": name, "max_ctas": cap or "full wave", "kernel_ms": round(kms, 4),
                   "payload_GBps": round(gbs, 1),
                   "payload_GBps_per_cta": round(gbs / cap, 1) if cap else None}
            out["results"].append(row)
            print(json.dumps(row), file=sys.stderr)
            P.close()
            D.close()
    return out


def swap_sweep():
    seed = seed_for(4)
    B = SHAPE.block_tokens
    n_hbm, n_dram = 8192, 4096
    t0 = time.perf_counter()
    S = pool(0, n_hbm, dram_blocks=n_dram)
    pin_s = time.perf_counter() - t0
    rng = np.random.default_rng(seed)
    base = [rng.integers(3, 32000, size=40 * B, dtype=np.int32) for _ in range(8)]
    seqs = []
    for i in range(96):   # 96 historical sequences of 48-80 blocks, shared prefixes
        pre = base[i % 8][: int(rng.integers(0, 41)) * B]
        tail = rng.integers(3, 32000, size=int(rng.integers(48, 81)) * B - len(pre),
                            dtype=np.int32)
        t = np.concatenate([pre, tail]).astype(np.int32)
        _, matched = S.match(t)
        new = S.alloc_mem(len(t) // B - len(matched))
        S.debug_fill(new, seed)
        S.insert(t, np.concatenate([matched, new]))
        seqs.append(t)
    info = S.info()
    # pinned-memcpy peak (torch), the host-link reference
    a = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:0")
    h = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    for _ in range(2):
        h.copy_(a)
        a.copy_(h)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    h.copy_(a, non_blocking=True)
    ev[1].record()
    a.copy_(h, non_blocking=True)
    ev[2].record()
    torch.cuda.synchronize()
    d2h = (1 << 30) / (ev[0].elapsed_time(ev[1]) * 1e-3) / 1e9
    h2d = (1 << 30) / (ev[1].elapsed_time(ev[2]) * 1e-3) / 1e9
    del a, h
    out = {"workload": "configs[4]: Llama-2-7B pool, 8192 HBM + 4096 pinned DRAM blocks, "
                       f"96 historical sequences ({info.index_blocks} indexed blocks)",
           "pinned_alloc_s": round(pin_s, 2),
           "pcie_memcpy_GBps": {"d2h": round(d2h, 2), "h2d": round(h2d, 2)},
           "results": []}
    for mode, flags in (("zero_copy", M.SWAP_ZERO_COPY), ("ce_staged", M.SWAP_CE)):
        for n in (1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096):
            # small calls are latency-sized: the median of several round
            # trips (the first also pays one-time costs, reported apart)
            reps = 7 if n <= 64 else 1
            tout, tin = [], []
            for _ in range(reps):
                t0 = time.perf_counter()
                old, new = S.swap_out(n, flags)
                t1 = time.perf_counter()
                back = S.swap_in(new, flags)
                t2 = time.perf_counter()
                tout.append(t1 - t0)
                tin.append(t2 - t1)
            to, ti = float(np.median(tout)), float(np.median(tin))
            row = {"mode": mode, "n": n, "moved": len(old), "bytes": len(old) * Pb,
                   "swap_out_GBps": round(len(old) * Pb / to / 1e9, 2),
                   "swap_in_GBps": round(len(back) * Pb / ti / 1e9, 2),
                   "swap_out_ms": round(to * 1e3, 3),
                   "swap_in_ms": round(ti * 1e3, 3), "reps": reps,
                   "first_call_ms": [round(tout[0] * 1e3, 3), round(tin[0] * 1e3, 3)]}
            out["results"].append(row)
            print(json.dumps(row), file=sys.stderr)
    S.close()
    return out


def dram_source_sweep():
    """SURVEY f1 (memory asymmetry): historical KV swapped out to the
    sender's pinned DRAM goes straight into the receiver's HBM (copy engine
    into the sender's staging + a scatter per slot, or one kernel reading
    mapped host memory), vs the two-step alternative swap_in + HBM transfer.
    Payload GB/s, synchronous calls, loopback receiver."""
    seed = seed_for(4)
    P = pool(0, 1024, dram_blocks=1024)
    D = pool(1, 1024)
    M.connect(P, D)
    a = P.alloc_mem(768)
    P.debug_fill(a, seed)
    toks = (np.arange(768 * SHAPE.block_tokens, dtype=np.int64) % 31000 + 3).astype(np.int32)
    P.insert(toks, a)
    _old, dram = P.swap_out(512)
    rng = np.random.default_rng(seed)
    out = {"workload": "Llama-2-7B blocks (8 MiB) in the sender's pinned DRAM -> receiver "
                       "HBM on one B200, synchronous calls", "results": []}
    # direct (the DRAM blocks stay where they are): the default copy-engine
    # path (H2D into the sender's staging, scattered per slot) and the
    # zero-copy kernel reading mapped DRAM (MP_DRAM_SOURCE=sm)
    for mode in ("ce", "sm"):
        os.environ["MP_DRAM_SOURCE"] = mode
        for n in (1, 16, 128, 256):
            best = None
            for _ in range(3):
                sel = dram[np.sort(rng.permutation(len(dram))[:n])]
                t0 = time.perf_counter()
                d = P.transfer(1, sel)
                t1 = time.perf_counter()
                D.free_mem(d)
                best = t1 - t0 if best is None else min(best, t1 - t0)
            out["results"].append({"mode": f"direct_dram_to_peer_hbm_{mode}", "n": n,
                                   "GBps": round(n * Pb / best / 1e9, 2),
                                   "ms": round(best * 1e3, 3)})
            print(json.dumps(out["results"][-1]), file=sys.stderr)
    os.environ.pop("MP_DRAM_SOURCE")
    fresh = list(dram)           # the two-step mode consumes DRAM blocks (swap_in frees them)
    for n in (1, 16, 128, 256):
        sel, fresh = np.array(fresh[:n], np.uint64), fresh[n:]
        t0 = time.perf_counter()
        hb = P.swap_in(sel)
        d = P.transfer(1, hb)
        t1 = time.perf_counter()
        D.free_mem(d)
        out["results"].append({"mode": "swap_in_then_hbm_transfer", "n": n,
                               "GBps": round(n * Pb / (t1 - t0) / 1e9, 2),
                               "ms": round((t1 - t0) * 1e3, 3)})
        print(json.dumps(out["results"][-1]), file=sys.stderr)
    P.close()
    D.close()
    return out


def gs_latency():
    """global prompt trees, host-only.  8 instances
    (4 prefill, 4 decode), ShareGPT-like sessions: every turn routes its
    prompt to a prefill instance and the chosen instance's tree is updated
    (P:645); per-call host time vs the number of prompts held."""
    from workloads import traces
    gs = M.GlobalScheduler(16, 3600.0)
    for i in range(8):
        gs.register(i, gs.PREFILL if i < 4 else gs.DECODE)
    sessions = traces.sharegpt_like(seed_for(1), n_sessions=3000)
    prompts = [t.prompt for s_ in sessions for t in s_.turns]
    out = {"workload": "global scheduler: 8 instances, ShareGPT-like prompts (route to a "
                       "prefill instance, then update its tree)", "results": []}
    now, done, t_route, t_upd = 0.0, 0, 0.0, 0.0
    marks = {500, 2000, 5000, len(prompts)}
    for p_ in prompts:
        now += 0.001
        t0 = time.perf_counter()
        inst, mt, extra = gs.route(gs.PREFILL, p_, now)
        t1 = time.perf_counter()
        gs.update(inst, p_, now)
        gs.update(4 + inst, p_, now)          # its decode partner holds it too
        t2 = time.perf_counter()
        t_route += t1 - t0
        t_upd += (t2 - t1) / 2
        done += 1
        if done in marks:
            out["results"].append({"prompts_seen": done,
                                   "route_us": round(t_route / done * 1e6, 2),
                                   "update_us": round(t_upd / done * 1e6, 2),
                                   "avg_prompt_tokens": int(np.mean([len(x) for x in
                                                                     prompts[:done]]))})
            print(json.dumps(out["results"][-1]), file=sys.stderr)
    gs.close()
    return out


def api_latency():
    """The paper's MemPool API study: memory-API latency vs block
    count ("~800 ns per block, linear") and index insert / match of a 4K-token
    prompt ("<= 0.7 ms", flat in the cached ratio).  Host clock, per call."""
    import time as _t
    out = {"workload": "Llama-2-7B pool of 8192 blocks on one B200; per-call host time",
           "alloc_free": [], "index": []}
    P = pool(0, 8192)
    for so in (False, True):            # drained (default) / MP_ALLOC_STREAM_ORDERED
        for n in (1, 16, 64, 256, 1024, 4096):
            reps, warm = 20, 3
            ta = tf = 0.0
            for r in range(warm + reps):
                t0 = _t.perf_counter()
                a = P.alloc_mem(n, stream_ordered=so)
                t1 = _t.perf_counter()
                P.free_mem(a)
                t2 = _t.perf_counter()
                if r >= warm:
                    ta += t1 - t0
                    tf += t2 - t1
            out["alloc_free"].append({"blocks": n, "stream_ordered": so,
                                      "alloc_us": round(ta / reps * 1e6, 2),
                                      "free_us": round(tf / reps * 1e6, 2),
                                      "alloc_ns_per_block": round(ta / reps / n * 1e9, 1)})
    rng = np.random.default_rng(0)
    B = SHAPE.block_tokens
    base = rng.integers(3, 32000, size=4096, dtype=np.int32)       # 256 blocks
    for cached in (0.0, 0.25, 0.5, 0.75, 1.0):
        k = int(256 * cached)
        ti = tm = 0.0
        reps = 10
        for r in range(reps):
            prompt = np.concatenate([base[: k * B],
                                     rng.integers(3, 32000, size=4096 - k * B, dtype=np.int32)])
            if k:
                _, m = P.match(base[: k * B])
                if len(m) < k:
                    a = P.alloc_mem(k - len(m))
                    P.insert(base[: k * B], np.concatenate([m, a]))
            t0 = _t.perf_counter()
            mt, m = P.match(prompt)
            t1 = _t.perf_counter()
            new = P.alloc_mem(256 - len(m))
            t2 = _t.perf_counter()
            P.insert(prompt, np.concatenate([m, new]))
            t3 = _t.perf_counter()
            tm += t1 - t0
            ti += t3 - t2
            P.delete(prompt)
        out["index"].append({"prompt_tokens": 4096, "cached_ratio": cached,
                             "match_us": round(tm / reps * 1e6, 1),
                             "insert_us": round(ti / reps * 1e6, 1)})
    P.close()
    return out


def chain_sweep():
    """Back-to-back ASYNC transfers of n scattered blocks (no sync between
    them): device time per transfer from CUDA events around the whole chain.
    Run once with MP_PDL=1 and once with MP_PDL=0 to see what programmatic
    dependent launch hides between consecutive migration kernels."""
    import torch
    out = {"workload": "chains of up to 400 back-to-back ASYNC mp_transfer calls of n scattered "
                       "Llama-2-7B blocks, loopback, one B200",
           "pdl": os.environ.get("MP_PDL", "1") != "0", "rows": []}
    # one launch per transfer (no coalescing); the pools' stream is gated
    # behind a sleeping kernel while the host issues the whole chain, so the
    # events time the device back to back, not the host's issue rate
    P, D = pool(0, 4096, coalesce_mib=-1), pool(1, 4096, coalesce_mib=-1)
    M.connect(P, D)
    rng = np.random.default_rng(3)
    src = P.alloc_mem(2048)
    P.debug_fill(src, 1)
    P.sync()
    side = torch.cuda.Stream()
    for n in (1, 2, 4, 8, 16, 64):
        reps = min(400, 3800 // n)       # every destination stays allocated until the end
        sels = [src[rng.choice(len(src), n, replace=False)] for _ in range(reps)]
        for warm in (True, False):
            P.sync()
            D.sync()
            gate = torch.cuda.Event()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(side):
                torch.cuda._sleep(200_000_000)       # ~0.1 s: longer than issuing the chain
                gate.record()
            P.wait_event(gate)
            P.record_event(e0)
            got = []
            for s in sels[: 20 if warm else reps]:
                got.append(P.transfer(1, s, flags=M.XFER_ASYNC))
            D.record_event(e1)
            torch.cuda.synchronize()
            if not warm:
                ms = e0.elapsed_time(e1)
            for g in got:
                D.free_mem(g)
        out["rows"].append({"n_blocks": n, "us_per_transfer": round(ms * 1e3 / reps, 2),
                            "GBps": round(n * Pb * reps / (ms * 1e-3) / 1e9, 1)})
    P.close()
    D.close()
    return out


def nccl_sweep():
    """The paper's transport (NCCL send/recv) beside the
    fused one-sided kernel, on one B200 through a one-rank communicator (NCCL's
    self send/recv = its local copy path), n scattered Llama-2-7B blocks:
      nccl_discrete_per_block  one NCCL group per block of 2L chunk sends (the
                               paper's discrete layout, one call per block)
      nccl_discrete_grouped    all n * 2L chunk sends in one group
      nccl_aggregated          mp_pack -> one send of n * Pb -> mp_unpack
                               (the paper's aggregation)
      fused                    mp_transfer (the product path)
    Host clock per synchronous transfer; destination bytes checked against
    the source on the device after every mode."""
    import time as _t
    import torch
    from bench import make_pool
    from paper_2406_17565_b200 import nccl_arm as N
    S = SHAPE
    nb = 1024
    P = make_pool(M, torch, 0, 0, S, nb)
    D = make_pool(M, torch, 1, 0, S, nb)
    M.connect(P, D)
    c, L = S.chunk_bytes, S.layers
    pv = P._region.view(2 * L, nb, c)
    dv = D._region.view(2 * L, nb, c)
    comm = N.NcclComm.create_single(0)
    stream = torch.cuda.current_stream()
    rng = np.random.default_rng(7)
    src_all = P.alloc_mem(512)
    P.debug_fill(src_all, 11)
    P.sync()
    stg = torch.empty(2, 256 * Pb, dtype=torch.uint8, device="cuda:0")
    out = {"workload": "n scattered Llama-2-7B blocks (Pb = 8 MiB) P -> D on one B200; NCCL "
                       f"{N.version()} one-rank communicator (self send/recv)", "rows": []}

    def chunk_ptrs(view, ids):
        base = view.data_ptr()
        return [base + (j * nb + int(b)) * c for b in ids for j in range(2 * L)]

    def check(src, dst):
        s = torch.as_tensor(M.addr_indices(src), device="cuda:0")
        d = torch.as_tensor(M.addr_indices(dst), device="cuda:0")
        for j in (0, 2 * L - 1):
            assert bool((pv[j, s] == dv[j, d]).all()), "bytes differ"

    for n in (1, 16, 128, 256):
        row = {"n_blocks": n}
        for mode in ("nccl_discrete_per_block", "nccl_discrete_grouped", "nccl_aggregated",
                     "fused"):
            reps = 5 if n >= 128 or mode != "nccl_discrete_per_block" else 3
            ts = []
            for r in range(reps + 1):
                src = src_all[rng.choice(len(src_all), n, replace=False)]
                dst = D.alloc_mem(n)
                dv[:, torch.as_tensor(M.addr_indices(dst), device="cuda:0")] = 0
                torch.cuda.synchronize()
                t0 = _t.perf_counter()
                if mode == "fused":      # the receiver allocates inside the call
                    D.free_mem(dst)
                    dst = P.transfer(1, src)
                elif mode == "nccl_aggregated":
                    P.pack(src, 0, L, stg[0].data_ptr())
                    P.sync()
                    comm.exchange(0, [stg[0].data_ptr()], [n * Pb], 0, [stg[1].data_ptr()],
                                  [n * Pb], stream.cuda_stream)
                    stream.synchronize()
                    D.unpack(stg[1].data_ptr(), dst, 0, L)
                    D.sync()
                else:
                    sp, dp = chunk_ptrs(pv, M.addr_indices(src)), chunk_ptrs(dv, M.addr_indices(dst))
                    step = 2 * L if mode == "nccl_discrete_per_block" else len(sp)
                    for k in range(0, len(sp), step):
                        comm.exchange(0, sp[k:k + step], [c] * step, 0, dp[k:k + step],
                                      [c] * step, stream.cuda_stream)
                    stream.synchronize()
                dt = _t.perf_counter() - t0
                check(src, dst)
                D.free_mem(dst)
                if r:
                    ts.append(dt)
            ms = float(np.median(ts)) * 1e3
            row[mode] = {"ms": round(ms, 3), "GBps": round(n * Pb / (ms * 1e-3) / 1e9, 1),
                         "calls": (n if mode == "nccl_discrete_per_block" else 1)}
        out["rows"].append(row)
        print(row, file=sys.stderr)
    comm.close()
    P.close()
    D.close()
    return out


def tiny_latency():
    """BASELINE configs[0] (tiny pool: L2 H2 D64 fp16, B16, 64 blocks per
    instance) is latency-bound, not roofline-graded: host
    µs per call of the golden run's operations, p10 / p50 / p90 over 300
    rounds of the three prompts (each round deletes them again)."""
    from workloads.configs import TINY as T
    from workloads.traces import golden_prompts
    import time as _t
    P = M.Pool(0, 0, T.layers, T.kv_heads, T.head_dim, T.block_tokens, 64)
    D = M.Pool(1, 0, T.layers, T.kv_heads, T.head_dim, T.block_tokens, 64)
    M.connect(P, D)
    _, p1, p2, p3 = golden_prompts()
    B = T.block_tokens
    acc = {k: [] for k in ("match", "alloc_mem", "insert", "twi_dedup_sync", "twi_dedup_async",
                           "free_mem", "delete")}
    for rnd in range(320):
        keep = rnd >= 20
        flags = M.XFER_DEDUP | (M.XFER_ASYNC if rnd % 2 else 0)
        parts = []
        for p in (p1, p2, p3):
            t0 = _t.perf_counter()
            _, m = P.match(p)
            t1 = _t.perf_counter()
            new = P.alloc_mem(-(-len(p) // B) - len(m), stream_ordered=True)
            t2 = _t.perf_counter()
            full = np.concatenate([m, new])
            t3 = _t.perf_counter()
            P.insert(p, full[: len(p) // B])
            t4 = _t.perf_counter()
            fin, _ = P.transfer_with_insert(1, p, full, flags=flags)
            t5 = _t.perf_counter()
            if keep:
                acc["match"].append(t1 - t0)
                acc["alloc_mem"].append(t2 - t1)
                acc["insert"].append(t4 - t3)
                acc["twi_dedup_async" if flags & M.XFER_ASYNC else "twi_dedup_sync"].append(t5 - t4)
            parts.append((p, full[len(p) // B:], fin[len(p) // B:]))
        for p, pp, dp in parts:
            t0 = _t.perf_counter()
            P.free_mem(pp)
            t1 = _t.perf_counter()
            P.delete(p)
            t2 = _t.perf_counter()
            D.free_mem(dp)
            D.delete(p)
            if keep:
                acc["free_mem"].append(t1 - t0)
                acc["delete"].append(t2 - t1)
    P.sync()
    D.sync()
    P.close()
    D.close()
    return {"workload": "configs[0] tiny pools (16 KiB blocks), golden prompts p1-p3, P->D DEDUP "
                        "transfer_with_insert, host clock per call through the Python binding",
            "us_p10_p50_p90": {k: [round(float(np.percentile(v, q)) * 1e6, 2) for q in (10, 50, 90)]
                               for k, v in acc.items()}}


if __name__ == "__main__":
    fn = {"transfer": transfer_sweep, "swap": swap_sweep, "api": api_latency,
          "dram_source": dram_source_sweep, "gs": gs_latency, "chain": chain_sweep,
          "tiny": tiny_latency, "nccl": nccl_sweep, "sms": sm_budget_sweep}[sys.argv[1]]
    print(json.dumps(fn(), indent=1))

#!/usr/bin/env python
"""bench.py -- KV migration GB/s & blocks/s vs the HBM / NVLink roofline.

BASELINE.json metric: "KV migration GB/s & blocks/s vs HBM/NVLink roofline at
1/2/4/8 B200".  Workload (N=1): configs[1], Llama-2-7B-shaped KV (L=32, H=32,
D=128, fp16, B=16 -> Pb = 8 MiB per token block), ShareGPT-like prompts,
1P1D.  On one GPU the prefill (P) and decode (D) instances are two pools on
cuda:0 and the "wire" is a device-local copy.

One STEP = one pass of the migration hot path over one batch of requests
(PD-Caching-2, §5.1):
    for each request: P.match(prompt)                          (A3)
                      P.transfer_with_insert(D, prompt, src, DEDUP)
                        -> D: match, alloc (A2), gather->store (A6f), insert (A7)
    then D retires the batch: free_mem(partial blocks) + delete(prompts).
value = payload bytes actually moved (blocks moved x Pb) / step time.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Under torchrun (N>1) every rank runs its own P/D pair (weak scaling).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads.configs import LLAMA2_7B, seed_for  # noqa: E402
from workloads import traces  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0   # B200_PROFILING.md fallback
NVLINK_GBS = 900.0          # nominal per direction per GPU (BJ:5)


def load_peaks():
    try:
        with open(PEAKS_PATH) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: copy read+write)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------- workload
def build_requests(shape, seed, hbm_blocks, fill_budget):
    """ShareGPT-like sessions until `fill_budget` blocks."""
    B = shape.block_tokens
    sessions = traces.sharegpt_like(seed, n_sessions=4096)
    reqs, used = [], 0
    for s in sessions:
        blocks = -(-len(s.turns[-1].prompt) // B) + len(s.turns)
        if used + blocks > fill_budget:
            if used > 0.95 * fill_budget:
                break
            continue
        used += blocks
        for t in s.turns:
            reqs.append((s.sid, t.prompt))
    return reqs


class Clocks:
    """nvidia-smi sampler running DURING the timed region."""

    def __init__(self, path, device):
        self.path = path
        self.p = None
        self.device = device

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            self.p.wait()
            self.f.close()

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            rows = [ln.split(",") for ln in open(self.path) if ln.strip()]
            sm = [float(r[0]) for r in rows]
            mx = max(float(r[1]) for r in rows)
            reasons = sorted({names[i] for r in rows for i in range(4)
                              if r[3 + i].strip().lower() == "active"})
            return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": reasons,
                    "samples": len(rows)}
        except Exception as e:  # no nvidia-smi: say so
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": str(e)}


def make_pool(M, torch, inst, dev, shape, n_blocks, **kw):
    """HBM slabs are torch allocations (PyTorch owns device memory)."""
    c = shape.chunk_bytes
    region = torch.empty(2 * shape.layers * n_blocks * c, dtype=torch.uint8, device=f"cuda:{dev}")
    slabs = [region.data_ptr() + j * n_blocks * c for j in range(2 * shape.layers)]
    p = M.Pool(inst, dev, shape.layers, shape.kv_heads, shape.head_dim, shape.block_tokens,
               n_blocks, slabs=slabs, **kw)
    p._region = region
    return p


def run_ours(args, rank, world, dist):
    import torch
    from paper_2406_17565_b200 import mempool as M

    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    shape = LLAMA2_7B
    B, Pb = shape.block_tokens, shape.block_bytes
    seed = seed_for(1) + 1000 * rank
    n_blocks = args.pool_blocks
    P = make_pool(M, torch, 2 * rank, dev, shape, n_blocks, copy_kernel=args.copy_kernel)
    D = make_pool(M, torch, 2 * rank + 1, dev, shape, n_blocks, copy_kernel=args.copy_kernel)
    M.connect(P, D)

    # ---- untimed setup: the prefill instance's cache (PD-Caching-1 step 2)
    reqs = build_requests(shape, seed, n_blocks, int(n_blocks * 0.9))
    req_src = []
    for sid, prompt in reqs:
        mt, matched = P.match(prompt)
        new = P.alloc_mem(-(-len(prompt) // B) - len(matched))
        P.debug_fill(new, seed)
        full = np.concatenate([matched, new])
        P.insert(prompt, full[: len(prompt) // B])
        partial = full[len(prompt) // B:]       # trailing partial block (active)
        req_src.append((prompt, partial))
    # batches of whole sessions, each about batch_blocks blocks
    batches, cur, cur_blocks = [], [], 0
    last_sid = None
    for (sid, prompt), (_, partial) in zip(reqs, req_src):
        if sid != last_sid and cur_blocks >= args.batch_blocks:
            batches.append(cur)
            cur, cur_blocks = [], 0
        cur.append((prompt, partial))
        cur_blocks += -(-len(prompt) // B)
        last_sid = sid
    if cur:
        batches.append(cur)

    def step(bi, h2d_d2h=None):
        moved = 0
        dst_partials = []
        for prompt, partial in batches[bi % len(batches)]:
            mt, matched = P.match(prompt)
            src = np.concatenate([matched, partial])
            final, nm = P.transfer_with_insert(D.inst, prompt, src,
                                               flags=M.XFER_DEDUP | M.XFER_ASYNC)
            moved += nm
            dst_partials.append(final[len(prompt) // B:])
            if h2d_d2h is not None:
                h2d_d2h[0] += prompt.nbytes + src.nbytes
                h2d_d2h[1] += final.nbytes
        D.free_mem(np.concatenate(dst_partials))
        for prompt, _ in batches[bi % len(batches)]:
            D.delete(prompt)
        D.sync()      # the step ends when every block of the batch has landed
        return moved

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    st0, st1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = Clocks(os.path.join(ROOT, "gpurun_out", f"clocks_rank{rank}.csv")
                    if os.path.isdir(os.path.join(ROOT, "gpurun_out"))
                    else f"/tmp/clocks_rank{rank}.csv", dev)
    moved = 0
    io = [0, 0]
    with clocks:
        for w in range(args.warmup):
            step(w)
        barrier()
        D.stats_reset()
        P.stats_reset()
        D.profile(True)
        barrier()
        torch.cuda.profiler.start()     # ncu --profile-from-start off sees the timed region only
        st0.record()
        t0 = time.perf_counter()
        for k in range(args.steps):
            moved += step(args.warmup + k, io)
        st1.record()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        torch.cuda.profiler.stop()
    ms = st0.elapsed_time(st1)
    wall_ms = (t1 - t0) * 1e3
    D.profile(False)
    sd, sp = D.stats(), P.stats()
    # max over ranks
    tms = torch.tensor([ms, wall_ms], dtype=torch.float64, device=f"cuda:{dev}")
    tot = torch.tensor([float(moved)], dtype=torch.float64, device=f"cuda:{dev}")
    if dist is not None:
        dist.all_reduce(tms, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    ms, wall_ms = float(tms[0]), float(tms[1])
    blocks_all = float(tot[0])
    gbs = blocks_all * Pb / (ms * 1e-3) / 1e9
    blocks_s = blocks_all / (ms * 1e-3)
    e2e_gbs = blocks_all * Pb / (wall_ms * 1e-3) / 1e9

    peak, peak_src = load_peaks()
    kernel_ms = sd["kernel_ms"] / max(sd["timed_launches"], 1)
    bytes_per_launch = 2.0 * sd["timed_bytes"] / max(sd["timed_launches"], 1)  # read + write
    achieved = bytes_per_launch / (kernel_ms * 1e-3) / 1e9 if kernel_ms > 0 else None
    extras = {}
    if rank == 0 and not args.no_extras:
        extras = side_measurements(M, torch, P, D, shape, seed, peak, args)
    result = None
    if rank == 0:
        result = {
            "metric": "KV migration GB/s (P->D transfer_with_insert payload)",
            "value": round(gbs, 2),
            "unit": "GB/s",
            "blocks_per_s": round(blocks_s, 1),
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms / args.steps, 4),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "u16 (fp16 KV copied as opaque 16-bit words)",
            "data": "synthetic (seeded ShareGPT-like token traces; counter-based KV fill)",
            "config": {
                "workload": "configs[1]: Llama-2-7B-shaped KV (L32 H32 D128 fp16 B16, "
                            "Pb=8 MiB) ShareGPT-like 1P1D, PD-Caching-2 P->D with DEDUP",
                "placement": ("P and D as two pools on one GPU (loopback wire)" if world == 1
                              else f"{world} independent loopback P/D pairs, one per GPU"),
                "pool_blocks_per_instance": n_blocks,
                "batch_blocks": args.batch_blocks,
                "blocks_moved_total": int(blocks_all),
                "l2": "inputs larger than L2 (each step moves GiBs of distinct blocks)",
            },
            "e2e": {"value": round(e2e_gbs, 2), "unit": "GB/s",
                    "what": "host wall clock around the public Python API calls",
                    "h2d_bytes_per_step": int(io[0] / args.steps),
                    "d2h_bytes_per_step": int(io[1] / args.steps)},
            "gpu_launches": int(sd["kernel_launches"] + sd["aux_launches"] +
                                sp["kernel_launches"] + sp["aux_launches"]),
            "roofline": {
                "kernel": "migrate_kernel<pool,pool> (fused gather->store, A6f)",
                "bound": "hbm",
                "achieved": round(achieved, 1) if achieved else None,
                "peak": peak,
                "peak_source": peak_src,
                "unit": "GB/s",
                "frac": round(achieved / peak, 4) if achieved else None,
                "traffic": None,
                "bytes_per_launch_algorithmic": bytes_per_launch,
                "avg_launch_ms": round(kernel_ms, 5),
                "launches": int(sd["timed_launches"]),
                "share_of_step": round(sd["kernel_ms"] / ms, 4) if ms > 0 else None,
            },
            "clocks": clocks.summary(),
        }
        result.update(extras)
    return result


def side_measurements(M, torch, P, D, shape, seed, peak, args):
    """Standalone pack / unpack (A4/A6, HBM roofline) and swap (A8/A9)."""
    out = {}
    Pb = shape.block_bytes
    n = 128   # 2048-token prompt = 1 GiB at 7B: 8x the 126 MB L2
    dev = torch.cuda.current_device()
    del P, D
    for ck, ck_name in ((1, "vector"), (2, "bulk")):
        X = make_pool(M, torch, 200 + ck, dev, shape, 2 * n + 8, copy_kernel=ck)
        a = X.alloc_mem(n)
        X.debug_fill(a, seed)
        a = a[np.random.default_rng(seed).permutation(n)]      # scattered ids
        stg = torch.empty(n * Pb, dtype=torch.uint8, device=f"cuda:{dev}")
        b = X.alloc_mem(n)
        for name, fn in (("pack", lambda: X.pack(a, 0, shape.layers, stg.data_ptr())),
                         ("unpack", lambda: X.unpack(stg.data_ptr(), b, 0, shape.layers))):
            for _ in range(3):
                fn()
            X.stats_reset()
            X.profile(True)
            for _ in range(10):
                fn()
            X.profile(False)
            s = X.stats()
            kms = s["kernel_ms"] / s["timed_launches"]
            ach = 2.0 * n * Pb / (kms * 1e-3) / 1e9
            out[f"{name}_{ck_name}"] = {
                "blocks": n, "GBps_payload": round(n * Pb / (kms * 1e-3) / 1e9, 1),
                "hbm_GBps_rw": round(ach, 1), "frac_of_hbm": round(ach / peak, 4),
                "avg_kernel_ms": round(kms, 4)}
        X.close()
        del stg, X
    # swap sweep point: a separate small pool with pinned DRAM
    if not args.no_swap:
        try:
            out["swap"] = swap_point(M, torch, shape, seed, args)
        except Exception as e:  # report, never hide
            out["swap"] = {"error": str(e)}
    return out


def swap_point(M, torch, shape, seed, args):
    B, Pb = shape.block_tokens, shape.block_bytes
    nblk = 512
    dev = torch.cuda.current_device()
    S = make_pool(M, torch, 100, dev, shape, nblk, dram_blocks=nblk)
    rng = np.random.default_rng(seed)
    seqs = []
    for i in range(8):
        t = rng.integers(3, 32000, size=48 * B, dtype=np.int32)
        a = S.alloc_mem(48)
        S.debug_fill(a, seed)
        S.insert(t, a)
        seqs.append(t)
    res = {}
    for n in (64, 256):
        S.stats_reset()
        S.profile(True)
        t0 = time.perf_counter()
        old, new = S.swap_out(n)
        t1 = time.perf_counter()
        back = S.swap_in(new)
        t2 = time.perf_counter()
        S.profile(False)
        res[f"n{n}"] = {"swap_out_GBps": round(len(old) * Pb / (t1 - t0) / 1e9, 2),
                        "swap_in_GBps": round(len(back) * Pb / (t2 - t1) / 1e9, 2),
                        "path": "zero-copy SM loads/stores to mapped pinned DRAM"}
    S.close()
    return res


# ------------------------------------------------------------ cpu baseline
def run_oracle(seconds_budget, steps=1):
    """The CPU oracle as it stands (materialised numpy byte path), same
    workload shape, on a bounded sample: a 7B-shaped pool of 160 blocks per
    instance and as many whole requests as fit the time budget."""
    import oracle as O
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
        cores = 1
    except Exception:
        cores = os.cpu_count()
    shape = LLAMA2_7B
    B, Pb = shape.block_tokens, shape.block_bytes
    nb = 160
    seed = seed_for(1)
    mk = lambda inst: O.OraclePool(inst, shape.layers, shape.kv_heads, shape.head_dim, B, nb,
                                   seed=seed, materialize=True)
    P, D = mk(0), mk(1)
    reqs = build_requests(shape, seed, nb, int(nb * 0.8))
    srcs = []
    for sid, prompt in reqs:
        mt, matched = P.match(prompt)
        new = P.alloc_mem(-(-len(prompt) // B) - len(matched), O.HBM)
        P.fill(new)
        full = matched + new
        P.insert(prompt, full[: len(prompt) // B])
        srcs.append(full[len(prompt) // B:])
    moved = 0
    t_total = 0.0
    n_req = 0
    for _ in range(steps):
        t0 = time.perf_counter()
        done = []
        for (sid, prompt), partial in zip(reqs, srcs):
            _, matched = P.match(prompt)
            final, nm, _ = O.transfer_with_insert(P, D, prompt, matched + partial,
                                                  flags=O.FLAG_DEDUP)
            moved += nm
            n_req += 1
            done.append((prompt, final[len(prompt) // B:]))
            if time.perf_counter() - t0 > seconds_budget:
                break
        for prompt, part in done:
            D.free_mem(part)
            D.delete(prompt)
        t_total += time.perf_counter() - t0
    return {"value": round(moved * Pb / t_total / 1e9, 4), "unit": "GB/s", "cores": cores,
            "kind": "oracle",
            "sample": f"{n_req} ShareGPT-like requests x {steps} step(s), 7B shape, "
                      f"{nb}-block pools, DEDUP P->D transfer_with_insert, numpy byte path",
            "blocks_moved": moved, "seconds": round(t_total, 3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pool-blocks", type=int, default=4096)
    ap.add_argument("--batch-blocks", type=int, default=1024)
    ap.add_argument("--copy-kernel", type=int, default=0,
                    help="0 auto, 1 vector LD/ST, 2 bulk cp.async (TMA) copy engine")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-swap", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))

    if args.impl == "reference":
        # The reference arm is the CPU oracle (no upstream code exists); rank 0 only.
        if rank != 0:
            return
        steps = []
        r = None
        for _ in range(args.warmup):
            run_oracle(min(2.0, args.cpu_seconds))
        for _ in range(args.steps):
            r = run_oracle(max(1.0, args.cpu_seconds / max(args.steps, 1)))
            steps.append(r)
        tot_b = sum(x["blocks_moved"] for x in steps)
        tot_s = sum(x["seconds"] for x in steps)
        val = tot_b * LLAMA2_7B.block_bytes / tot_s / 1e9
        print(json.dumps({
            "impl": "reference",
            "metric": "KV migration GB/s (P->D transfer_with_insert payload)",
            "value": round(val, 4), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(tot_s * 1e3 / max(args.steps, 1), 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u16 (fp16 KV copied as opaque 16-bit words)", "data": "synthetic",
            "config": {"workload": "configs[1]: Llama-2-7B-shaped KV ShareGPT-like 1P1D "
                                   "(bounded sample per step, CPU oracle)"},
            "cpu_baseline": {"value": round(val, 4), "unit": "GB/s", "cores": r["cores"],
                             "kind": "oracle", "sample": r["sample"]},
            "e2e": {"value": round(val, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
        }))
        return

    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist_mod
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist_mod.init_process_group("nccl")
        dist = dist_mod
    res = run_ours(args, rank, world, dist)
    if rank == 0:
        if not args.no_cpu_baseline:
            cb = run_oracle(args.cpu_seconds)
            cb.pop("blocks_moved", None)
            cb.pop("seconds", None)
            res["cpu_baseline"] = cb
        print(json.dumps(res))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

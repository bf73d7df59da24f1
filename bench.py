#!/usr/bin/env python
"""bench.py -- KV migration GB/s & blocks/s vs the HBM / NVLink roofline.

BASELINE.json metric: "KV migration GB/s & blocks/s vs HBM/NVLink roofline at
1/2/4/8 B200".  Workload: configs[1], Llama-2-7B-shaped KV (L=32, H=32,
D=128, fp16, B=16 -> Pb = 8 MiB per token block), ShareGPT-like prompts,
1P1D per pair.  Placement (paper_2406_17565_b200/topology.py):
N = 1 puts P and D as two pools on cuda:0 (the wire is a device-local copy);
N > 1 (torchrun) runs one process per GPU, P_i = rank i and D_i = rank i+N/2,
and P_i's fused kernel stores straight into D_i's IPC-mapped pool over NVLink.

One STEP = one pass of the migration hot path over one batch of requests
(PD-Caching-2, §5.1):
    for each request: P.match(prompt)                              (A3)
                      P.transfer_with_insert(D, prompt, src, DEDUP)
                        -> D: match, alloc (A2), gather->store (A6f), insert (A7)
    then D retires the batch: free_mem(partial blocks) + delete(prompts).
value = payload bytes actually moved (blocks moved x Pb) / step time, summed
over pairs, time = max over ranks (CUDA events).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
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
NOMINAL_HBM_GBS = 7700.0    # B200_PROFILING.md: HBM3e 7.7 TB/s (HGX figure); the measured
                            # peak above is torch's contiguous copy_, which the ring beats
NVLINK_GBS = 900.0          # nominal per direction per GPU (BJ:5)
NVLINK_GUIDE_GBS = 770.0    # B200_PROFILING.md: measured peer copy per direction (fallback
                            # when the in-run probe below is off)
PATHS = {"fused": "PATH_FUSED", "staged": "PATH_STAGED", "ce": "PATH_CE"}
PATH_NOTES = {
    "fused": "FUSED: one gather -> store kernel per transfer (A6f), straight into the "
             "receiver's blocks (peer stores over NVLink across GPUs)",
    "staged": "STAGED: pack into a staging slot (A4), one copy-engine copy into the "
              "receiver's inbound ring (A5), unpack there (A6), pipelined over the ring",
    "ce": "CE: one copy-engine memcpy per (block, layer, K/V) chunk (the paper's discrete "
          "per-block transfer, P:546-547)"}
METRIC = "KV migration GB/s (P->D transfer_with_insert payload)"
WORKLOAD = ("configs[1]: Llama-2-7B-shaped KV (L32 H32 D128 fp16 B16, Pb=8 MiB) ShareGPT-like "
            "1P1D per pair, PD-Caching-2 P->D with DEDUP")
DTYPE = "u16"          # the path computes nothing: fp16 KV is copied as opaque 16-bit words
KV_DTYPE = "fp16 KV copied as opaque 16-bit words (bit-exact, NaN payloads preserved)"


def ncu_traffic_ratio(engine):
    """DRAM traffic / algorithmic bytes of the migration kernel from the latest
    committed `ncu --set full` capture (profiles/ncu_traffic_r*.json; the
    longest captured launch).  None when no capture exists."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_traffic_r*.json")))
    for path in reversed(files):    # the latest capture of this engine
        with open(path) as f:
            launches = json.load(f).get(engine) or []
        if launches:
            big = max(launches, key=lambda l: l["duration_us"])
            return big["traffic_over_algorithmic"], os.path.relpath(path, ROOT)
    return None, None


def load_peaks():
    try:
        with open(PEAKS_PATH) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: copy read+write)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------- workload
def build_requests(shape, seed, fill_budget):
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


def make_batches(reqs, partials, batch_blocks, B):
    """Batches of whole sessions, each about batch_blocks prompt blocks."""
    batches, cur, cur_blocks, last_sid = [], [], 0, None
    for (sid, prompt), partial in zip(reqs, partials):
        if sid != last_sid and cur_blocks >= batch_blocks:
            batches.append(cur)
            cur, cur_blocks = [], 0
        cur.append((prompt, partial))
        cur_blocks += -(-len(prompt) // B)
        last_sid = sid
    if cur:
        batches.append(cur)
    return batches


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
    """HBM slabs are torch allocations (PyTorch owns device memory).  With the
    caching allocator's expandable segments (cuMemMap-backed, no CUDA-IPC
    handle) the library cudaMallocs the slabs itself, so the cross-process
    path can still export them."""
    if "expandable_segments:true" in os.environ.get("PYTORCH_CUDA_ALLOC_CONF", "").lower():
        p = M.Pool(inst, dev, shape.layers, shape.kv_heads, shape.head_dim, shape.block_tokens,
                   n_blocks, **kw)
        p._region = None
        return p
    c = shape.chunk_bytes
    region = torch.empty(2 * shape.layers * n_blocks * c, dtype=torch.uint8, device=f"cuda:{dev}")
    slabs = [region.data_ptr() + j * n_blocks * c for j in range(2 * shape.layers)]
    p = M.Pool(inst, dev, shape.layers, shape.kv_heads, shape.head_dim, shape.block_tokens,
               n_blocks, slabs=slabs, **kw)
    p._region = region
    return p


def populate_prefill(P, shape, seed, n_blocks):
    """Untimed setup: the prefill instance's cache (PD-Caching-1 step 2)."""
    B = shape.block_tokens
    reqs = build_requests(shape, seed, int(n_blocks * 0.9))
    partials = []
    for sid, prompt in reqs:
        mt, matched = P.match(prompt)
        new = P.alloc_mem(-(-len(prompt) // B) - len(matched))
        P.debug_fill(new, seed)
        full = np.concatenate([matched, new])
        P.insert(prompt, full[: len(prompt) // B])
        partials.append(full[len(prompt) // B:])       # trailing partial block (active)
    return reqs, partials


def pair_table(recs, Pb):
    """Per pair and direction from every rank's record: each P
    rank's own payload over its own device time, against the nominal link and
    its own in-run probe.  Pure host arithmetic (tested on CPU)."""
    per_pair = []
    for r in recs:
        if r["kind"] not in ("P", "PD"):
            continue
        g = r["moved"] * Pb / (r["ms"] * 1e-3) / 1e9 if r["ms"] > 0 else 0.0
        pk = (r["probe"] or {}).get("GBps")
        e = {"pair": r["pair"], "direction": "P->D" if r["kind"] == "P" else "loopback",
             "p_rank": r["rank"], "d_rank": r["partner"], "GBps": round(g, 1),
             "blocks_per_s": round(r["moved"] / (r["ms"] * 1e-3), 1) if r["ms"] > 0 else 0.0,
             "kernel_GBps": r["kernel_GBps"]}
        if r["kind"] == "P":
            e["frac_of_nominal_900"] = round(g / NVLINK_GBS, 4)
            e["probe_GBps"] = pk
            e["frac_of_probe"] = round(g / pk, 4) if pk else None
            e["kernel_frac_of_probe"] = (round(r["kernel_GBps"] / pk, 4)
                                         if pk and r["kernel_GBps"] else None)
        per_pair.append(e)
    return sorted(per_pair, key=lambda e: e["pair"])


def run_ours(args, rank, world, dist):
    import torch
    from paper_2406_17565_b200 import mempool as M
    from paper_2406_17565_b200.topology import role_of

    role = role_of(rank, world)
    dev = int(os.environ.get("LOCAL_RANK", 0)) if args.device < 0 else args.device
    torch.cuda.set_device(dev)
    shape = LLAMA2_7B
    B, Pb = shape.block_tokens, shape.block_bytes
    seed = seed_for(1) + 1000 * role.pair
    n_blocks = args.pool_blocks
    P = D = None
    knobs = dict(copy_kernel=args.copy_kernel, peer_engine=args.peer_engine,
                 peer_sched=args.peer_sched, max_ctas=args.max_ctas,
                 coalesce_mib=args.coalesce_mib)
    probe = None
    if role.kind != "PD" and not args.no_probe:
        # before the pools take HBM: the box's own large peer copy P_i -> D_i
        probe = link_probe(torch, dist, role, dev, world)
    if role.kind in ("PD", "P"):
        P = make_pool(M, torch, role.p_inst, dev, shape, n_blocks, **knobs)
    if role.kind in ("PD", "D"):
        D = make_pool(M, torch, role.d_inst, dev, shape, n_blocks, **knobs)
    if role.kind == "PD":
        M.connect(P, D)
    else:
        me = P if role.kind == "P" else D
        blobs = M.exchange_handles(me)
        me.import_peer(blobs[role.partner][1])
        dist.barrier()
    batches = None
    if P is not None:
        reqs, partials = populate_prefill(P, shape, seed, n_blocks)
        batches = make_batches(reqs, partials, args.batch_blocks, B)
    wire = None
    if role.kind in ("P", "D"):
        wire = wire_check(M, torch, dist, role, P if P is not None else D, shape, world, dev,
                          getattr(M, PATHS[args.xfer_path]))
        if not wire["ok"]:
            raise RuntimeError(f"rank {rank}: wire check failed (bytes differ)")

    host_t = {"match": 0.0, "twi": 0.0, "n": 0}
    # D needs each batch's request count (it retires exactly that batch while
    # the sender's next requests may already be queued): P tells it once
    batch_sizes = [len(b) for b in batches] if batches is not None else None
    if role.kind in ("P", "D"):
        sizes = [None] * world
        dist.all_gather_object(sizes, batch_sizes)
        if role.kind == "D":
            batch_sizes = sizes[role.partner]
    pending_msgs = [0]
    xflags = M.XFER_DEDUP | M.XFER_ASYNC | getattr(M, PATHS[args.xfer_path])
    if role.kind == "P" and not args.no_pipeline:
        # cross-process: each copy is enqueued at the next call, right after
        # that call's request went out (overlaps the launch with the round trip)
        xflags |= M.XFER_PIPELINE

    def p_step(bi, io=None):
        """Prefill side of one step."""
        moved = 0
        sent = []
        for prompt, partial in batches[bi % len(batches)]:
            t0 = time.perf_counter()
            mt, matched = P.match(prompt)
            src = np.concatenate([matched, partial])
            priv = prompt.tobytes() if role.kind == "P" else b""
            t1 = time.perf_counter()
            final, nm = P.transfer_with_insert(role.d_inst, prompt, src, flags=xflags,
                                               priv=priv)
            t2 = time.perf_counter()
            if io is not None:
                host_t["match"] += t1 - t0
                host_t["twi"] += t2 - t1
                host_t["n"] += 1
            moved += nm
            sent.append((prompt, final))
            if io is not None:
                io[0] += prompt.nbytes + src.nbytes + len(priv)
                io[1] += final.nbytes
        return moved, sent

    def d_retire(done):
        """Decode side: the batch is retired (partials freed, prompts deleted)."""
        D.free_mem(np.concatenate([f[len(p) // B:] for p, f in done]))
        for prompt, _ in done:
            D.delete(prompt)

    def step(bi, io=None):
        if role.kind == "D":
            pending_msgs[0] = batch_sizes[bi % len(batch_sizes)]
        if role.kind == "PD":
            # no host sync between steps: step k's copies stream on while the
            # host issues step k+1 (stream order keeps every reuse of a block
            # behind its earlier copies); the timed region ends with a sync
            moved, sent = p_step(bi, io)
            d_retire(sent)
            return moved
        if role.kind == "P":
            moved, _ = p_step(bi, io)
            P.send_mark(role.d_inst, bi)   # end of batch: D retires it
            return moved
        served, mark = D.serve(timeout_ms=600_000, until_mark=True)
        if mark != bi:
            raise RuntimeError(f"decode rank {rank}: expected mark {bi}, got {mark}")
        done = []
        while len(done) < pending_msgs[0]:    # this batch's messages (not the next one's)
            m = D.recv_poll()
            if m is None:
                raise RuntimeError(f"decode rank {rank}: batch {bi} short of messages")
            done.append((np.frombuffer(m[2], dtype=np.int32), m[3]))
        # retire the batch (host-side; stream order protects reused blocks),
        # answering the sender's next requests between prompts, as a serving
        # engine interleaves its own work with the pool's service loop
        D.free_mem(np.concatenate([f[len(p) // B:] for p, f in done]))
        for k, (prompt, _) in enumerate(done):
            D.delete(prompt)
            if k % 4 == 3:
                D.serve(timeout_ms=0, until_mark=False)
        return 0

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    timed_pool = D if role.kind == "PD" else (P if role.kind == "P" else D)
    st0, st1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out_dir = os.path.join(ROOT, "gpurun_out")
    clocks = Clocks(os.path.join(out_dir if os.path.isdir(out_dir) else "/tmp",
                                 f"clocks_rank{rank}.csv"), dev)
    moved = moved_e2e = 0
    io = [0, 0]
    with clocks:
        time.sleep(1.0)                 # nvidia-smi needs a moment before its first sample
        for w in range(args.warmup):
            step(w)
        barrier()
        for pl in (P, D):
            if pl is not None:
                pl.stats_reset()
        timed_pool.profile(True, every=args.profile_every)
        barrier()
        torch.cuda.profiler.start()     # ncu --profile-from-start off sees the timed region only
        st0.record()
        t0 = time.perf_counter()
        # per-step device boundaries: an event after each step's work on the
        # stream the copies run on (the sender's; at N=1 both pools share it)
        mark_pool = P if role.kind in ("PD", "P") else None
        step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        step_moved = []
        if mark_pool is not None:
            mark_pool.record_event(step_ev[0])
        for k in range(args.steps):
            mk = step(args.warmup + k, io)
            moved += mk
            step_moved.append(mk)
            if mark_pool is not None:
                mark_pool.record_event(step_ev[k + 1])
        for pl in (P, D):      # every block of every step has landed
            if pl is not None:
                pl.sync()
        st1.record()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        # e2e: K more steps through the public API, each ending with the
        # completion a serving loop waits for before decoding (the "ok" of
        # the step's KV has landed and the receiver inserted it), so
        # there is no pipelining across steps; host wall clock
        st = timed_pool.stats()
        launches = sum(pl.stats()["kernel_launches"] + pl.stats()["aux_launches"]
                       for pl in (P, D) if pl is not None)
        timed_pool.profile(False)
        barrier()
        t0 = time.perf_counter()
        for k in range(args.steps):
            moved_e2e += step(args.warmup + args.steps + k, io)
            # receiver first: its queued bitmap frees go to the device behind
            # the step's copies instead of after them (one wait, not two)
            for pl in (D, P):
                if pl is not None and (role.kind != "D"):
                    pl.sync()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
    ms = st0.elapsed_time(st1)
    wall_ms = (t1 - t0) * 1e3
    step_stats = None
    if mark_pool is not None and args.steps >= 2:
        sms = np.array([step_ev[k].elapsed_time(step_ev[k + 1]) for k in range(args.steps)])
        sgb = np.array(step_moved, dtype=np.float64) * Pb / (sms * 1e-3) / 1e9
        step_stats = {"what": "device time between consecutive end-of-step events on the "
                              "copy stream (this rank), and that step's payload rate",
                      "ms_p10_p50_p90": [round(float(np.percentile(sms, q)), 4) for q in (10, 50, 90)],
                      "GBps_p10_p50_p90": [round(float(np.percentile(sgb, q)), 1)
                                           for q in (10, 50, 90)]}
    # whole job: time = max over ranks, blocks and launches = sum over ranks
    rdev = f"cuda:{dev}" if args.dist_backend == "nccl" else "cpu"
    tms = torch.tensor([ms, wall_ms], dtype=torch.float64, device=rdev)
    tot = torch.tensor([float(moved), float(launches), float(io[0]), float(io[1]),
                        float(moved_e2e)], dtype=torch.float64, device=rdev)
    if dist is not None:
        dist.all_reduce(tms, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    ms, wall_ms = float(tms[0]), float(tms[1])
    blocks_all, launches_all = float(tot[0]), int(tot[1])
    gbs = blocks_all * Pb / (ms * 1e-3) / 1e9
    blocks_s = blocks_all / (ms * 1e-3)
    e2e_gbs = float(tot[4]) * Pb / (wall_ms * 1e-3) / 1e9

    peak, peak_src = load_peaks()
    kernel_ms = st["kernel_ms"] / max(st["timed_launches"], 1)
    # sampled launches stand for all the data-stream migrations of the region
    # (ratio estimator: kernel time per byte of the sampled launches x all bytes)
    kernel_ms_total = (st["kernel_ms"] * st["profiled_bytes"] / st["timed_bytes"]
                       if st["timed_bytes"] else 0.0)
    payload_per_launch = st["timed_bytes"] / max(st["timed_launches"], 1)
    same_gpu = role.kind == "PD" or args.device >= 0   # --device: every rank on one GPU
    # engine the library picks (pool.cpp launch_migrate_timed): copies within
    # one GPU's HBM -- loopback, or an IPC peer on the same GPU -- take
    # copy_kernel (auto = the bulk ring); stores into another GPU take
    # peer_engine (auto = vector LD/ST unless MP_PEER_ENGINE=bulk)
    if same_gpu:
        bulk = args.copy_kernel != 1
    else:
        eng = args.peer_engine or args.copy_kernel
        bulk = eng == 2 or (eng == 0 and os.environ.get("MP_PEER_ENGINE", "").startswith("b"))
    kname = "migrate_bulk_kernel" if bulk else "migrate_kernel"
    if same_gpu:
        # loopback: the kernel reads Pb and writes Pb of HBM per block
        alg = 2.0 * payload_per_launch
        roof = {"kernel": f"{kname}<pool,pool> (fused gather->store, A6f), "
                          + ("loopback" if role.kind == "PD" else
                             "two processes on one GPU (IPC-mapped receiver pool)"),
                "bound": "hbm", "peak": peak, "peak_source": peak_src}
    else:
        # across GPUs the bound is the NVLink direction P -> D: Pb per block
        alg = payload_per_launch
        if probe and probe.get("GBps"):
            lpeak, lsrc = probe["GBps"], ("in-run peer copy P_0 -> D_0: " + probe["what"])
        else:
            lpeak, lsrc = NVLINK_GUIDE_GBS, "B200_PROFILING.md measured peer copy per direction"
        roof = {"kernel": f"{kname}<pool,pool> (fused gather->peer store over NVLink)",
                "bound": "nvlink", "peak": lpeak,
                "peak_source": f"{lsrc} (nominal {NVLINK_GBS} GB/s)"}
    achieved = alg / (kernel_ms * 1e-3) / 1e9 if kernel_ms > 0 else None
    # per pair and direction: every P rank's own payload over its
    # own device time, against the nominal link and its own in-run probe
    rec = {"rank": rank, "kind": role.kind, "pair": role.pair, "partner": role.partner,
           "moved": moved, "ms": ms,
           "kernel_GBps": round(achieved, 1) if achieved else None,
           "probe": probe}
    recs = [rec]
    if dist is not None:
        recs = [None] * world
        dist.all_gather_object(recs, rec)
    per_pair = pair_table(recs, Pb)
    ratio, ratio_src = (ncu_traffic_ratio("bulk" if bulk else "vector")
                        if same_gpu else (None, None))
    roof.update({
        "achieved": round(achieved, 1) if achieved else None, "unit": "GB/s",
        "frac": round(achieved / roof["peak"], 4) if achieved else None,
        "nominal_peak": NOMINAL_HBM_GBS if same_gpu else NVLINK_GBS,
        "frac_of_nominal": (round(achieved / (NOMINAL_HBM_GBS if same_gpu else NVLINK_GBS), 4)
                            if achieved else None),
        "traffic": round(ratio * alg) if ratio else None,
        "traffic_note": (f"dram read+write per launch = {ratio} x algorithmic, from the ncu "
                         f"capture {ratio_src} (writes still in L2 at kernel end are not "
                         "counted; no re-reads)") if ratio else None,
        "bytes_per_launch_algorithmic": alg,
        "avg_launch_ms": round(kernel_ms, 5), "launches": int(st["profiled_launches"]),
        "timed_launches": int(st["timed_launches"]),
        "timing": (f"CUDA events on the launching stream around every {args.profile_every}-th "
                   "migration launch of the timed region (the events cost a few us per "
                   "launch; sampling keeps that out of the step)"),
        "share_of_step": round(kernel_ms_total / ms, 4) if ms > 0 else None,
        "share_note": ("estimated as the sampled launches' time per byte x every launch's "
                       "bytes / step time; a timed launch is bracketed by events, so it cannot "
                       "overlap its neighbours under PDL and the estimate may slightly exceed 1"),
        "idle_between_launches_share": (round(st["gap_ms"] / ms, 4)
                                        if ms > 0 and args.profile_every == 1 else None)})
    extras = {}
    if not args.no_extras:
        # CUPTI (kineto) durations of the migration kernels over extra steps:
        # not bracketed by events, so PDL overlap is kept and the union of the
        # kernels' busy intervals is at most the pass's device time
        try:
            cupti = cupti_share(torch, step, mark_pool, args, 2 * args.steps + args.warmup,
                                (2 if same_gpu else 1) * Pb)
            if cupti and cupti.get("achieved_over_busy_GBps"):
                cupti["frac_over_busy"] = round(cupti["achieved_over_busy_GBps"] / roof["peak"], 4)
        except Exception as e:     # report, never hide
            cupti = {"error": str(e)[:300]}
        if rank == 0:
            roof["cupti"] = cupti
            if cupti and cupti.get("share_of_step") is not None:
                # the step's kernel share from un-bracketed (CUPTI) durations
                roof["share_of_step_events"] = roof["share_of_step"]
                roof["share_of_step"] = cupti["share_of_step"]
                roof["share_source"] = "cupti (roofline.cupti); share_of_step_events: the " \
                                       "event-sampled estimate"
    if not args.no_extras and dist is not None and role.kind != "PD":
        try:
            pair_nccl = nccl_pair_point(M, torch, dist, role, P if P is not None else D,
                                        shape, seed, world)
        except Exception as e:     # report, never hide
            pair_nccl = {"error": str(e)[:300]}
        if rank == 0:
            extras["paper_transport_nccl"] = pair_nccl
    if rank == 0 and not args.no_extras:
        extras.update(side_measurements(M, torch, shape, seed, peak, args,
                                        nccl_local=dist is None or role.kind == "PD"))
    if rank != 0:
        return None
    placement = ("P and D as two pools on one GPU (loopback wire)" if world == 1 else
                 f"{world // 2}P{world // 2}D: P_i on GPU i, D_i on GPU i+{world // 2}, "
                 "one process per GPU, one-sided NVLink stores into IPC-mapped peer pools")
    result = {
        "metric": METRIC,
        "value": round(gbs, 2),
        "unit": "GB/s",
        "blocks_per_s": round(blocks_s, 1),
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms / args.steps, 4),
        "per_step": step_stats,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": DTYPE,
        "data": "synthetic (seeded ShareGPT-like token traces; counter-based KV fill)",
        "config": {
            "workload": WORKLOAD,
            "kv_dtype": KV_DTYPE,
            "placement": placement,
            "wire_bound": ("HBM read+write of one GPU (loopback; N=1 has no wire)" if world == 1
                           else f"NVLink per direction, {world // 2} independent pair(s): "
                                "N=1 -> 2 changes the bound from HBM to NVLink, so weak "
                                "scaling is meaningful from N=2 on"),
            "xfer_path": PATH_NOTES[args.xfer_path],
            "peer_engine": ["auto", "vector LD/ST", "bulk cp.async ring"][args.peer_engine],
            "peer_sched": ["auto", "static split", "dynamic unit claiming"][args.peer_sched],
            "pipelined_issue": (world > 1 and not args.no_pipeline),
            "pool_blocks_per_instance": n_blocks,
            "batch_blocks": args.batch_blocks,
            "copy_kernel": ["auto (bulk cp.async ring in HBM)", "vector LD/ST",
                            "bulk cp.async ring"][args.copy_kernel],
            "max_ctas": args.max_ctas or "one full wave",
            "coalesce_mib": args.coalesce_mib or 4096,
            "blocks_moved_total": int(blocks_all),
            "l2": "inputs larger than L2 (each step moves GiBs of distinct blocks)",
            "step_sync": ("no host sync between steps (stream-ordered); the timed region "
                          "ends with a full sync of every pool" +
                          ("" if world == 1 else
                           "; an end-of-step mark from P to D makes D retire the batch")),
        },
        "e2e": {"value": round(e2e_gbs, 2), "unit": "GB/s",
                "what": "host wall clock over K further steps through the public Python API, "
                        "each ending with a completion sync of the pools (the step's KV has "
                        "landed, P:365) -- no pipelining across steps.  Inputs: token lists "
                        "and source block addrs from host memory (ids reach the device in "
                        "kernel parameters); results: the receiver's block addrs back",
                "h2d_bytes_per_step": int(float(tot[2]) / (2 * args.steps)),
                "d2h_bytes_per_step": int(float(tot[3]) / (2 * args.steps))},
        "gpu_launches": launches_all,
        "host_us_per_request": {k: round(v / max(host_t["n"], 1) * 1e6, 2)
                                for k, v in host_t.items() if k != "n"},
        "roofline": roof,
        "per_pair": per_pair,
        "wire_check": wire,
        "nvlink_peak_measured": ({"GBps_per_pair": [(r["probe"] or {}).get("GBps")
                                                    for r in recs if r["kind"] == "P"],
                                  "nominal_GBps": NVLINK_GBS,
                                  "what": probe["what"] if probe else None}
                                 if world > 1 else None),
        "clocks": clocks.summary(),
    }
    result.update(extras)
    return result


def link_probe(torch, dist, role, dev, world, nbytes=1 << 30, reps=8):
    """The box's own large peer copy P_i -> D_i, per pair (the achievable peak
    beside the 900 GB/s nominal): D_i exports a 1 GiB buffer by
    CUDA IPC (torch's own sharing), P_i maps it and times `reps` copies from
    its HBM into it with CUDA events (cudaMemcpyAsync over NVLink, P2P).
    Returns {"GBps", "what"} on P ranks, None on D ranks."""
    from torch.multiprocessing.reductions import reduce_tensor
    buf = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{dev}")
    mine = reduce_tensor(buf) if role.kind == "D" else None
    objs = [None] * world
    dist.all_gather_object(objs, mine)
    out = None
    if role.kind == "P":
        fn, fargs = objs[role.partner]
        remote = fn(*fargs)
        buf.fill_(1)
        remote.copy_(buf)                          # warm: peer access, first touch
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            remote.copy_(buf, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        ok = bool((remote[:: 1 << 20] == 1).all())
        out = {"GBps": round(reps * nbytes / (ms * 1e-3) / 1e9, 1),
               "what": (f"{reps} x 1 GiB torch copy_ from GPU {dev} into GPU "
                        f"{remote.device.index}'s IPC-mapped buffer (cudaMemcpyAsync, P2P), "
                        "CUDA events" + ("" if ok else "; VERIFY FAILED"))}
        del remote
    torch.cuda.synchronize()
    dist.barrier()                                 # D keeps its buffer until P is done
    del buf
    torch.cuda.empty_cache()
    return out


def wire_check(M, torch, dist, role, pool, shape, world, dev, flags, n=8):
    """Before timing at N > 1: P_i moves n freshly filled blocks to D_i over
    the bench's transport (synchronous transfer), both sides checksum every
    chunk of them (weighted int64 sums, same weights on both GPUs), and the
    sums are compared.  Returns {"blocks", "ok", ...} on every rank."""
    L2, c, nb = 2 * shape.layers, shape.chunk_bytes, pool.hbm_blocks
    view = pool._region.view(L2, nb, c).view(torch.int64)
    g = torch.Generator().manual_seed(11)
    w = torch.randint(-2**31, 2**31, (c // 8,), generator=g).to(f"cuda:{dev}")

    def sums(addrs):
        pool.sync()
        t = torch.as_tensor(M.addr_indices(addrs).astype(np.int64), device=f"cuda:{dev}")
        return torch.stack([(view[j][t] * w).sum(-1) for j in range(L2)], 1).cpu().tolist()

    mine = None
    if role.kind == "P":
        src = pool.alloc_mem(n)
        pool.debug_fill(src, 4242)
        pool.transfer(role.d_inst, src, flags=flags)
        mine = sums(src)
        pool.send_mark(role.d_inst, 1 << 29)
        pool.free_mem(src)
    else:
        _s, mark = pool.serve(timeout_ms=300_000, until_mark=True)
        if mark != 1 << 29:
            raise RuntimeError(f"wire check: unexpected mark {mark}")
        m = pool.recv_poll()
        mine = sums(m[3])
        pool.free_mem(m[3])
        pool.sync()
    allsums = [None] * world
    dist.all_gather_object(allsums, mine)
    ok = allsums[role.rank] == allsums[role.partner]
    return {"blocks": n, "ok": bool(ok),
            "what": "P_i -> D_i transfer of freshly filled blocks over the bench's transport; "
                    "weighted checksums of every chunk on both GPUs compared"}


def cupti_busy(prof, match="migrate"):
    """(launches, summed duration us, union of the [start, end) intervals us)
    of the device kernels whose name contains `match` (None: every kernel),
    from a torch.profiler run's CUPTI (kineto) activity records -- durations
    not bracketed by events."""
    from torch.autograd import DeviceType
    iv = sorted((ev.time_range.start, ev.time_range.end) for ev in prof.events()
                if ev.device_type == DeviceType.CUDA and (match is None or match in ev.name)
                and ev.time_range.end > ev.time_range.start)
    if not iv:
        return 0, 0.0, 0.0
    busy, cs, ce = 0.0, iv[0][0], iv[0][1]
    for a, b in iv[1:]:
        if a > ce:
            busy += ce - cs
            cs, ce = a, b
        else:
            ce = max(ce, b)
    busy += ce - cs
    return len(iv), float(sum(b - a for a, b in iv)), busy


def cupti_share(torch, step, mark_pool, args, first, alg_per_block):
    """Kernel share of the step from CUPTI activity records (torch.profiler /
    kineto; no events around the launches): union of the migration kernels'
    [start, end) intervals over a pass of extra steps / that pass's device
    time (end-of-step events on the copy stream).  Also the average CUPTI
    duration per migration launch."""
    from torch.profiler import ProfilerActivity, profile
    n = max(2, min(args.steps, 20))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    moved = 0
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        if mark_pool is not None:
            mark_pool.record_event(e0)
        for k in range(n):
            moved += step(first + k)
        if mark_pool is not None:
            mark_pool.sync()
            mark_pool.record_event(e1)
        torch.cuda.synchronize()
    if mark_pool is None:
        return None
    nl, tot, busy = cupti_busy(prof)
    if not nl:
        return {"error": "no migration kernels in the CUPTI records"}
    na, tot_all, _ = cupti_busy(prof, None)
    pass_ms = e0.elapsed_time(e1)
    return {"steps": n, "launches": nl, "avg_launch_us": round(tot / nl, 3),
            "all_kernel_launches": na,
            "share_of_kernel_time": round(tot / tot_all, 4) if tot_all else None,
            "busy_ms": round(busy / 1e3, 4), "pass_ms": round(pass_ms, 4),
            "share_of_step": round(busy / 1e3 / pass_ms, 4) if pass_ms > 0 else None,
            "payload_blocks": int(moved),
            "achieved_over_busy_GBps": round(moved * alg_per_block / (busy * 1e-6) / 1e9, 1),
            "what": "CUPTI kernel records (torch.profiler) of the migration kernels over extra "
                    "untimed steps; busy = union of their intervals"}


def nccl_pair_point(M, torch, dist, role, pool, shape, seed, world, n=128):
    """The paper's transport across a real pair (P:546-547, P:668-672,
    P:860-868): a 2-rank NCCL communicator per (P_i, D_i), the same 128
    scattered blocks (a 2048-token prompt) sent (1) discrete: one ncclSend /
    ncclRecv per (layer, K/V) chunk, one group per block, (2) aggregated:
    mp_pack -> one send -> mp_unpack, beside (3) our transfer (the bench's
    transport).  Wall clock per synchronous transfer, bracketed by barriers
    of the pair's two ranks, median of 3 after one warm-up.  Every run's
    destination is checked chunk by chunk against the source on the
    receiver (first chunk of every block, via the pool's debug read)."""
    from paper_2406_17565_b200 import nccl_arm as N
    dev = torch.cuda.current_device()
    Pb, L, c = shape.block_bytes, shape.layers, shape.chunk_bytes
    uid = N.unique_id() if role.kind == "P" else None
    uids = [None] * world
    dist.all_gather_object(uids, uid)
    p_rank = role.rank if role.kind == "P" else role.partner
    comm = N.NcclComm.create(2, 0 if role.kind == "P" else 1, dev, uids[p_rank])
    peer = 1 if role.kind == "P" else 0
    st = torch.cuda.current_stream()
    stg = torch.empty(n * Pb, dtype=torch.uint8, device=f"cuda:{dev}")
    base = pool._region.data_ptr() if pool._region is not None else None
    if base is None:
        raise RuntimeError("needs torch-allocated slabs")
    nb = pool.hbm_blocks

    def chunk_ptrs(ids):
        return [base + (j * nb + int(i)) * c for i in ids for j in range(2 * L)]

    rng = np.random.default_rng(seed + 7)
    if role.kind == "P":
        src = pool.alloc_mem(n)
        pool.debug_fill(src, seed)
        src = src[rng.permutation(n)]
        pool.sync()
    res = {"blocks": n, "nccl_version": N.version(), "pair": role.pair}

    def check(dst):
        # receiver: KV of dst block k must equal P's source block k; P sends its
        # first chunk of each block as the reference through the same comm
        ref = torch.empty(n, c, dtype=torch.uint8, device=f"cuda:{dev}")
        if role.kind == "P":
            comm.exchange(peer, chunk_ptrs(M.addr_indices(src))[:: 2 * L], [c] * n, peer, [],
                          [], st.cuda_stream)
            st.synchronize()
            return True
        comm.exchange(peer, [], [], peer, [ref.data_ptr() + k * c for k in range(n)], [c] * n,
                      st.cuda_stream)
        st.synchronize()
        got = pool._region.view(2 * L, nb, c)[0, torch.as_tensor(M.addr_indices(dst),
                                                                 device=f"cuda:{dev}")]
        return bool((got == ref).all())

    def run(name):
        dst = None
        if role.kind == "D":
            dst = pool.alloc_mem(n)
            pool.sync()
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        if name == "nccl_discrete_per_block":
            for k in range(n):
                if role.kind == "P":
                    comm.exchange(peer, chunk_ptrs([M.addr_indices(src)[k]]), [c] * (2 * L),
                                  peer, [], [], st.cuda_stream)
                else:
                    comm.exchange(peer, [], [], peer, chunk_ptrs([M.addr_indices(dst)[k]]),
                                  [c] * (2 * L), st.cuda_stream)
            st.synchronize()
        elif name == "nccl_aggregated":
            if role.kind == "P":
                pool.pack(src, 0, L, stg.data_ptr())
                pool.sync()
                comm.exchange(peer, [stg.data_ptr()], [n * Pb], peer, [], [], st.cuda_stream)
                st.synchronize()
            else:
                comm.exchange(peer, [], [], peer, [stg.data_ptr()], [n * Pb], st.cuda_stream)
                st.synchronize()
                pool.unpack(stg.data_ptr(), dst, 0, L)
                pool.sync()
        else:                                   # ours: the receiver allocates
            if role.kind == "P":
                pool.transfer(role.d_inst, src)
                pool.send_mark(role.d_inst, 7)
            else:
                pool.free_mem(dst)
                pool.serve(timeout_ms=120_000, until_mark=True)
                m = pool.recv_poll()
                dst = m[3]
                pool.sync()
        torch.cuda.synchronize()
        dist.barrier()
        dt = time.perf_counter() - t0
        ok = check(dst)
        if role.kind == "D":
            pool.free_mem(dst)
            pool.sync()
        return dt, ok

    for name in ("nccl_discrete_per_block", "nccl_aggregated", "ours"):
        ts, oks = [], []
        for r in range(4):
            dt, ok = run(name)
            oks.append(ok)
            if r:
                ts.append(dt)
        okv = [None] * world
        dist.all_gather_object(okv, all(oks))
        if not all(v for v in okv):
            raise RuntimeError(f"{name}: destination bytes differ")
        res[f"{name}_GBps"] = round(n * Pb / float(np.median(ts)) / 1e9, 1)
    res["what"] = ("2-rank NCCL communicator per pair, P_i -> D_i; wall clock between the "
                   "pair's barriers per synchronous transfer, median of 3; receiver bytes "
                   "checked each run")
    if role.kind == "P":
        pool.free_mem(src)
    comm.close()
    return res


def side_measurements(M, torch, shape, seed, peak, args, nccl_local=True):
    """Standalone pack / unpack (A4/A6, HBM roofline) per copy engine, and swap (A8/A9)."""
    out = {}
    Pb = shape.block_bytes
    n = 128   # 2048-token prompt = 1 GiB at 7B: 8x the 126 MB L2
    dev = torch.cuda.current_device()
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
                "avg_kernel_ms": round(kms, 4),
                "bytes_checked": pack_check(torch, X, shape, a, b, stg, name)}
        X.close()
        del stg, X
    if not args.no_swap:
        try:
            out["swap"] = swap_point(M, torch, shape, seed)
        except Exception as e:  # report, never hide
            out["swap"] = {"error": str(e)}
    if nccl_local:
        try:
            out["paper_transport_nccl"] = nccl_point(M, torch, shape, seed)
        except Exception as e:      # report, never hide
            out["paper_transport_nccl"] = {"error": str(e)}
    return out


def pack_check(torch, X, shape, a, b, stg, name):
    """Every byte of the side measurement's result, compared on the device
    with torch indexing of the pool's slabs (plain definition: staging block
    i = chunks (K_0, V_0, K_1, ...) of block a[i]; unpack: block b[i] = staging
    block i).  Raises on a mismatch."""
    M = sys.modules["paper_2406_17565_b200.mempool"]
    L2, c, nb = 2 * shape.layers, shape.chunk_bytes, X.hbm_blocks
    slab = X._region.view(L2, nb, c)
    dev = slab.device
    st = stg.view(len(a), L2, c)
    ids = torch.as_tensor(M.addr_indices(a if name == "pack" else b).astype(np.int64),
                          device=dev)
    X.sync()
    ok = bool((slab[:, ids].transpose(0, 1) == st).all())
    if not ok:
        raise RuntimeError(f"{name}: bytes differ from the plain gather")
    return "all bytes, device compare against torch indexing of the slabs"


def nccl_point(M, torch, shape, seed, n=128):
    """The paper's transport beside ours on the same 128 scattered blocks (a
    2048-token prompt): NCCL send/recv of every (layer, K/V) chunk, one
    group per block (the discrete layout), and of the aggregated
    staging (mp_pack -> one send -> mp_unpack), through a one-rank
    communicator (NCCL's self send/recv: the wire is this GPU's HBM), vs the
    fused mp_transfer.  Host clock per synchronous transfer, median of 3."""
    from paper_2406_17565_b200 import nccl_arm as N
    dev = torch.cuda.current_device()
    nb, c, L, Pb = 2 * n + 8, shape.chunk_bytes, shape.layers, shape.block_bytes
    P = make_pool(M, torch, 210, dev, shape, nb)
    D = make_pool(M, torch, 211, dev, shape, nb)
    M.connect(P, D)
    pv = P._region.view(2 * L, nb, c)
    dv = D._region.view(2 * L, nb, c)
    comm = N.NcclComm.create_single(dev)
    st = torch.cuda.current_stream()
    src = P.alloc_mem(n)
    P.debug_fill(src, seed)
    src = src[np.random.default_rng(seed).permutation(n)]
    P.sync()
    stg = torch.empty(2, n * Pb, dtype=torch.uint8, device=f"cuda:{dev}")
    res = {"blocks": n, "nccl_version": N.version()}

    def discrete(dst):
        for s, d in zip(M.addr_indices(src), M.addr_indices(dst)):
            sp = [pv.data_ptr() + (j * nb + int(s)) * c for j in range(2 * L)]
            dp = [dv.data_ptr() + (j * nb + int(d)) * c for j in range(2 * L)]
            comm.exchange(0, sp, [c] * (2 * L), 0, dp, [c] * (2 * L), st.cuda_stream)
        st.synchronize()
        return dst

    def aggregated(dst):
        P.pack(src, 0, L, stg[0].data_ptr())
        P.sync()
        comm.exchange(0, [stg[0].data_ptr()], [n * Pb], 0, [stg[1].data_ptr()], [n * Pb],
                      st.cuda_stream)
        st.synchronize()
        D.unpack(stg[1].data_ptr(), dst, 0, L)
        D.sync()
        return dst

    def fused(dst):
        D.free_mem(dst)
        return P.transfer(D.inst, src)

    for name, fn in (("nccl_discrete_per_block", discrete), ("nccl_aggregated", aggregated),
                     ("fused", fused)):
        ts = []
        for r in range(4):
            dst = D.alloc_mem(n)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dst = fn(dst)
            dt = time.perf_counter() - t0
            s_ids = torch.as_tensor(M.addr_indices(src), device=f"cuda:{dev}")
            d_ids = torch.as_tensor(M.addr_indices(dst), device=f"cuda:{dev}")
            if not bool((pv[0, s_ids] == dv[0, d_ids]).all()):
                raise RuntimeError(f"{name}: destination bytes differ")
            D.free_mem(dst)
            if r:
                ts.append(dt)
        res[f"{name}_GBps"] = round(n * Pb / float(np.median(ts)) / 1e9, 1)
    comm.close()
    P.close()
    D.close()
    return res


def swap_point(M, torch, shape, seed):
    """HBM <-> pinned DRAM (configs[4] shape): swap_out(n) then swap_in of the moved."""
    B, Pb = shape.block_tokens, shape.block_bytes
    nblk = 512
    dev = torch.cuda.current_device()
    S = make_pool(M, torch, 100, dev, shape, nblk, dram_blocks=nblk)
    rng = np.random.default_rng(seed)
    for i in range(8):
        t = rng.integers(3, 32000, size=48 * B, dtype=np.int32)
        a = S.alloc_mem(48)
        S.debug_fill(a, seed)
        S.insert(t, a)
    res = {}
    for n in (64, 256):
        t0 = time.perf_counter()
        old, new = S.swap_out(n)
        t1 = time.perf_counter()
        back = S.swap_in(new)
        t2 = time.perf_counter()
        res[f"n{n}"] = {"swap_out_GBps": round(len(old) * Pb / (t1 - t0) / 1e9, 2),
                        "swap_in_GBps": round(len(back) * Pb / (t2 - t1) / 1e9, 2),
                        "path": "default swap transport: double-buffered device staging "
                                "(pack / unpack of one half overlaps the copy-engine D2H / "
                                "H2D of the other, one copy per run of consecutive DRAM "
                                "blocks)",
                        "bound": "PCIe Gen5 x16 (pinned 1 GiB memcpy ~56 GB/s on this box)"}
    S.close()
    return res


# ------------------------------------------------------------ cpu baseline
class OracleArm:
    """The CPU oracle as it stands (materialised numpy byte path) on the same
    workload shape, bounded: a 7B-shaped pool of 160 blocks per instance
    (1.25 GiB each) and as many whole requests per step as fit a time budget."""

    def __init__(self):
        import oracle as O
        self.O = O
        self.host_cpus = os.cpu_count()
        try:
            aff = sorted(os.sched_getaffinity(0))
            self.affinity_cpus = len(aff)
            os.sched_setaffinity(0, {aff[0]})
            self.cores = 1
        except Exception:
            self.affinity_cpus = None
            self.cores = os.cpu_count()
        shape = LLAMA2_7B
        self.B, self.Pb = shape.block_tokens, shape.block_bytes
        self.nb = 160
        seed = seed_for(1)
        mk = lambda inst: O.OraclePool(inst, shape.layers, shape.kv_heads, shape.head_dim,
                                       self.B, self.nb, seed=seed, materialize=True)
        self.P, self.D = mk(0), mk(1)
        self.reqs = build_requests(shape, seed, int(self.nb * 0.8))
        self.srcs = []
        for sid, prompt in self.reqs:
            mt, matched = self.P.match(prompt)
            new = self.P.alloc_mem(-(-len(prompt) // self.B) - len(matched), O.HBM)
            self.P.fill(new)
            full = matched + new
            self.P.insert(prompt, full[: len(prompt) // self.B])
            self.srcs.append(full[len(prompt) // self.B:])
        self.next = 0

    def step(self, budget_s):
        O, B = self.O, self.B
        t0 = time.perf_counter()
        done, moved, n_req = [], 0, 0
        def retire():
            for prompt, part in done:
                self.D.free_mem(part)
                self.D.delete(prompt)
            done.clear()

        # whole passes over the request set until the budget is spent; D
        # retires each pass (as bench.py's D retires each batch)
        while time.perf_counter() - t0 < budget_s:
            (sid, prompt), partial = self.reqs[self.next], self.srcs[self.next]
            self.next = (self.next + 1) % len(self.reqs)
            _, matched = self.P.match(prompt)
            final, nm, _ = O.transfer_with_insert(self.P, self.D, prompt, matched + partial,
                                                  flags=O.FLAG_DEDUP)
            moved += nm
            n_req += 1
            done.append((prompt, final[len(prompt) // B:]))
            if self.next == 0:
                retire()
        retire()
        return moved, n_req, time.perf_counter() - t0

    def sample(self, n_req, steps):
        return (f"{n_req} ShareGPT-like requests over {steps} step(s), 7B shape, "
                f"{self.nb}-block pools, DEDUP P->D transfer_with_insert, numpy byte path")

    def describe(self):
        return {"cores": self.cores, "host_cpus": self.host_cpus,
                "affinity_cpus_before_pinning": self.affinity_cpus,
                "threads": "1 (pinned to the first CPU of the original affinity set; numpy "
                           "copies are single-threaded)",
                "normalization": ("per moved block: value = blocks moved x Pb (8 MiB) / CPU "
                                  "time.  The oracle's cost per block (an 8 MiB numpy copy + "
                                  "dict-based index ops on the same prompts) does not depend "
                                  "on the pool size, so the 160-block pools (1.25 GiB "
                                  "materialised each) stand for the 4096-block pools of the "
                                  "GPU run (32 GiB each, more than a bounded CPU sample can "
                                  "fill)")}


def cpu_baseline(seconds):
    arm = OracleArm()
    moved, n_req, t = arm.step(seconds)
    return {"value": round(moved * arm.Pb / t / 1e9, 4), "unit": "GB/s", "kind": "oracle",
            "sample": arm.sample(n_req, 1), **arm.describe()}


def run_reference(args, world):
    """--impl reference: the CPU oracle is this tier's reference arm."""
    arm = OracleArm()
    per_step = max(0.2, min(5.0, args.cpu_seconds / max(args.steps, 1)))
    for _ in range(args.warmup):
        arm.step(min(per_step, 1.0))
    moved = n_req = 0
    secs = 0.0
    for _ in range(args.steps):
        m, r, t = arm.step(per_step)
        moved, n_req, secs = moved + m, n_req + r, secs + t
    val = moved * arm.Pb / secs / 1e9
    print(json.dumps({
        "impl": "reference",
        "metric": METRIC, "value": round(val, 4), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(secs * 1e3 / max(args.steps, 1), 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": DTYPE, "data": "synthetic",
        "config": {"workload": WORKLOAD, "kv_dtype": KV_DTYPE,
                   "sample": "bounded sample of the workload per step (CPU oracle)"},
        "cpu_baseline": {"value": round(val, 4), "unit": "GB/s", "kind": "oracle",
                         "sample": arm.sample(n_req, args.steps), **arm.describe()},
        "e2e": {"value": round(val, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
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
    # testing the multi-process path on a 1-GPU box: every rank on --device,
    # gloo for the bootstrap / reductions (NCCL refuses two ranks on one GPU)
    ap.add_argument("--device", type=int, default=-1, help=argparse.SUPPRESS)
    ap.add_argument("--profile-every", type=int, default=8,
                    help="time every k-th migration launch with CUDA events (1: all)")
    ap.add_argument("--dist-backend", default="nccl", help=argparse.SUPPRESS)
    ap.add_argument("--xfer-path", default="fused", choices=list(PATHS),
                    help="transport of P -> D transfers (named in config.xfer_path)")
    ap.add_argument("--coalesce-mib", type=int, default=0,
                    help="payload limit of one coalesced migration launch (0: the library default, 4096 MiB; "
                         "-1: no coalescing)")
    ap.add_argument("--max-ctas", type=int, default=0,
                    help="cap the migration grid at this many CTAs (0: one full wave)")
    ap.add_argument("--peer-engine", type=int, default=0, choices=[0, 1, 2],
                    help="stores into peer memory: 0 auto, 1 vector LD/ST, 2 bulk cp.async")
    ap.add_argument("--peer-sched", type=int, default=0, choices=[0, 1, 2],
                    help="split of peer stores: 0 auto, 1 static, 2 dynamic claiming")
    ap.add_argument("--no-pipeline", action="store_true",
                    help="N>1: enqueue each copy inside its own call (no MP_XFER_PIPELINE)")
    ap.add_argument("--no-probe", action="store_true",
                    help="N>1: skip the in-run peer-copy probe (NVLink peak)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))

    if args.impl == "reference":
        if rank == 0:        # rank 0 alone runs it; the other ranks exit 0
            run_reference(args, world)
        return

    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist_mod
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)) if args.device < 0
                              else args.device)
        dist_mod.init_process_group(args.dist_backend)
        dist = dist_mod
    res = run_ours(args, rank, world, dist)
    if rank == 0:
        if not args.no_cpu_baseline and world == 1:   # the contract: rank 0 at N=1 only
            res["cpu_baseline"] = cpu_baseline(args.cpu_seconds)
        print(json.dumps(res))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

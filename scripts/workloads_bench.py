#!/usr/bin/env python
"""BASELINE.json configs[2] and configs[3] measured on one B200 (P and D as two
pools on cuda:0, loopback wire), same conventions as bench.py (CUDA events
around K sessions, the library's per-launch kernel timing, clocks sampled).

  loogle  configs[2]: Llama-2-13B KV (Pb = 12.5 MiB), LooGLE-like sessions --
          a 16-32K-token document and 5 questions; PD-Caching-2: every
          turn P -> D transfer_with_insert with DEDUP, so turn 1 moves the
          document (1024-2048 blocks, 12.5-25 GiB) and turns 2-5 only their
          new blocks.
  react   configs[3]: Llama-2-13B KV, ReAct-like sessions -- a shared 1536-token
          two-shot prefix, 3-6 steps of long generation;
          PD-Caching-3: P -> D (DEDUP) of the prompt, D appends the generated
          blocks, D -> P transfer_with_insert returns them (the suffix from
          block floor(prompt/B) on, R3).

value = payload bytes moved in both directions / time.  Prefill / decode
compute is out of scope (no model): blocks are allocated and indexed by the
stand-in engine steps, their KV bytes are whatever the pool holds.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import Clocks, cupti_busy, load_peaks, make_pool  # noqa: E402
from paper_2406_17565_b200 import mempool as M  # noqa: E402
from workloads import traces  # noqa: E402
from workloads.configs import LLAMA2_13B, seed_for  # noqa: E402

S = LLAMA2_13B
B = S.block_tokens
FLAGS = M.XFER_DEDUP | M.XFER_ASYNC
STREAM_ORDERED = True
RETAIN = False          # --retain: sessions stay cached; full pools evict (R8)


class Timed:
    """Proxy accumulating host time per pool method (--phase-times)."""
    acc = {}

    def __init__(self, pool):
        self._p = pool

    def __getattr__(self, name):
        f = getattr(self._p, name)
        if not callable(f):
            return f

        def w(*a, **k):
            t0 = time.perf_counter()
            r = f(*a, **k)
            d = Timed.acc.setdefault(name, [0, 0.0])
            d[0] += 1
            d[1] += time.perf_counter() - t0
            return r
        return w


_EV = None


def prefill(P, prompt):
    """Engine stand-in: match, allocate the rest (stream-ordered: the engine's
    stream waits on the pool's event before it would write the KV), retire
    the full blocks."""
    _, m = P.match(prompt)
    new = P.alloc_mem(-(-len(prompt) // B) - len(m), stream_ordered=STREAM_ORDERED)
    if STREAM_ORDERED:
        global _EV
        if _EV is None:
            _EV = (torch.cuda.Event(), torch.cuda.current_stream())
        P.record_event(_EV[0])
        _EV[1].wait_event(_EV[0])
    full = np.concatenate([m, new])
    P.insert(prompt, full[: len(prompt) // B])
    return full


TURN_EV = None   # list collecting (turn, start_event, end_event) when set


def loogle_session(P, D, sess):
    moved = 0
    prompts = []
    for ti, t in enumerate(sess.turns):
        src = prefill(P, t.prompt)
        if TURN_EV is not None:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            P.record_event(ev[0])
        final, nm = P.transfer_with_insert(D.inst, t.prompt, src, flags=FLAGS)
        if TURN_EV is not None:
            D.record_event(ev[1])
            TURN_EV.append((ti, nm, ev))
        moved += nm
        prompts.append((t.prompt, src[len(t.prompt) // B:], final[len(t.prompt) // B:]))
    for prompt, p_part, d_part in prompts:       # the session ends: both sides retire it
        P.free_mem(p_part)
        D.free_mem(d_part)
        if not RETAIN:
            P.delete(prompt)
            D.delete(prompt)
    return moved


def react_session(P, D, sess):
    return sum(react_steps(P, D, sess))


DIR = {"p2d_sent": 0, "p2d_moved": 0, "d2p_moved": 0}   # ReAct per-direction block counts


def react_steps(P, D, sess):
    """One ReAct session as a generator: yields the blocks moved per turn, so
    several sessions can be interleaved turn by turn (--concurrent)."""
    retire = []
    for t in sess.turns:
        moved = 0
        src = prefill(P, t.prompt)
        fin_d, nm = P.transfer_with_insert(D.inst, t.prompt, src, flags=FLAGS)
        moved += nm
        DIR["p2d_sent"] += len(src)
        DIR["p2d_moved"] += nm
        whole = np.concatenate([t.prompt, t.gen])
        k = len(t.prompt) // B
        D.free_mem(fin_d[k:])                                 # the prompt's partial block
        d_addrs = prefill(D, whole)                           # decode appends blocks
        fin_p, nm2 = D.transfer_with_insert(P.inst, whole, d_addrs[k:], flags=M.XFER_ASYNC)
        moved += nm2
        DIR["d2p_moved"] += nm2
        D.free_mem(d_addrs[len(whole) // B:])
        P.free_mem(fin_p[len(whole) // B:])                   # P's copy of whole's partial
        P.free_mem(src[k:])
        retire.append(whole)
        yield moved
    for whole in retire if not RETAIN else ():
        P.delete(whole)
        D.delete(whole)


def interleaved(P, D, sessions, k):
    """k ReAct sessions in flight, advanced one turn each in round robin (a
    serving loop with k concurrent agents); a finished one is replaced by
    the next session."""
    moved = 0
    pending = list(sessions)
    live = []
    while pending or live:
        while pending and len(live) < k:
            live.append(react_steps(P, D, pending.pop(0)))
        nxt = []
        for g in live:
            try:
                moved += next(g)
                nxt.append(g)
            except StopIteration:
                pass
        live = nxt
    return moved


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", choices=["loogle", "react"])
    ap.add_argument("--sessions", type=int, default=0)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--pool-blocks", type=int, default=4096)
    ap.add_argument("--drain-alloc", action="store_true",
                    help="engine allocations drain the pool (no MP_ALLOC_STREAM_ORDERED)")
    ap.add_argument("--phase-times", action="store_true",
                    help="host time per pool method in the timed loop (stderr)")
    ap.add_argument("--retain", action="store_true",
                    help="keep finished sessions cached (pools fill up and evict LRU leaves)")
    ap.add_argument("--prof", action="store_true", help="cProfile the timed loop (stderr)")
    ap.add_argument("--profile-every", type=int, default=4,
                    help="time every k-th migration launch (1: all; events cost a few us each)")
    ap.add_argument("--no-profile", action="store_true",
                    help="no per-launch timing events (kernel shares are then unavailable)")
    ap.add_argument("--cupti-sessions", type=int, default=8,
                    help="sessions of the untimed CUPTI pass (0: skip)")
    ap.add_argument("--concurrent", type=int, default=1,
                    help="react: sessions in flight, interleaved turn by turn")
    ap.add_argument("--max-ctas", type=int, default=0,
                    help="cap the migration grid (0: one full wave)")
    ap.add_argument("--coalesce-mib", type=int, default=0,
                    help="launch coalescing limit (0: library default 1 GiB, <0: off)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    global STREAM_ORDERED
    STREAM_ORDERED = not args.drain_alloc
    global RETAIN
    RETAIN = args.retain
    idx = 2 if args.workload == "loogle" else 3
    seed = seed_for(idx)
    if args.workload == "loogle":
        sessions = traces.loogle_like(seed, n_sessions=args.sessions or 8)
        fn = loogle_session
    else:
        sessions = traces.react_like(seed, n_sessions=args.sessions or 32)
        fn = react_session
    P = make_pool(M, torch, 0, 0, S, args.pool_blocks, coalesce_mib=args.coalesce_mib,
                  max_ctas=args.max_ctas)
    D = make_pool(M, torch, 1, 0, S, args.pool_blocks, coalesce_mib=args.coalesce_mib,
                  max_ctas=args.max_ctas)
    M.connect(P, D)
    clocks = Clocks("/tmp/clocks_wl.csv", 0)
    with clocks:
        time.sleep(1.0)
        for s in sessions[: args.warmup]:
            fn(P, D, s)
        for x in (P, D):
            x.sync()
            x.stats_reset()
            x.profile(not args.no_profile, every=args.profile_every)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for key in DIR:
            DIR[key] = 0
        e0.record()
        h0 = time.perf_counter()
        if args.prof:
            import cProfile
            import pstats
            pr = cProfile.Profile()
            pr.enable()
        if args.phase_times:
            moved = sum(fn(Timed(P), Timed(D), s) for s in sessions)
            for k, (n, t) in sorted(Timed.acc.items(), key=lambda kv: -kv[1][1]):
                print(f"{k:24s} calls {n:5d}  total {t * 1e3:8.3f} ms  per call {t / n * 1e6:7.1f} us",
                      file=sys.stderr)
        else:
            if args.workload == "react" and args.concurrent > 1:
                moved = interleaved(P, D, sessions, args.concurrent)
            else:
                moved = sum(fn(P, D, s) for s in sessions)
        if args.prof:
            pr.disable()
            pstats.Stats(pr, stream=sys.stderr).sort_stats("tottime").print_stats(15)
        host_ms = (time.perf_counter() - h0) * 1e3
        for x in (P, D):
            x.sync()
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    st = [x.stats() for x in (P, D)]
    dirs = dict(DIR)             # the timed region's counts (later passes add to DIR)
    turn_lat = None
    if args.workload == "loogle":
        # device time of each turn's transfer (untimed pass after the region,
        # events on the shared copy stream): turn 1 moves the document,
        # turns 2-5 only their new blocks (DEDUP)
        global TURN_EV
        TURN_EV = []
        for s in sessions[:4]:
            fn(P, D, s)
        for x in (P, D):
            x.sync()
        first = [a.elapsed_time(b) for ti, _, (a, b) in TURN_EV if ti == 0]
        rest = [a.elapsed_time(b) for ti, _, (a, b) in TURN_EV if ti > 0]
        nrest = [nm for ti, nm, _ in TURN_EV if ti > 0]
        turn_lat = {"turn1_document_ms_p50": round(float(np.median(first)), 3),
                    "turns2to5_incremental_ms_p10_p50_p90":
                        [round(float(np.percentile(rest, q)), 4) for q in (10, 50, 90)],
                    "turns2to5_blocks_moved_p50": float(np.median(nrest)),
                    "sessions": 4}
        TURN_EV = None
    # CUPTI pass (untimed, no events around launches): the migration kernels'
    # busy time (union of their intervals) and the HBM rate while busy
    cupti = None
    if args.cupti_sessions > 0:
        from torch.profiler import ProfilerActivity, profile
        for x in (P, D):
            x.sync()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            c0.record()
            cm = sum(fn(P, D, s) for s in sessions[: args.cupti_sessions])
            for x in (P, D):
                x.sync()
            c1.record()
            torch.cuda.synchronize()
        nl, tot, busy = cupti_busy(prof)
        pms = c0.elapsed_time(c1)
        cab = 2 * cm * S.block_bytes / (busy * 1e-6) / 1e9 if busy else None
        cupti = {"sessions": args.cupti_sessions, "launches": nl,
                 "avg_launch_us": round(tot / nl, 3) if nl else None,
                 "busy_ms": round(busy / 1e3, 3), "pass_ms": round(pms, 3),
                 "share_of_time": round(busy / 1e3 / pms, 4) if pms else None,
                 "achieved_over_busy_GBps": round(cab, 1) if cab else None,
                 "what": "CUPTI records (torch.profiler) of the migration kernels over an untimed "
                         "pass; achieved = 2 x payload / union of the kernels' intervals"}
    # sampled launches stand for every profiled one (per pool; ratio
    # estimator: kernel time per byte of the sampled launches x all bytes)
    kms = sum(s["kernel_ms"] * s["profiled_bytes"] / s["timed_bytes"]
              for s in st if s["timed_bytes"])
    kl = sum(s["profiled_launches"] for s in st)
    kb = sum(s["profiled_bytes"] for s in st)
    peak, src = load_peaks()
    if cupti and cupti["achieved_over_busy_GBps"]:
        cupti["frac_over_busy"] = round(cupti["achieved_over_busy_GBps"] / peak, 4)
    ach = 2 * kb / (kms * 1e-3) / 1e9 if kms else None
    print(json.dumps({
        "metric": "KV migration GB/s (payload, both directions)",
        "workload": f"configs[{idx}] {args.workload}-like, Llama-2-13B KV (Pb = 12.5 MiB), "
                    f"{len(sessions)} sessions, one B200 (P, D loopback)",
        "value": round(moved * S.block_bytes / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
        "blocks_per_s": round(moved / (ms * 1e-3), 1), "blocks_moved": int(moved),
        "ms": round(ms, 3),
        "roofline": {"bound": "hbm", "achieved": round(ach, 1) if ach else None, "peak": peak,
                     "peak_source": src, "frac": round(ach / peak, 4) if ach else None,
                     "launches": kl, "share_of_time": round(kms / ms, 4),
                     "timed_every": args.profile_every,
                     "host_ms": round(host_ms, 3)},
        "cupti": cupti,
        "turn_latency": turn_lat,
        "directions": ({"p_to_d_blocks_sent": dirs["p2d_sent"],
                        "p_to_d_blocks_moved": dirs["p2d_moved"],
                        "p_to_d_blocks_avoided_by_dedup": dirs["p2d_sent"] - dirs["p2d_moved"],
                        "d_to_p_blocks_moved": dirs["d2p_moved"]}
                       if args.workload == "react" else None),
        "engine_alloc": "drain" if args.drain_alloc else "stream_ordered",
        "sessions_retained": RETAIN,
        "clocks": clocks.summary()}))


if __name__ == "__main__":
    main()

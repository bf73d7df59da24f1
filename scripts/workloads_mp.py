#!/usr/bin/env python
"""BASELINE.json configs[2] and configs[3] at their GPU counts, one process
per GPU (torchrun), the same conventions as bench.py's N>1 line.

  loogle  configs[2]: Llama-2-13B KV (Pb = 12.5 MiB), LooGLE-like sessions --
          a 16-32K-token document and its questions -- 2P2D on 4 GPUs:
          every turn P_i -> D_i transfer_with_insert with DEDUP (PD-Caching-2,
          P:490-495), so turn 1 moves the document (1024-2048 blocks,
          12.5-25 GiB) and later turns only their new blocks.
  react   configs[3]: Llama-2-13B KV, ReAct-like sessions (a shared two-shot
          prefix, 3-6 steps of long generation) -- 4P4D on 8 GPUs,
          PD-Caching-3: P_i -> D_i of every prompt (DEDUP), D_i
          appends the generated blocks and returns them D_i -> P_i with a
          suffix transfer_with_insert (R3).  --window sessions are in flight
          per pair, so D_i's returns run while P_i sends the next prompts
          (full duplex over the pair's link).

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \\
        scripts/workloads_mp.py loogle
    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \\
        scripts/workloads_mp.py react
    (--device 0 --dist-backend gloo: every rank on one GPU, for testing)

Weak scaling: every pair runs its own seeded session list (seed_for(idx) +
1000 * pair).  value = payload bytes moved in both directions by all pairs /
the slowest rank's time (CUDA events from a barrier to its pools' final
sync).  Prefill / decode compute is out of scope (no model): the stand-in
engine allocates, fills (--check) and indexes blocks.

--check adds an untimed pass with content verification: the sender fills its
new blocks (mp_debug_fill), ships per-block checksums of every source block in
the transfer's `private` bytes, and the receiver checksums the blocks it got
(DEDUP-kept ones included) -- every transferred block of that pass is compared.
"""
import argparse
import json
import os
import struct
import sys
import time
from collections import deque

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import Clocks, make_pool  # noqa: E402
from paper_2406_17565_b200 import mempool as M  # noqa: E402
from paper_2406_17565_b200.topology import role_of  # noqa: E402
from workloads import traces  # noqa: E402
from workloads.configs import LLAMA2_13B, seed_for  # noqa: E402

S = LLAMA2_13B
B = S.block_tokens
NVLINK_GBS = 900.0


class Engine:
    """Stand-in for one instance's serving engine around its pool."""

    def __init__(self, pool, dev, check, fill_seed):
        self.p = pool
        self.dev = dev
        self.check = check
        self.fill_seed = fill_seed
        self.ev = torch.cuda.Event()
        self.st = torch.cuda.current_stream()
        self.moved = 0
        self.checked = 0
        self.bad = 0
        if check:
            L2, nb, c = 2 * S.layers, pool.hbm_blocks, S.chunk_bytes
            self.view = pool._region.view(L2, nb, c).view(torch.int64)
            g = torch.Generator(device=f"cuda:{dev}").manual_seed(5)
            self.w = torch.randint(-2**31, 2**31, (c // 8,), generator=g, device=f"cuda:{dev}")

    def prefill(self, prompt):
        """match, allocate the rest stream-ordered (the engine's stream waits on
        the pool's event before it would write), retire the full blocks."""
        _, m = self.p.match(prompt)
        new = self.p.alloc_mem(-(-len(prompt) // B) - len(m), stream_ordered=not self.check)
        if self.check and len(new):
            self.p.debug_fill(new, self.fill_seed)
        else:
            self.p.record_event(self.ev)
            self.st.wait_event(self.ev)
        full = np.concatenate([m, new])
        self.p.insert(prompt, full[: len(prompt) // B])
        return full

    def sums(self, addrs):
        """Per-block checksums (weighted int64 sums of every chunk) on the device."""
        if not self.check or len(addrs) == 0:
            return b""
        self.p.sync()
        t = torch.as_tensor(M.addr_indices(addrs).astype(np.int64), device=f"cuda:{self.dev}")
        out = torch.stack([(self.view[j][t] * self.w).sum(-1) for j in range(self.view.shape[0])],
                          1)
        return out.cpu().numpy().tobytes()

    def verify(self, addrs, ref):
        if not self.check:
            return
        got = self.sums(addrs)
        n = len(ref) // (8 * 2 * S.layers)
        self.checked += n
        a = np.frombuffer(got, np.int64).reshape(-1, 2 * S.layers)[-n:] if n else None
        b = np.frombuffer(ref, np.int64).reshape(-1, 2 * S.layers)
        if n and not np.array_equal(a, b):
            self.bad += int((a != b).any(1).sum())

    PIPELINE = M.XFER_PIPELINE

    def send(self, dst, tokens, src, flags, head):
        """transfer_with_insert with `private` = header + checksums of src;
        ASYNC sends are pipelined (the copy is enqueued at the next call)."""
        if flags & M.XFER_ASYNC:
            flags |= self.PIPELINE
        priv = head + self.sums(src)
        fin, nm = self.p.transfer_with_insert(dst, tokens, src, flags=flags, priv=priv)
        self.moved += nm
        return fin

    def messages(self):
        out = []
        while True:
            m = self.p.recv_poll()
            if m is None:
                return out
            out.append(m)


# ------------------------------------------------------------------ loogle
def loogle_p(E, role, sessions):
    for s in sessions:
        parts, prompts = [], []
        for ti, t in enumerate(s.turns):
            src = E.prefill(t.prompt)
            E.send(role.d_inst, t.prompt, src, M.XFER_DEDUP | M.XFER_ASYNC,
                   struct.pack("<ii", s.sid, ti))
            parts.append(src[len(t.prompt) // B:])
            prompts.append(t.prompt)
        for prompt, part in zip(prompts, parts):        # the session ends
            E.p.free_mem(part)
            E.p.delete(prompt)
        E.p.send_mark(role.d_inst, s.sid)


def loogle_d(E, role, sessions):
    for s in sessions:
        _served, mark = E.p.serve(timeout_ms=600_000, until_mark=True)
        if mark != s.sid:
            raise RuntimeError(f"D: expected mark {s.sid}, got {mark}")
        for kind, _src, priv, addrs in E.messages():
            sid, ti = struct.unpack_from("<ii", priv)
            prompt = s.turns[ti].prompt
            E.verify(addrs, priv[8:])
            E.p.free_mem(addrs[len(prompt) // B:])
            E.p.delete(prompt)


# ------------------------------------------------------------------- react
DONE_TAG = 1 << 30


def react_p(E, role, sessions, window):
    """Keeps `window` sessions in flight: issues the next prompt of a session
    as soon as its previous step came back from D (full duplex with D's
    returns of the others)."""
    pending = deque(sessions)
    live = {}                         # sid -> [session, turn index, P's partial src]
    ready = deque()
    sent_turns = 0
    while pending or live:
        while pending and len(live) < window:
            s = pending.popleft()
            live[s.sid] = [s, 0, None]
            ready.append(s.sid)
        while ready:
            sid = ready.popleft()
            s, ti, _ = live[sid]
            t = s.turns[ti]
            src = E.prefill(t.prompt)
            E.send(role.d_inst, t.prompt, src, M.XFER_DEDUP | M.XFER_ASYNC,
                   struct.pack("<ii", sid, ti))
            live[sid][2] = src[len(t.prompt) // B:]
            sent_turns += 1
        E.p.serve(timeout_ms=0, until_mark=False)        # D -> P returns
        for kind, _src, priv, addrs in E.messages():
            sid, ti = struct.unpack_from("<ii", priv)
            s, _, part = live[sid]
            t = s.turns[ti]
            whole = np.concatenate([t.prompt, t.gen])
            E.verify(addrs[len(t.prompt) // B:], priv[8:])
            E.p.free_mem(addrs[len(whole) // B:])          # P's partial of the return
            E.p.free_mem(part)                             # P's partial of the prompt
            if ti + 1 < len(s.turns):
                live[sid][1] = ti + 1
                ready.append(sid)
            else:                                          # the session ends
                for u in s.turns:
                    E.p.delete(np.concatenate([u.prompt, u.gen]))
                del live[sid]
    E.p.send_mark(role.d_inst, DONE_TAG)
    return sent_turns


def react_d(E, role, sessions):
    by_sid = {s.sid: s for s in sessions}
    while True:
        _served, mark = E.p.serve(timeout_ms=0, until_mark=True)
        for kind, _src, priv, addrs in E.messages():
            sid, ti = struct.unpack_from("<ii", priv)
            s = by_sid[sid]
            t = s.turns[ti]
            E.verify(addrs, priv[8:])
            k = len(t.prompt) // B
            E.p.free_mem(addrs[k:])                        # the prompt's partial block
            whole = np.concatenate([t.prompt, t.gen])
            d = E.prefill(whole)                           # decode appends blocks
            E.send(role.p_inst, whole, d[k:], M.XFER_ASYNC, struct.pack("<ii", sid, ti))
            E.p.free_mem(d[len(whole) // B:])
            if ti + 1 == len(s.turns):
                for u in s.turns:
                    E.p.delete(np.concatenate([u.prompt, u.gen]))
        if mark == DONE_TAG:
            return


def run_pass(E, role, wl, sessions, window):
    if wl == "loogle":
        (loogle_p if role.kind == "P" else loogle_d)(E, role, sessions)
    elif role.kind == "P":
        react_p(E, role, sessions, window)
    else:
        react_d(E, role, sessions)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", choices=["loogle", "react"])
    ap.add_argument("--sessions", type=int, default=0, help="per pair")
    ap.add_argument("--warmup", type=int, default=1, help="warm-up sessions per pair")
    ap.add_argument("--pool-blocks", type=int, default=4096)
    ap.add_argument("--window", type=int, default=4, help="react: sessions in flight per pair")
    ap.add_argument("--doc-hi", type=int, default=32768, help="loogle: longest document")
    ap.add_argument("--check", action="store_true",
                    help="untimed verification pass (checksums of every transferred block)")
    ap.add_argument("--check-sessions", type=int, default=2)
    ap.add_argument("--prof", action="store_true", help="cProfile the timed pass (stderr)")
    ap.add_argument("--no-pipeline", action="store_true",
                    help="enqueue each copy inside its own call (no MP_XFER_PIPELINE)")
    ap.add_argument("--device", type=int, default=-1)
    ap.add_argument("--dist-backend", default="nccl")
    args = ap.parse_args()

    if args.no_pipeline:
        Engine.PIPELINE = 0
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if world < 2:
        raise SystemExit("run under torchrun with an even number of processes "
                         "(scripts/workloads_bench.py is the one-GPU loopback driver)")
    import torch.distributed as dist
    dev = int(os.environ.get("LOCAL_RANK", 0)) if args.device < 0 else args.device
    torch.cuda.set_device(dev)
    dist.init_process_group(args.dist_backend)
    role = role_of(rank, world)
    idx = 2 if args.workload == "loogle" else 3
    seed = seed_for(idx) + 1000 * role.pair
    if args.workload == "loogle":
        n = args.sessions or 4
        sessions = traces.loogle_like(seed, n_sessions=n + args.warmup + args.check_sessions,
                                      doc_hi=args.doc_hi)
    else:
        n = args.sessions or 32
        sessions = traces.react_like(seed, n_sessions=n + args.warmup + args.check_sessions)
    warm = sessions[: args.warmup]
    timed = sessions[args.warmup: args.warmup + n]
    checked = sessions[args.warmup + n:]

    inst = role.p_inst if role.kind == "P" else role.d_inst
    pool = make_pool(M, torch, inst, dev, S, args.pool_blocks)
    blobs = M.exchange_handles(pool)
    pool.import_peer(blobs[role.partner][1])
    dist.barrier()
    E = Engine(pool, dev, False, seed)

    clocks = Clocks(f"/tmp/clocks_wmp_{rank}.csv", dev)
    with clocks:
        time.sleep(1.0)
        run_pass(E, role, args.workload, warm, args.window)
        pool.sync()
        torch.cuda.synchronize()
        pool.stats_reset()
        pool.profile(True, every=4)
        E.moved = 0
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h0 = time.perf_counter()
        if args.prof:
            import cProfile
            import pstats
            pr = cProfile.Profile()
            pr.enable()
        run_pass(E, role, args.workload, timed, args.window)
        if args.prof:
            pr.disable()
            print(f"---- rank {rank} ({role.kind})", file=sys.stderr)
            pstats.Stats(pr, stream=sys.stderr).sort_stats("tottime").print_stats(12)
        pool.sync()
        e1.record()
        torch.cuda.synchronize()
        host_ms = (time.perf_counter() - h0) * 1e3
        dist.barrier()
    ms = e0.elapsed_time(e1)
    st = pool.stats()
    pool.profile(False)
    moved = E.moved

    chk = None
    if args.check and checked:
        C = Engine(pool, dev, True, seed + 1)
        run_pass(C, role, args.workload, checked, args.window)
        pool.sync()
        chk = {"rank": rank, "checked_blocks": C.checked, "bad_blocks": C.bad}

    kms = (st["kernel_ms"] * st["profiled_bytes"] / st["timed_bytes"]) if st["timed_bytes"] else 0
    rec = {"rank": rank, "kind": role.kind, "pair": role.pair, "moved": moved, "ms": ms,
           "host_ms": host_ms, "kernel_ms": kms, "launches": st["profiled_launches"],
           "kernel_GBps": (st["timed_bytes"] / (st["kernel_ms"] * 1e-3) / 1e9
                           if st["kernel_ms"] else None),
           "check": chk, "clocks": clocks.summary()}
    recs = [None] * world
    dist.all_gather_object(recs, rec)
    if rank == 0:
        Pb = S.block_bytes
        tmax = max(r["ms"] for r in recs)
        tot = sum(r["moved"] for r in recs)
        per_pair = []
        for i in range(world // 2):
            p = next(r for r in recs if r["kind"] == "P" and r["pair"] == i)
            d = next(r for r in recs if r["kind"] == "D" and r["pair"] == i)
            e = {"pair": i, "p_rank": p["rank"], "d_rank": d["rank"]}
            for nm, r in (("p_to_d", p), ("d_to_p", d)):
                g = r["moved"] * Pb / (r["ms"] * 1e-3) / 1e9
                e[nm] = {"blocks": r["moved"], "GBps": round(g, 1),
                         "frac_of_nominal_900": round(g / NVLINK_GBS, 4),
                         "kernel_GBps": round(r["kernel_GBps"], 1) if r["kernel_GBps"] else None,
                         "kernel_share_of_time": round(r["kernel_ms"] / r["ms"], 4),
                         "launches": r["launches"]}
            per_pair.append(e)
        checks = [r["check"] for r in recs if r["check"]]
        print(json.dumps({
            "metric": "KV migration GB/s (payload, both directions)",
            "workload": (f"configs[{idx}] {args.workload}-like, Llama-2-13B KV (Pb = 12.5 MiB), "
                         f"{len(timed)} sessions per pair"
                         + (f", {args.window} in flight" if args.workload == "react" else "")),
            "n_gpus": world, "placement": f"{world // 2}P{world // 2}D, one process per GPU"
                                         + (f" (all on GPU {args.device})"
                                            if args.device >= 0 else ""),
            "value": round(tot * Pb / (tmax * 1e-3) / 1e9, 2), "unit": "GB/s",
            "blocks_per_s": round(tot / (tmax * 1e-3), 1), "blocks_moved": int(tot),
            "ms": round(tmax, 3), "scaling": "weak",
            "pipelined_issue": not args.no_pipeline,
            "host_ms_max": round(max(r["host_ms"] for r in recs), 3),
            "per_pair": per_pair,
            "check": ({"blocks_checked": sum(c["checked_blocks"] for c in checks),
                       "bad_blocks": sum(c["bad_blocks"] for c in checks),
                       "what": "receiver checksums of every transferred block vs the sender's "
                               "(untimed pass)"} if args.check else None),
            "clocks": recs[0]["clocks"]}))
    dist.barrier()
    pool.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

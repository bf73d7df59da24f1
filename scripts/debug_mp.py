#!/usr/bin/env python
"""Run one two-process GPU test worker pair standalone with MP_REMOTE_TRACE=1
(stall diagnostics) and per-process tracebacks after a timeout.
    python scripts/debug_mp.py golden ce-staged [dedup]"""
import faulthandler
import multiprocessing as mp
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(kind, rank, port, q, transport, dedup):
    faulthandler.dump_traceback_later(60, exit=False)
    import tests.test_gpu_multiproc as T
    if kind == "golden":
        T._run(rank, port, dedup, q, transport)
    else:
        T._react_worker(rank, port, 47, q, transport)


if __name__ == "__main__":
    os.environ["MP_REMOTE_TRACE"] = "1"
    kind, transport = sys.argv[1], sys.argv[2]
    dedup = len(sys.argv) > 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(kind, r, 29871, q, transport, dedup)) for r in range(2)]
    for p in ps:
        p.start()
    for _ in ps:
        try:
            r, out = q.get(timeout=90)
            print("rank", r, "error" if "error" in out else "ok", out.get("error", "")[:2000])
        except Exception as e:
            print("timeout", e)
            break
    for p in ps:
        p.kill()

#!/usr/bin/env python
"""Extended randomized parity campaign (test infrastructure, run by hand on a
GPU box; not collected by pytest): the random-op sequences of
tests/test_gpu_parity.py over many more seeds than the suite runs, every
transport x copy engine x coalescing mode x pool count, each op compared with
the oracle (results, errors, index dumps, block states, device bitmap, bytes).
  python tests/parity_campaign.py [n_seeds] > campaign.json"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2406_17565_b200 import mempool as M  # noqa: E402
from tests import test_gpu_parity as T  # noqa: E402
from workloads.configs import TINY, KVShape  # noqa: E402

n_seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 8
modes = [
    ("fused", M.PATH_FUSED, {}),
    ("fused_async", M.PATH_FUSED | M.XFER_ASYNC, {}),
    ("fused_async_sizeonly_3pools", M.PATH_FUSED | M.XFER_ASYNC, {"coalesce_mib": 1, "n_pools": 3}),
    ("fused_async_nocoalesce", M.PATH_FUSED | M.XFER_ASYNC, {"coalesce_mib": -1}),
    ("fused_vector", M.PATH_FUSED, {"copy_kernel": 1}),
    ("fused_bulk_async", M.PATH_FUSED | M.XFER_ASYNC, {"copy_kernel": 2}),
    ("staged", M.PATH_STAGED, {}),
    ("ce", M.PATH_CE, {}),
    ("fused_swap_zerocopy", M.PATH_FUSED, {"swap_flags": M.SWAP_ZERO_COPY}),
    # DRAM-resident sources through round 1's zero-copy kernel instead of the
    # copy engine + staging scatter (env knob, read per call)
    ("fused_async_dram_sm", M.PATH_FUSED | M.XFER_ASYNC, {"env": {"MP_DRAM_SOURCE": "sm"}}),
    ("fused_async_small_staging", M.PATH_FUSED | M.XFER_ASYNC,
     {"staging_blocks": 2}),
]
# chunk shapes: tiny (4 KiB), ragged (1152 B: predicated tails), multi-piece
# (45056 B = 2.75 bulk pieces / 11 vector units)
shapes = [("tiny", TINY), ("ragged", KVShape("ragged", 3, 3, 24, 8)),
          ("multipiece", KVShape("mp", 2, 16, 88, 16))]
out = {"seeds_per_mode": n_seeds, "ops_per_sequence": 300, "modes": {}}
for sname, shape in shapes:
    for name, path, kw in modes:
        if sname != "tiny" and "swap" in name:
            continue
        kw = dict(kw)
        env = kw.pop("env", {})
        if "staging_blocks" in kw:   # two one-block slots: every DRAM-source slot alternates
            nb = kw.pop("staging_blocks")
            kw.update(staging_bytes=nb * shape.block_bytes, staging_slots=nb)
        os.environ.update(env)
        t0 = time.time()
        for s in range(n_seeds):
            T.random_ops(10_000 + 97 * s, shape, 300, path, **kw)
        for k in env:
            os.environ.pop(k)
        out["modes"][f"{sname}/{name}"] = {"sequences": n_seeds, "status": "bit-exact",
                                           "seconds": round(time.time() - t0, 1)}
        print(sname, name, "ok", file=sys.stderr)
out["sequences_total"] = sum(m["sequences"] for m in out["modes"].values())
print(json.dumps(out, indent=1))

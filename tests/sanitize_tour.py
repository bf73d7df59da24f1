#!/usr/bin/env python
"""A short tour of every kernel and transport for compute-sanitizer
(memcheck / racecheck / synccheck): golden run on each transport, random ops
with both copy engines and coalescing, swap, pack/unpack, head-range copies.
Checked against the oracle as it goes (tests/twin.py)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))  # tests/ -> repo root
sys.path.insert(0, ROOT)

from paper_2406_17565_b200 import mempool as M  # noqa: E402
from tests import test_gpu_alloc_claims as AC  # noqa: E402
from tests import test_gpu_parity as T  # noqa: E402
from workloads.configs import TINY  # noqa: E402

for path in (M.PATH_FUSED, M.PATH_STAGED, M.PATH_CE, M.PATH_FUSED | M.XFER_ASYNC):
    for dedup in (False, True):
        T.test_golden_tiny(dedup, path)
T.test_golden_swap_evict()
T.test_private_and_transfer_layers()
for ck in (1, 2):
    T.random_ops(5, TINY, 120, M.PATH_FUSED | M.XFER_ASYNC, copy_kernel=ck)
    T.random_ops(6, TINY, 80, M.PATH_STAGED, copy_kernel=ck)
T.test_pack_unpack_np_take()
AC.test_claims_cancel_and_overflow_against_device_scan()
AC.test_pending_list_bound_flushes()
print("sanitize tour: ok")

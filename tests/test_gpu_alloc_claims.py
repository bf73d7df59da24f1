"""The device bitmap allocator under deferred claims (include/mempool.h,
mp_alloc_mem): a caller's alloc_mem is decided by the host shadow and its
claim reaches the device bitmap only with the next stream-ordered update,
while a transfer's receiver allocates on the device (lowest-first scan, R2).
Seeded sequences drive every case of that bookkeeping -- claims and frees
that cancel before they are applied, more pending updates than fit in a
launch's parameters (the id-arena upload), the pending list's host-side
compaction -- and every receiver allocation is compared with the oracle's
lowest-first choice, then the device bitmap with the oracle's free set."""
import numpy as np
import pytest

from tests.twin import Twin, connect, transfer
from workloads.configs import TINY

pytestmark = pytest.mark.gpu

N = 8192          # blocks per pool (tiny shape: 16 KiB each)


def test_claims_cancel_and_overflow_against_device_scan():
    rng = np.random.default_rng(2406)
    P, D = Twin(0, TINY, 512), Twin(1, TINY, N)
    connect(P, D)
    src = P.alloc(64)
    P.fill(src)
    held = []                                   # D's caller-owned blocks (oracle addrs)
    for step in range(40):
        op = rng.integers(0, 4)
        if op == 0 or not held:                 # big caller allocation: deferred claims
            k = int(rng.integers(1, 2600))
            if k <= D.o.free_count(0):
                held += D.alloc(k, stream_ordered=bool(rng.integers(0, 2)))
        elif op == 1:                           # free a random part (cancels unapplied claims)
            take = rng.random(len(held)) < rng.uniform(0.1, 0.9)
            D.free([a for a, t in zip(held, take) if t])
            held = [a for a, t in zip(held, take) if not t]
        elif op == 2:                           # reuse just-freed ids (cancels unapplied frees)
            k = int(rng.integers(1, 300))
            if held:
                back = held[-k:]
                held = held[:-k]
                D.free(back)
                held += D.alloc(len(back), stream_ordered=True)
        else:                                   # receiver allocation on the device
            n = int(rng.integers(1, 64))
            if n <= D.o.free_count(0):
                held += transfer(P, D, src[:n])
        if step % 10 == 9:
            D.check_state(check_bytes=False)
    D.check_state(check_bytes=False)
    D.check_bytes(sample=64, rng=rng)


def test_pending_list_bound_flushes():
    """Thousands of claims pending (past the queue's compaction bound): the
    queue is compacted on the host, and the device scan afterwards applies
    every claim and free (through the id arena) and still sees each one."""
    P, D = Twin(0, TINY, 64), Twin(1, TINY, N)
    connect(P, D)
    src = P.alloc(32)
    P.fill(src)
    a = D.alloc(2500, stream_ordered=True)
    b = D.alloc(2500, stream_ordered=True)      # 5000 pending: compacted on the host
    D.free(a[::3])                              # frees of applied claims
    got = transfer(P, D, src)                   # device scan: lowest free ids
    assert sorted(x[2] for x in got) == sorted(x[2] for x in a[::3])[:32]
    D.free(b)
    D.check_state(check_bytes=False)


def test_host_compaction_of_a_long_claim_queue():
    """A small receiver cycled through many stream-ordered alloc / free
    rounds with no device scan in between: the pending queue passes its bound
    (4 x kInlineIds + 2 x blocks) several times and is compacted on the host
    (no kernel); the next device scans still pick the oracle's lowest-first
    ids and the bitmap equals the oracle's free set."""
    rng = np.random.default_rng(17)
    P, D = Twin(0, TINY, 128), Twin(1, TINY, 64)
    connect(P, D)
    src = P.alloc(16)
    P.fill(src)
    held = []
    for rnd in range(6):
        for _ in range(150):                    # ~300 queue entries per 150 cycles
            k = int(rng.integers(1, 8))
            if k <= D.o.free_count(0):
                held += D.alloc(k, stream_ordered=True)
            if held:
                take = rng.random(len(held)) < 0.5
                D.free([a for a, t in zip(held, take) if t])
                held = [a for a, t in zip(held, take) if not t]
        n = int(rng.integers(1, 16))
        if n <= D.o.free_count(0):
            held += transfer(P, D, src[:n])     # device scan after the compactions
        D.check_state(check_bytes=False)

"""bench.py's contract pieces that run without a GPU: the reference arm
(`--impl reference`: the CPU oracle, this tier's reference) prints exactly one
JSON line with the driver's keys, on one process and under a world_size-2
launch (rank 0 alone runs and prints, the other rank exits 0 without work)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
        "cpu_baseline", "e2e"}


def _lines(out):
    return [l for l in out.splitlines() if l.startswith("{")]


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--cpu-seconds", "1"], cwd=ROOT, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert KEYS <= set(d)
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["dtype"] == "u16" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_two_ranks_rank0_prints():
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", str(29700 + os.getpid() % 50), "bench.py", "--impl",
                        "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
                        "--cpu-seconds", "1"], cwd=ROOT, capture_output=True, text=True,
                       timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1
    assert json.loads(lines[0])["n_gpus"] == 2


def _pair_worker(rank, world, port, q):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    from paper_2406_17565_b200.topology import role_of
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    role = role_of(rank, world)
    # what run_ours gathers: P ranks moved 100*(pair+1) blocks in 10 ms and
    # probed 700 GB/s; D ranks moved nothing (the copies run on the sender)
    rec = {"rank": rank, "kind": role.kind, "pair": role.pair, "partner": role.partner,
           "moved": 100 * (role.pair + 1) if role.kind == "P" else 0, "ms": 10.0,
           "kernel_GBps": 600.0 if role.kind == "P" else None,
           "probe": {"GBps": 700.0} if role.kind == "P" else None}
    recs = [None] * world
    dist.all_gather_object(recs, rec)
    q.put((rank, bench.pair_table(recs, 1 << 23)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_per_pair_table_gloo(world):
    """bench.py's N>1 per-pair table over a gloo world: one entry per pair,
    P_i on rank i -> D_i on rank i+N/2, each pair's own payload / its own time,
    and the fractions against 900 GB/s and the pair's probe."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29900 + (os.getpid() % 50) + world
    ps = [ctx.Process(target=_pair_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    half = world // 2
    for r in range(world):
        tab = res[r]
        assert [e["pair"] for e in tab] == list(range(half))
        for e in tab:
            i = e["pair"]
            assert (e["p_rank"], e["d_rank"], e["direction"]) == (i, i + half, "P->D")
            gbs = 100 * (i + 1) * (1 << 23) / 10e-3 / 1e9
            assert e["GBps"] == round(gbs, 1)
            assert e["frac_of_nominal_900"] == round(gbs / 900.0, 4)
            assert e["frac_of_probe"] == round(gbs / 700.0, 4)
            assert e["kernel_frac_of_probe"] == round(600.0 / 700.0, 4)


def test_cupti_busy_union_of_intervals():
    """bench.cupti_busy: launches, summed duration and the UNION of the
    kernels' [start, end) intervals (overlapping PDL grids count once; other
    kernels and host events are ignored)."""
    sys.path.insert(0, ROOT)
    import bench
    from torch.autograd import DeviceType

    class R:
        def __init__(self, a, b):
            self.start, self.end = a, b

    class E:
        def __init__(self, name, a, b, dev=DeviceType.CUDA):
            self.name, self.time_range, self.device_type = name, R(a, b), dev

    class P:
        def events(self):
            return [E("migrate_bulk_kernel<65536>", 0, 10), E("migrate_bulk_kernel<16384>", 8, 12),
                    E("migrate_kernel", 20, 25), E("alloc_kernel", 12, 30),
                    E("migrate (host op)", 0, 100, DeviceType.CPU), E("migrate_empty", 40, 40)]

    n, tot, busy = bench.cupti_busy(P())
    assert (n, tot, busy) == (3, 10 + 4 + 5, 12 + 5)
    n, tot, busy = bench.cupti_busy(P(), None)
    assert (n, tot, busy) == (4, 37, 30)

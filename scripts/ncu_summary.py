"""Summarise ncu outputs (run here, no GPU): launch-list shares per kernel and
the key counters of a --set full capture.  Usage:
  python scripts/ncu_summary.py launches <launches.csv>
  python scripts/ncu_summary.py full <prof.ncu-rep>
  python scripts/ncu_summary.py traffic <out.json> vector=<rep> bulk=<rep> [note]
"""
import json
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__waves_per_multiprocessor", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "l1tex__t_bytes.sum"]


def launches(path):
    txt = open(path).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
    agg = collections.defaultdict(list)
    for r in rows:
        if r["Metric Name"] == "gpu__time_duration.sum":
            agg[r["Kernel Name"].split("(")[0]].append(float(r["Metric Value"]))
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':60s} {'launches':>8s} {'avg_us':>9s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k[:60]:60s} {len(v):8d} {sum(v) / len(v) / 1e3:9.2f} {sum(v) / tot:7.4f}")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")][:70] if "Kernel Name" in hdr else "?"
        print("kernel:", name)
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:60s} {r[i]:>16s} {units[i]}")


def _raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def _mb(v, unit):
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}[unit]
    return float(v.replace(",", "")) * scale


def _us(v, unit):
    return float(v.replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[unit]


def traffic(out_path, *specs):
    """DRAM traffic vs the algorithmic bytes of every captured migrate launch:
    algorithmic = what the kernel requested (L2 sectors from the SMs, read +
    write: lts__t_sectors_srcunit_tex_op_{read,write} x 32 B = 2 x payload);
    traffic = dram__bytes_{read,write}."""
    res = {"source": " ".join(a for a in specs if "=" not in a) or
           "ncu --set full --clock-control none, bench.py --steps 2 (one transfer_with_insert per "
           "launch under ncu's serialisation)"}
    for spec in specs:
        if "=" not in spec:
            continue
        label, path = spec.split("=", 1)
        rows, units = _raw(path)
        lst = []
        for r in rows:
            rd = _mb(r["dram__bytes_read.sum"], units["dram__bytes_read.sum"])
            wr = _mb(r["dram__bytes_write.sum"], units["dram__bytes_write.sum"])
            # bytes the kernel itself requested from L2 (TMA / LSU), read + write
            tr = float(r["lts__t_sectors_srcunit_tex_op_read.sum"].replace(",", "")) * 32e-6
            tw = float(r["lts__t_sectors_srcunit_tex_op_write.sum"].replace(",", "")) * 32e-6
            alg = tr + tw
            lst.append({"kernel": r.get("Kernel Name", "?")[:60],
                        "duration_us": _us(r["gpu__time_duration.sum"],
                                           units["gpu__time_duration.sum"]),
                        "dram_read_MB": rd, "dram_write_MB": wr, "algorithmic_MB": round(alg, 3),
                        "sm_read_MB": round(tr, 3), "sm_write_MB": round(tw, 3),
                        "traffic_MB": rd + wr,
                        "traffic_over_algorithmic": round((rd + wr) / alg, 4)})
        res[label] = lst
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        traffic(*sys.argv[2:])
        sys.exit(0)
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])

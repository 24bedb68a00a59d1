"""Summaries of ncu captures for profiles/ (run here, on the CPU box).

    python scripts/ncu_summarize.py launches LAUNCHES.csv OUT.json   # share of step time per kernel
    python scripts/ncu_summarize.py full REPORT.ncu-rep OUT.json      # per-launch counters of a --set full capture

`launches`: the `--metrics gpu__time_duration.sum` launch list (cold-cache,
serialised: compare shares, not absolutes).  `full`: dram bytes, tensor-pipe and
memory throughput, registers, achieved occupancy per captured launch.
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

NCU = "/usr/local/cuda/bin/ncu"


def short(name):
    name = name.replace("bm::tc::", "").replace("bm::", "").replace("(anonymous namespace)::", "")
    return name.split("(")[0]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    per = defaultdict(lambda: [0, 0.0])
    total = 0.0
    n = 0
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "nsecond"
        ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
        k = short(r[ki])
        per[k][0] += 1
        per[k][1] += ns
        total += ns
        n += 1
    tab = sorted(({"kernel": k, "launches": c, "ms": t / 1e6, "share": t / total} for k, (c, t) in per.items()),
                 key=lambda x: -x["ms"])
    json.dump({"source": path, "launches": n, "total_ms": total / 1e6, "kernels": tab}, open(out, "w"), indent=1)
    for x in tab[:15]:
        print(f'{x["share"]:.3f} {x["ms"]:9.3f} ms {x["launches"]:6d}  {x["kernel"]}')


def full(path, out):
    raw = subprocess.run([NCU, "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    want = {"gpu__time_duration.sum": "us", "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
            "launch__registers_per_thread": "regs", "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
            "launch__grid_size": "grid", "sm__cycles_elapsed.avg.per_second": "sm_hz"}
    idx = {want[h]: i for i, h in enumerate(hdr) if h in want}
    units = rows[1] if len(rows) > 1 else []
    out_rows = []
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for k, i in idx.items():
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i] if i < len(units) else ""
            if k in ("dram_read", "dram_write"):
                v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
            if k == "us":
                v *= {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(u, 1)
            d[k] = v
        if "dram_read" in d and "dram_write" in d:
            d["dram_bytes"] = d["dram_read"] + d["dram_write"]
        out_rows.append(d)
    json.dump({"source": path, "launches": out_rows}, open(out, "w"), indent=1)
    for d in out_rows:
        print(json.dumps(d))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])

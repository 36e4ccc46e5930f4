"""Summarise ncu captures into markdown/JSON for profiles/ (run in the build container).

  python tools/summarize_ncu.py launches <launches.csv>            # per-kernel share of a launch list
  python tools/summarize_ncu.py full <report.ncu-rep> [...]         # key metrics of --set full captures
  python tools/summarize_ncu.py traffic <report.ncu-rep> <out.json> # dram bytes per launch, per kernel
"""
from __future__ import annotations

import collections
import csv
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 read sectors (from L1)"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC / SM"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
]


def raw_rows(rep):
    """Rows of an ncu report's raw page (a .ncu-rep, or its `--page raw --csv` export)."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def to_bytes(val: str, unit: str) -> float:
    v = float(val.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return v * scale


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
              "s": 1e6, "second": 1e6}.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name].append(v)
    total = sum(sum(v) for v in agg.values())
    print("| kernel | launches | mean us | total ms | share |")
    print("|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{k}` | {len(v)} | {sum(v) / len(v):.1f} | {sum(v) / 1e3:.3f} | {sum(v) / total * 100:.1f}% |")


def full(reps):
    print("| kernel | " + " | ".join(label for _, label in KEYS) + " |")
    print("|---|" + "---|" * len(KEYS))
    for rep in reps:
        h, units, rows = raw_rows(rep)
        for r in rows:
            name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
            vals = []
            for key, _ in KEYS:
                if key in h:
                    i = h.index(key)
                    vals.append(f"{r[i]} {units[i]}".strip())
                else:
                    vals.append("n/a")
            print(f"| `{name}` | " + " | ".join(vals) + " |")


def traffic(rep, out):
    h, units, rows = raw_rows(rep)
    res = {}
    for r in rows:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        rd = to_bytes(r[h.index("dram__bytes_read.sum")], units[h.index("dram__bytes_read.sum")])
        wr = to_bytes(r[h.index("dram__bytes_write.sum")], units[h.index("dram__bytes_write.sum")])
        res.setdefault(name, []).append(rd + wr)
    res = {k: sum(v) / len(v) for k, v in res.items()}
    json.dump({"source": rep, "dram_bytes_per_launch": res}, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2])
    elif mode == "full":
        full(sys.argv[2:])
    elif mode == "traffic":
        traffic(sys.argv[2], sys.argv[3])

"""Print the key metrics of an ncu report (all kernels in it): python tools/ncu_summary.py rep [filter]"""
import csv
import subprocess
import sys

KEYS = ["Duration", "Executed Instructions", "Executed Ipc Active", "Issue Slots Busy", "DRAM Throughput",
        "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Achieved Occupancy", "Registers Per Thread", "Warp Cycles Per Issued Instruction",
        "Eligible Warps Per Scheduler", "Compute (SM) Throughput", "Branch Instructions"]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ik, iname, iv, iu = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    seen = {}
    for r in rows[1:]:
        if len(r) <= iv:
            continue
        k = r[ik].split("(")[0]
        if len(sys.argv) > 2 and sys.argv[2] not in k:
            continue
        if r[iname] in KEYS:
            seen.setdefault(k, {})[r[iname]] = f"{r[iv]} {r[iu]}"
    for k, m in seen.items():
        print(k)
        for key in KEYS:
            if key in m:
                print(f"   {key:38s} {m[key]}")


if __name__ == "__main__":
    main()

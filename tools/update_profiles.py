"""Copy a tools/gpu_final.sh capture (gpurun_out/) into profiles/ (run in the build container)."""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")


def last_line(path):
    return open(path).read().strip().splitlines()[-1]


def summ(*args):
    return subprocess.run([sys.executable, os.path.join(ROOT, "tools", "summarize_ncu.py"), *args],
                          capture_output=True, text=True).stdout


for c in ("cfg2", "cfg2_exact", "cfg1", "cfg3", "cfg4", "ref_cfg2"):
    open(os.path.join(P, f"round1_bench_{c}.json"), "w").write(last_line(os.path.join(G, f"bench_{c}.json")) + "\n")
shutil.copy(os.path.join(G, "launches_cfg2.csv"), os.path.join(P, "round1_launches_cfg2.csv"))
lines = [l for l in open(os.path.join(G, "bench_cfg3_prof.err")) if "build_csr" in l or "reslice total" in l]
open(os.path.join(P, "round1_cfg3_recon_phases.txt"), "w").writelines(lines[:12])
old = json.load(open(os.path.join(P, "round1_traffic.json")))["dram_bytes_per_launch"]
tr = {}
for rep in ("full_reslice", "full_recon"):
    out = "/tmp/_tr.json"
    summ("traffic", os.path.join(G, rep + ".ncu-rep"), out)
    tr.update(json.load(open(out))["dram_bytes_per_launch"])
for k in ("compound_k<1>", "reslice_k<1>"):
    tr.setdefault(k, old.get(k))
json.dump({"source": "ncu --set full --clock-control none, one launch each, cfg2 bench (tools/gpu_final.sh)",
           "dram_bytes_per_launch": tr,
           "note": "reslice launches = one 64-pose batch at 256x256 on the cfg2 volume (ncu prints bool template "
                   "arguments as 0/1); recon kernels = one cfg2 build (frames in HBM); compound_k<1> and "
                   "reslice_k<1> (exact path, captured before z-binning) from the earlier round-1 capture"},
          open(os.path.join(P, "round1_traffic.json"), "w"), indent=1)
full = summ("full", os.path.join(G, "full_reslice.ncu-rep"), os.path.join(G, "full_recon.ncu-rep")).strip().splitlines()
seen, rows = set(), []
for l in full:
    k = l.split("|")[1] if l.startswith("| `") else None
    if k and k in seen:
        continue
    if k:
        seen.add(k)
    rows.append(l)
md = open(os.path.join(P, "round1_cfg2.md")).read()
head = md.split("Bench line (plain run")[0]
tail = md.split("Reading:")[1]
launch = summ("launches", os.path.join(P, "round1_launches_cfg2.csv"))
b, bx = last_line(os.path.join(G, "bench_cfg2.json")), last_line(os.path.join(G, "bench_cfg2_exact.json"))
intro = md.split("## Launch list")[1].split("| kernel |")[0]
new = (head + "Bench line (plain run, no profiler; `python bench.py`, default = certified reslice path):\n```json\n"
       + b + "\n```\n\nExact-FP64 mode for comparison (`python bench.py --exact --no-cpu-baseline --no-scalar`):\n"
       "```json\n" + bx + "\n```\n\n## Launch list" + intro + launch + "\n## ncu --set full (one launch each)\n\n"
       + "\n".join(rows) + "\n\nReading:" + tail)
open(os.path.join(P, "round1_cfg2.md"), "w").write(new)
print("profiles updated")

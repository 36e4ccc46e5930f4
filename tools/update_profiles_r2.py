"""Copy a tools/gpu_evidence_r2.sh capture (gpurun_out/ev_*) into profiles/round2_* (build container)."""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
TAG = sys.argv[1] if len(sys.argv) > 1 else "round2"


def last_line(path):
    return open(path).read().strip().splitlines()[-1]


def summ(*args):
    return subprocess.run([sys.executable, os.path.join(ROOT, "tools", "summarize_ncu.py"), *args],
                          capture_output=True, text=True).stdout


for c in ("cfg2", "ref_cfg2", "cfg1", "cfg3", "cfg4"):
    src = os.path.join(G, f"ev_bench_{c}.json")
    if os.path.exists(src):
        open(os.path.join(P, f"{TAG}_bench_{c}.json"), "w").write(last_line(src) + "\n")
for f in ("ev_pytest_gpu.log", "ev_smoke.log"):
    if os.path.exists(os.path.join(G, f)):
        shutil.copy(os.path.join(G, f), os.path.join(P, f"{TAG}_{f[3:]}"))
shutil.copy(os.path.join(G, "ev_launches_cfg2.csv"), os.path.join(P, f"{TAG}_launches_cfg2.csv"))
reps = {t: os.path.join(G, f"ev_raw_{t}.csv") for t in
        ("reslice", "fallback", "prep", "count", "fill", "seal", "compound", "fillpass", "trilinear")}
reps = {t: r for t, r in reps.items() if os.path.exists(r)}
tr = {}
for t, r in reps.items():
    out = "/tmp/_tr.json"
    summ("traffic", r, out)
    tr.update(json.load(open(out))["dram_bytes_per_launch"])
recon = sum(v for k, v in tr.items() if any(s in k for s in ("frame_count", "frame_fill", "seal_k")))
json.dump({"source": "ncu --set full --clock-control none, one launch each, cfg2 bench (tools/gpu_evidence_r2.sh)",
           "dram_bytes_per_launch": tr,
           "recon": {"cfg2": {"dram_bytes": recon, "kernels": "count + fill + seal of one cfg2 build"}},
           "note": "reslice launches = one 64-pose batch at 256x256 on the cfg2 volume; recon kernels = one cfg2 "
                   "build (frames in HBM)"}, open(os.path.join(P, f"{TAG}_traffic.json"), "w"), indent=1)
full = summ("full", *reps.values()).strip()
launch = summ("launches", os.path.join(P, f"{TAG}_launches_cfg2.csv"))
b = last_line(os.path.join(G, "ev_bench_cfg2.json"))
ref = last_line(os.path.join(G, "ev_bench_ref_cfg2.json"))
md = ["# Round 2 — cfg2 evidence (B200, tools/gpu_evidence_r2.sh -> tools/update_profiles_r2.py)", "",
      "Bench line (plain run, no profiler; `python bench.py --steps 20 --warmup 5`):", "```json", b, "```", "",
      "Reference arm (`python bench.py --impl reference --steps 20 --warmup 5`, same box):", "```json", ref, "```", "",
      "## Launch list (ncu gpu__time_duration, --clock-control none; cold-cache, serialised — compare shares)",
      "Command: `python bench.py --steps 3 --warmup 3 --no-cpu-baseline` (raw CSV: "
      f"`{TAG}_launches_cfg2.csv`).", "", launch, "", "## ncu --set full (one launch each)", "", full, ""]
open(os.path.join(P, f"{TAG}_cfg2.md"), "w").write("\n".join(md))
print("profiles updated:", sorted(reps))

"""Writes profiles/bench_r01.md from the gpurun_out/all_*.log lines of scripts/all_configs.sh."""
import glob
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = ["# bench results, round 1 (one B200; `bash scripts/all_configs.sh`)", ""]
gpu = os.path.join(ROOT, "gpurun_out", "gpu.txt")
if os.path.exists(gpu):
    out += ["GPU: " + "; ".join(l.strip() for l in open(gpu) if l.strip()), ""]
out += ["Full JSON lines:", ""]
for f in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "all_*.log"))):
    name = os.path.basename(f)[4:-4]
    for line in open(f):
        if line.startswith("{"):
            out += [f"## {name}", "", "```json", json.dumps(json.loads(line), indent=1), "```", ""]
            break
with open(os.path.join(ROOT, "profiles", "bench_r01.md"), "w") as fh:
    fh.write("\n".join(out))
print("wrote", len(out), "lines")

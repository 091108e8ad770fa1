#!/bin/bash
# GPU M-H vs the exact baselines (alias / direct / rejection) per config.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
for c in cfg1 cfg2 cfg3a cfg3b; do
  for s in mh alias direct rejection; do
    timeout 600 $B --config $c --sampler $s > gpurun_out/s_${c}_${s}.log 2>&1
  done
done
for f in gpurun_out/s_*.log; do
  python - "$f" <<'PY'
import json, sys
p = sys.argv[1]
for line in open(p):
    if line.startswith("{"):
        d = json.loads(line); c = d["config"]
        print(f"{p}: {d['value']:.4g} steps/s  ms/step {d['ms_per_step']:.2f}  trials {c.get('rejection_trials')}")
        break
else:
    print(p, "FAILED:", open(p).read()[-300:].replace("\n", " | "))
PY
done

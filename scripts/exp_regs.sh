#!/bin/bash
# Experiment: register cap of the walk kernel (occupancy vs spills).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
for c in cfg2 cfg4 cfg3b; do
  for r in 64 80 255; do
    MHW_WALK_REGS=$r $B --config $c > gpurun_out/g_${c}_r$r.log 2>&1
  done
done
python scripts/summ.py gpurun_out/g_*.log

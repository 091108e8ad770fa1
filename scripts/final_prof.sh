#!/bin/bash
# Round-end captures: the launch list of a short cfg2 bench (kernel shares)
# and one --set full capture of the walk kernel per config.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py --config cfg2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/fp_plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_cfg2_final.csv python bench.py --config cfg2 --steps 2 --warmup 1 \
  --no-cpu-baseline --no-e2e > gpurun_out/fp_launches.log 2>&1
for c in cfg2 cfg4 cfg1 cfg3b; do bash scripts/prof.sh $c final; done
ls -la gpurun_out/*.ncu-rep

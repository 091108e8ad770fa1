#!/bin/bash
# Runs bench.py over every BASELINE config on one GPU (logs in gpurun_out/).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
python bench.py --config cfg2 --steps 5 --warmup 3 > gpurun_out/all_cfg2.log 2>&1
for c in cfg1 cfg3a cfg3b cfg4; do
  python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/all_$c.log 2>&1
done
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/all_cfg5.log 2>&1

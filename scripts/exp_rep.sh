#!/bin/bash
# Experiment: hub replica degree sweep for metapath2vec (cfg3a).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
for d in 1 2 4 8 16; do
  MHW_REP_MAX=65536 MHW_REP_DEG=$d $B --config cfg3a > gpurun_out/r_cfg3a_d$d.log 2>&1
done
python scripts/summ.py gpurun_out/r_*.log

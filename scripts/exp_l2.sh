#!/bin/bash
# Experiment: L2 persisting window for the chain table; deepwalk replica degree.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
$B --config cfg2 > gpurun_out/x_cfg2_base.log 2>&1
MHW_L2_PERSIST_MB=64 $B --config cfg2 > gpurun_out/x_cfg2_p64.log 2>&1
MHW_L2_PERSIST_MB=30 $B --config cfg2 > gpurun_out/x_cfg2_p30.log 2>&1
$B --config cfg1 > gpurun_out/x_cfg1_base.log 2>&1
MHW_REP_DEG=64 $B --config cfg1 > gpurun_out/x_cfg1_r64.log 2>&1
MHW_REP_DEG=256 $B --config cfg1 > gpurun_out/x_cfg1_r256.log 2>&1
MHW_L2_PERSIST_MB=64 $B --config cfg1 > gpurun_out/x_cfg1_p64.log 2>&1
$B --config cfg4 > gpurun_out/x_cfg4_base.log 2>&1
MHW_L2_PERSIST_MB=64 $B --config cfg4 > gpurun_out/x_cfg4_p64.log 2>&1
python scripts/summ.py gpurun_out/x_*.log
grep -h "L2 persist" gpurun_out/x_*.log | sort | uniq

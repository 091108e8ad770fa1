#!/bin/bash
# A/B of two libmhw.so builds on one config: bash scripts/ab2.sh <a.so> <b.so> <cfg> [reps]
cd "$(dirname "$0")/.."
A=$1; B=$2; CFG=${3:-cfg2}; N=${4:-3}
R="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --config $CFG"
for i in $(seq $N); do
  for L in $A $B; do
    MHW_LIB=$L $R | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$(basename $L)', '$CFG', round(d['ms_per_step'],2), round(d['roofline']['kernel_ms'],2))"
  done
done

#!/bin/bash
# A/B of two builds of libmhw.so on one config: bash scripts/ab.sh <old.so> <cfg> [reps]
cd "$(dirname "$0")/.."
OLD=$1; CFG=${2:-cfg2}; N=${3:-3}
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --config $CFG"
for i in $(seq $N); do
  MHW_LIB=$OLD $B | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('old', round(d['roofline']['kernel_ms'],2))"
  $B | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('new', round(d['roofline']['kernel_ms'],2))"
done

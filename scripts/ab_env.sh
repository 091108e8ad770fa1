#!/bin/bash
# A/B of environment knobs (and optionally a build variant) on one config:
#   bash scripts/ab_env.sh cfg2 2 "X=1" "MHW_LAST_EARLY=0" "MHW_LIB=$PWD/paper_2010_04895_b200/libmhw_ids32.so"
cd "$(dirname "$0")/.."
CFG=${1:-cfg2}; N=${2:-2}; shift 2
R="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --config $CFG"
for i in $(seq $N); do
  for mode in "$@"; do
    env $mode $R | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print('$mode', '$CFG', 'step', round(d['ms_per_step'],2), 'walk', round(r['kernel_ms'],2), 'init', round(r['init_ms'],2), 'retries', d['config']['chain_retries'])"
  done
done

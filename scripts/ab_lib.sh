#!/bin/bash
# A/B of libmhw build variants (scripts/build_variant.sh) on one config:
#   bash scripts/ab_lib.sh cfg2 2 default hashef stef ...
cd "$(dirname "$0")/.."
CFG=${1:-cfg2}; N=${2:-2}; shift 2
R="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --config $CFG"
for i in $(seq $N); do
  for v in "$@"; do
    if [ "$v" = default ]; then L=; else L="MHW_LIB=$PWD/paper_2010_04895_b200/libmhw_$v.so"; fi
    env $L $R | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print('$v', '$CFG', 'step', round(d['ms_per_step'],2), 'walk', round(r['kernel_ms'],2), 'init', round(r['init_ms'],2), 'retries', d['config']['chain_retries'])"
  done
done

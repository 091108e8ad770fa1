#!/bin/bash
# A/B of the node2vec chain layouts on one config: bash scripts/ab_c16.sh cfg2 [reps] [modes...]
cd "$(dirname "$0")/.."
CFG=${1:-cfg2}; N=${2:-2}; shift 2
MODES=("$@")
[ ${#MODES[@]} -eq 0 ] && MODES=("MHW_C16=0" "MHW_C16=1")
R="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --config $CFG"
for i in $(seq $N); do
  for mode in "${MODES[@]}"; do
    env $mode $R | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print('$mode', '$CFG', 'step', round(d['ms_per_step'],2), 'walk', round(r['kernel_ms'],2), 'init', round(r['init_ms'],2), 'retries', d['config']['chain_retries'])"
  done
done

#!/bin/bash
# Uniform vs alias proposal on the weighted configs: bash scripts/alias_bench.sh
cd "$(dirname "$0")/.."
for c in cfg1 cfg3a cfg3b cfg4; do
  for p in uniform alias; do
    python bench.py --config $c --proposal $p --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print('$c', '$p', 'step', round(d['ms_per_step'],2), 'walk', round(r['kernel_ms'],2), 'init', round(r['init_ms'],2), 'Gsteps/s', round(d['value']/1e9,2), 'retries', d['config']['chain_retries'])"
  done
done

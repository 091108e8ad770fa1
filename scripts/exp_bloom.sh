#!/bin/bash
# Experiment: edge Bloom filter size and L2 persistence.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
for c in cfg2 cfg4; do
  for b in ${BITS:-2 4}; do
    MHW_BLOOM_MB=160 MHW_BLOOM_BITS=$b $B --config $c > gpurun_out/bx_${c}_b$b.log 2>&1
    MHW_BLOOM_MB=160 MHW_BLOOM_BITS=$b MHW_BLOOM_PERSIST=1 $B --config $c > gpurun_out/bx_${c}_b${b}p.log 2>&1
  done
done
python scripts/summ.py gpurun_out/bx_*.log

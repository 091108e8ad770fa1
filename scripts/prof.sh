#!/bin/bash
# One ncu --set full capture of the first k_walk launch of a config:
#   bash scripts/prof.sh cfg2 tag   ->  gpurun_out/prof_<cfg>_<tag>.ncu-rep
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cfg=${1:-cfg2}; tag=${2:-x}
python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_${cfg}_${tag}_plain.log 2>&1 || exit 1
SET=${NCU_METRICS:+--metrics $NCU_METRICS}; SET=${SET:---set full}
timeout 1800 ncu $SET --clock-control none --import-source on -k regex:${KREGEX:-k_walk} -c 1 \
  -o gpurun_out/prof_${cfg}_${tag} -f python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/prof_${cfg}_${tag}_ncu.log 2>&1
tail -3 gpurun_out/prof_${cfg}_${tag}_ncu.log

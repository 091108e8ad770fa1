#!/bin/bash
# Round-end captures: the launch list of a short cfg2 bench (kernel shares)
# and one --set full capture of the walk kernel per config. Reports beyond
# KEEP are summarised on the box (profiles/summarize.py) and deleted, to stay
# under gpurun's 64 MiB return limit.
#   bash scripts/final_prof.sh "cfg2 cfg4" "cfg2"
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFGS=${1:-"cfg2 cfg4"}; KEEP=${2:-"cfg2"}
if [[ " $CFGS " == *" cfg2 "* ]]; then
  python bench.py --config cfg2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/fp_plain.log 2>&1 || exit 1
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_cfg2_final.csv python bench.py --config cfg2 --steps 2 --warmup 1 \
    --no-cpu-baseline --no-e2e > gpurun_out/fp_launches.log 2>&1
fi
for c in $CFGS; do
  bash scripts/prof.sh $c final
  L=""; [ "$c" == cfg2 ] && L=gpurun_out/launches_cfg2_final.csv
  python profiles/summarize.py gpurun_out/prof_${c}_final.ncu-rep ${c}_final $L > gpurun_out/summ_${c}.log 2>&1
  mkdir -p gpurun_out/profiles
  cp profiles/ncu_${c}_final.md gpurun_out/profiles/ 2>/dev/null
  cp profiles/traffic_${c}.json gpurun_out/profiles/ 2>/dev/null
  if [[ " $KEEP " != *" $c "* ]]; then rm -f gpurun_out/prof_${c}_final.ncu-rep; fi
done
ls -la gpurun_out/*.ncu-rep gpurun_out/profiles

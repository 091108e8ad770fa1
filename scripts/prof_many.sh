#!/bin/bash
# ncu --set full captures of k_walk for several env variants of one config,
# summarised on the box (profiles/summarize.py -> gpurun_out/profiles/) and
# the reports deleted (gpurun returns <= 64 MiB):
#   bash scripts/prof_many.sh cfg2 "narrow:MHW_C16=0" "c16:MHW_C16=1 MHW_C16_PIN=chain"
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/profiles
cfg=$1; shift
for spec in "$@"; do
  tag=${spec%%:*}; envs=${spec#*:}
  env $envs bash scripts/prof.sh $cfg $tag > /dev/null 2>&1
  env $envs python profiles/summarize.py gpurun_out/prof_${cfg}_${tag}.ncu-rep ${cfg}_${tag} > gpurun_out/summ_${cfg}_${tag}.log 2>&1
  cp profiles/ncu_${cfg}_${tag}.md gpurun_out/profiles/ 2>/dev/null
  cp profiles/traffic_${cfg}.json gpurun_out/profiles/traffic_${cfg}_${tag}.json 2>/dev/null
  ncu -i gpurun_out/prof_${cfg}_${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${cfg}_${tag}.csv 2>/dev/null
  python profiles/sass_top.py gpurun_out/src_${cfg}_${tag}.csv 40 > gpurun_out/profiles/sass_${cfg}_${tag}.txt 2>&1
  ncu -i gpurun_out/prof_${cfg}_${tag}.ncu-rep --page source --csv --print-source cuda > gpurun_out/srccu_${cfg}_${tag}.csv 2>/dev/null
  python profiles/cuda_top.py gpurun_out/srccu_${cfg}_${tag}.csv 40 > gpurun_out/profiles/cuda_${cfg}_${tag}.txt 2>&1
  rm -f gpurun_out/srccu_${cfg}_${tag}.csv
  rm -f gpurun_out/prof_${cfg}_${tag}.ncu-rep gpurun_out/src_${cfg}_${tag}.csv
done
ls -la gpurun_out/profiles

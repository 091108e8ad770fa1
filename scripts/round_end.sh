#!/bin/bash
# Evidence pass for the committed profiles (one B200): the full GPU suite, the
# default bench line, the ncu launch list of the same bench command, and one
# --set full capture of the cfg2 walk kernel (summarised on the box).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/profiles
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/gputest_final.log 2>&1
echo "pytest exit $?" >> gpurun_out/gputest_final.log
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
  > gpurun_out/launches_final.log 2>&1
bash scripts/prof_many.sh cfg2 "final:"
python profiles/launches.py gpurun_out/launches_final.csv "python bench.py --steps 2 --warmup 1 (cfg2)" > gpurun_out/profiles/launches_cfg2_final.md
tail -3 gpurun_out/gputest_final.log

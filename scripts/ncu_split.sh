#!/usr/bin/env bash
# ncu --set full of search_split_kernel at the C3 operating point (the
# artifacts cached by a plain bench run first, so the captured launch is the
# benchmark's own).
set -u
OUT=gpurun_out
TAG=${1:-split}
T=${2:-166}
mkdir -p $OUT
timeout 900 python bench.py --t $T --no-cpu-baseline --no-parity --steps 2 > $OUT/bench_pre_$TAG.json 2>/dev/null; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches_C3_$TAG.csv python bench.py --t $T --steps 2 --warmup 1 --no-cpu-baseline --no-parity \
  > $OUT/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:search_split -s 1 -c 1 \
  -o $OUT/search_C3_$TAG -f python bench.py --t $T --profile --no-cpu-baseline --no-parity \
  > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
tail -3 $OUT/ncu_full_$TAG.log

#!/usr/bin/env bash
# One GPU session: smoke, GPU parity tests, bench (both arms), ncu launch
# list + one full capture of the search kernel.  Usage (from the repo root):
#   gpurun --timeout 3000 -- 'bash scripts/gpu_round.sh [CONFIG] [TAG]'
set -u
CFG=${1:-C3}
TAG=${2:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi > $OUT/smi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 $OUT/pytest_gpu_$TAG.log
timeout 1500 python bench.py --config $CFG > $OUT/bench_${CFG}_$TAG.json 2> $OUT/bench_${CFG}_$TAG.err; echo "bench rc=$?"
cat $OUT/bench_${CFG}_$TAG.json
T=$(python -c "import json,sys; print(json.load(open('$OUT/bench_${CFG}_$TAG.json'))['config']['t'])" 2>/dev/null || echo 32)
timeout 600 python bench.py --config $CFG --t $T --phases --steps 2 --warmup 3 --no-cpu-baseline \
  > $OUT/phases_${CFG}_$TAG.json 2> $OUT/phases_${CFG}_$TAG.err; echo "phases rc=$?"
python -c "import json; print(json.load(open('$OUT/phases_${CFG}_$TAG.json'))['phase_cycles_per_iteration'])"
timeout 900 python bench.py --config $CFG --impl reference --steps 2 --warmup 1 > $OUT/bench_ref_${CFG}_$TAG.json 2> $OUT/bench_ref_${CFG}_$TAG.err; echo "ref rc=$?"
cat $OUT/bench_ref_${CFG}_$TAG.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches_${CFG}_$TAG.csv python bench.py --config $CFG --t $T --steps 2 --warmup 1 --no-cpu-baseline \
  > $OUT/ncu_launch_bench_$TAG.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:search -s 1 -c 1 \
  -o $OUT/search_${CFG}_$TAG -f python bench.py --config $CFG --t $T --profile --no-cpu-baseline \
  > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
tail -5 $OUT/ncu_full_$TAG.log

#!/usr/bin/env bash
# Round-end measurements (one box): smoke, GPU tests, C3 bench (both arms),
# ncu launch list + full capture of search_split_kernel, C2 and C1 lines.
set -u
OUT=gpurun_out; TAG=${1:-final2}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest_gpu_$TAG.log
timeout 1200 python bench.py > $OUT/bench_C3_$TAG.json 2> $OUT/bench_C3_$TAG.err; echo "bench C3 rc=$?"
python -c "import json; d=json.load(open('$OUT/bench_C3_$TAG.json')); print('C3', d['value'], d['e2e']['value'], d['parity']['mismatches'], d['roofline']['frac'], d['adc_kernel']['frac'], d['config']['t'])"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref_C3_$TAG.json 2> $OUT/bench_ref_C3_$TAG.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches_C3_$TAG.csv python bench.py --t 166 --steps 2 --warmup 1 --no-cpu-baseline --no-parity \
  > $OUT/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:search_split -s 1 -c 1 \
  -o $OUT/search_C3_$TAG -f python bench.py --t 166 --profile --no-cpu-baseline --no-parity \
  > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
timeout 900 python bench.py --config C2 > $OUT/bench_C2_$TAG.json 2> $OUT/bench_C2_$TAG.err; echo "bench C2 rc=$?"
python -c "import json; d=json.load(open('$OUT/bench_C2_$TAG.json')); print('C2', d['value'], d['e2e']['value'], d['parity']['mismatches'], d['config']['t'])"
timeout 900 python bench.py --config C1 > $OUT/bench_C1_$TAG.json 2> $OUT/bench_C1_$TAG.err; echo "bench C1 rc=$?"
python -c "import json; d=json.load(open('$OUT/bench_C1_$TAG.json')); print('C1', d['value'], d['e2e']['value'], d['parity'], d['config']['t'])"

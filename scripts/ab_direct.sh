#!/usr/bin/env bash
# bloom_direct A/B on one box: GPU tests, default bench, bloom_direct=0 at
# the same t, and the split kernel's row/list stage profiles.
set -u
OUT=gpurun_out
TAG=${1:-direct}
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 $OUT/pytest_gpu_$TAG.log
timeout 1200 python bench.py > $OUT/bench_C3_$TAG.json 2> $OUT/bench_C3_$TAG.err; echo "bench rc=$?"
head -c 400 $OUT/bench_C3_$TAG.json; echo
T=$(python -c "import json; print(json.load(open('$OUT/bench_C3_$TAG.json'))['config']['t'])" 2>/dev/null || echo 166)
for o in bloom_direct=0 bloom_direct=1; do
  timeout 600 python bench.py --t $T --opt $o --no-cpu-baseline --no-parity > $OUT/ab_${TAG}_$o.json 2>/dev/null
  python -c "import json; d=json.load(open('$OUT/ab_${TAG}_$o.json')); print('$o', d['value'], d['e2e']['value'])"
done
for pr in 2 3; do
  timeout 600 python bench.py --t $T --phases --opt profile=$pr --steps 2 --warmup 3 --no-cpu-baseline --no-parity \
    > $OUT/phases_${TAG}_p$pr.json 2>/dev/null
  python -c "import json; d=json.load(open('$OUT/phases_${TAG}_p$pr.json')); print('profile $pr', d.get('phase_cycles_per_iteration'))"
done

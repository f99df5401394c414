#!/usr/bin/env bash
# BASELINE configs[3] with a real graph: C4 (100M x 128 u8, partitioned
# Vamana build, graph + vectors in pinned host memory), then the bench line.
# Every build stage is checkpointed under /tmp (bench_data.build_artifacts):
# a call cut off by the session limit is resumed by the next call on the
# same box.  The build log streams to gpurun_out/bench_C4_<tag>.err.
set -u
OUT=gpurun_out
TAG=${1:-c4}
mkdir -p $OUT
df -h /tmp > $OUT/df_$TAG.txt 2>&1; free -g >> $OUT/df_$TAG.txt; du -sh /tmp/bang_C4_ckpt_* >> $OUT/df_$TAG.txt 2>&1
( while true; do date +%T; free -g | sed -n 2p; nvidia-smi --query-gpu=memory.used --format=csv,noheader; sleep 60; done ) \
  > $OUT/mem_$TAG.log 2>&1 &
MON=$!
timeout 600 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest_gpu_$TAG.log
timeout ${C4_TIMEOUT:-3300} python bench.py --config ${C4_CONFIG:-C4} --cache "" --steps 5 --warmup 3 \
  > $OUT/bench_C4_$TAG.json 2> $OUT/bench_C4_$TAG.err
echo "bench C4 rc=$?"
tail -5 $OUT/bench_C4_$TAG.err
head -c 1500 $OUT/bench_C4_$TAG.json; echo
T=$(python -c "import json; print(json.load(open('$OUT/bench_C4_$TAG.json'))['config']['t'])" 2>/dev/null)
if [ -n "$T" ]; then
  timeout 900 python bench.py --config ${C4_CONFIG:-C4} --cache "" --kernel split --t $T --no-cpu-baseline --no-parity \
    > $OUT/bench_C4_split_$TAG.json 2> $OUT/bench_C4_split_$TAG.err
  python -c "import json; d=json.load(open('$OUT/bench_C4_split_$TAG.json')); print('C4 split', d['value'], d['e2e']['value'], d['roofline']['frac'])"
fi
kill $MON

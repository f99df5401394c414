#!/usr/bin/env bash
# BASELINE configs[3] with a real graph: C4 (100M x 128 u8, partitioned
# Vamana build, graph + vectors in pinned host memory), then the bench line.
# The build log streams to gpurun_out/c4_build.log.
set -u
OUT=gpurun_out
TAG=${1:-c4}
mkdir -p $OUT
df -h /tmp > $OUT/df_$TAG.txt 2>&1; free -g >> $OUT/df_$TAG.txt
( while true; do date +%T; free -g | sed -n 2p; nvidia-smi --query-gpu=memory.used --format=csv,noheader; sleep 60; done ) \
  > $OUT/mem_$TAG.log 2>&1 &
MON=$!
timeout ${C4_TIMEOUT:-3300} python bench.py --config C4 --cache "" --steps 5 --warmup 3 \
  > $OUT/bench_C4_$TAG.json 2> $OUT/bench_C4_$TAG.err
echo "bench C4 rc=$?"
kill $MON
tail -5 $OUT/bench_C4_$TAG.err
head -c 1500 $OUT/bench_C4_$TAG.json; echo

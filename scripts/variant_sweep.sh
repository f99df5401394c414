#!/usr/bin/env bash
# Device QPS of every ADC data flow at one worklist size (diagnostic).
CFG=${1:-C2}; T=${2:-80}; TAG=${3:-sweep}
mkdir -p gpurun_out
for v in auto smem-table-warp codebook hbm-table smem-table-generic; do
  timeout 600 python bench.py --config $CFG --t $T --steps 5 --warmup 3 --no-cpu-baseline --variant $v \
    > gpurun_out/${TAG}_$v.json 2> gpurun_out/${TAG}_$v.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_$v.json')); print('$v', d['value'], d['e2e']['value'], d['roofline']['kernel_ms'], d['search_stats'])" || tail -3 gpurun_out/${TAG}_$v.err
done

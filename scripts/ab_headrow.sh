#!/usr/bin/env bash
set -u
OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_hr.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest_gpu_hr.log
for cfg in C2 C3; do
  T=$([ $cfg = C2 ] && echo 68 || echo 166)
  timeout 900 python bench.py --config $cfg --t $T --no-cpu-baseline --no-parity --steps 2 > /dev/null 2>&1
  for rep in 1 2; do
    for hr in 1 0; do
      timeout 600 python bench.py --config $cfg --t $T --opt head_row=$hr --no-cpu-baseline --no-parity > $OUT/ab_hr_${cfg}_${hr}_$rep.json 2>/dev/null
      python -c "import json; d=json.load(open('$OUT/ab_hr_${cfg}_${hr}_$rep.json')); print('$cfg head_row=$hr', $rep, d['value'], d['e2e']['value'])"
    done
  done
done

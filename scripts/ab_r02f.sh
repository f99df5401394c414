#!/usr/bin/env bash
set -u
OUT=gpurun_out; D=paper_2401_11324_b200
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_r02f.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest_gpu_r02f.log
bash scripts/ab_variants.sh f 166 base nohint nohr norr tab24 hrpf
for v in base norr; do
  cp $D/libbang_$v.so $D/libbang.so
  for pr in 1 2 3; do
    timeout 600 python bench.py --t 166 --phases --opt profile=$pr --steps 2 --warmup 3 --no-cpu-baseline --no-parity \
      > $OUT/phases_f_${v}_p$pr.json 2>/dev/null
    python -c "import json; d=json.load(open('$OUT/phases_f_${v}_p$pr.json')); print('$v profile $pr', d.get('phase_cycles_per_iteration'))"
  done
done

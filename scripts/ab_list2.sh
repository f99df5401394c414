#!/usr/bin/env bash
set -u
OUT=gpurun_out; D=paper_2401_11324_b200
cp $D/libbang_list2.so $D/libbang.so
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_list2.log 2>&1; echo "pytest(list2) rc=$?"; tail -2 $OUT/pytest_gpu_list2.log
bash scripts/ab_variants.sh l2 166 base list2
for v in base list2; do
  cp $D/libbang_$v.so $D/libbang.so
  timeout 600 python bench.py --t 166 --phases --opt profile=3 --steps 2 --warmup 3 --no-cpu-baseline --no-parity \
    > $OUT/phases_l2_${v}_p3.json 2>/dev/null
  python -c "import json; d=json.load(open('$OUT/phases_l2_${v}_p3.json')); print('$v profile 3', d.get('phase_cycles_per_iteration'))"
  timeout 600 python bench.py --t 166 --phases --opt profile=2 --steps 2 --warmup 3 --no-cpu-baseline --no-parity \
    > $OUT/phases_l2_${v}_p2.json 2>/dev/null
  python -c "import json; d=json.load(open('$OUT/phases_l2_${v}_p2.json')); print('$v profile 2', d.get('phase_cycles_per_iteration'))"
done

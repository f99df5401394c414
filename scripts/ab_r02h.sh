#!/usr/bin/env bash
set -u
OUT=gpurun_out; D=paper_2401_11324_b200
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_r02h.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest_gpu_r02h.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_r02h.log 2>&1; echo "smoke rc=$?"
bash scripts/ab_variants.sh h 166 base tab24 tab16 hall 2>&1 | grep -v "^ \|^Traceback\|json\|raise\|File\|^\s*\^"
cp $D/libbang_base.so $D/libbang.so
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches_C3_r02h.csv python bench.py --t 166 --steps 2 --warmup 1 --no-cpu-baseline --no-parity \
  > $OUT/ncu_launch_r02h.log 2>&1; echo "ncu launches rc=$?"

#!/usr/bin/env bash
set -u
OUT=gpurun_out; D=paper_2401_11324_b200
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_r02g.log 2>&1; echo "pytest(base) rc=$?"; tail -1 $OUT/pytest_gpu_r02g.log
bash scripts/ab_variants.sh g 166 base hatom hld hst hcp nohr norr 2>&1 | grep -v "^ \|^Traceback\|json\|raise\|File\|^\s*\^" 
for v in hatom hld hst hcp; do
  cp $D/libbang_$v.so $D/libbang.so
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "split_kernel_large_t and C3-166" > $OUT/pytest_$v.log 2>&1; echo "$v parity rc=$?"
done

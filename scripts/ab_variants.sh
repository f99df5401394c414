#!/usr/bin/env bash
# A/B of libbang_<variant>.so builds (scripts/build_variant.sh) on one box:
# each copied over libbang.so in this box's snapshot, then a bench at fixed t.
#   scripts/ab_variants.sh TAG T v1 v2 ...
set -u
OUT=gpurun_out; TAG=$1; T=$2; shift 2
D=paper_2401_11324_b200
mkdir -p $OUT
timeout 900 python bench.py --t $T --no-cpu-baseline --steps 2 > $OUT/ab_${TAG}_pre.json 2> $OUT/ab_${TAG}_pre.err
python -c "import json; d=json.load(open('$OUT/ab_${TAG}_pre.json')); print('pre', d['value'], d['parity'])"
for rep in 1 2; do
  for v in "$@"; do
    cp $D/libbang_$v.so $D/libbang.so
    timeout 600 python bench.py --t $T --no-cpu-baseline --no-parity > $OUT/ab_${TAG}_${v}_$rep.json 2>/dev/null
    python -c "import json; d=json.load(open('$OUT/ab_${TAG}_${v}_$rep.json')); print('$v', $rep, d['value'], d['e2e']['value'], d['roofline']['kernel_ms'])"
  done
done

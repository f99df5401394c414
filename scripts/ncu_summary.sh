#!/usr/bin/env bash
# Summaries of one ncu --set full report (details page + per-line hotspots)
# and of an ncu launch list, written under profiles/<tag>/.
#   scripts/ncu_summary.sh gpurun_out/search_C2_r01.ncu-rep gpurun_out/launches_C2_r01.csv profiles/r01 C2
set -e
REP=$1; LAUNCHES=$2; OUT=$3; NAME=${4:-C2}
mkdir -p $OUT
ncu -i $REP --page details --csv 2>/dev/null | python3 -c "
import csv,sys
r=csv.reader(sys.stdin); h=next(r)
for row in r:
    d=dict(zip(h,row))
    if d['Metric Name']: print(d['Section Name'][:28].ljust(28), d['Metric Name'][:60].ljust(60), d['Metric Unit'][:12].ljust(12), d['Metric Value'])
" > $OUT/ncu_search_${NAME}_details.txt
ncu -i $REP --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=csv.reader(sys.stdin); h=next(r); u=next(r)
want=('gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','lts__t_bytes.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','sm__throughput.avg.pct_of_peak_sustained_elapsed','dram__bytes_read.sum.per_second','lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum','lts__t_sectors_srcunit_tex_op_read.sum','smsp__inst_executed.sum','launch__grid_size','launch__block_size')
for row in r:
    for k,unit,v in zip(h,u,row):
        if k in want: print(k.ljust(56), unit.ljust(10), v)
" > $OUT/ncu_search_${NAME}_raw.txt
ncu -i $REP --page source --csv --print-source cuda,sass 2>/dev/null > /tmp/_ncu_src.csv
python3 $(dirname $0)/ncu_lines.py /tmp/_ncu_src.csv 60 > $OUT/ncu_search_${NAME}_lines.txt
python3 - "$LAUNCHES" > $OUT/launches_${NAME}.txt <<'PY'
import csv, sys
from collections import defaultdict
lines = [l for l in open(sys.argv[1]) if not l.startswith('==')]
agg = defaultdict(lambda: [0, 0.0])
for d in csv.DictReader(lines):
    if d.get('Metric Name') != 'gpu__time_duration.sum':
        continue
    v = float(d['Metric Value'].replace(',', ''))
    unit = d.get('Metric Unit', 'ns')
    v = v * {'ns': 1, 'us': 1e3, 'usecond': 1e3, 'nsecond': 1, 'ms': 1e6, 'msecond': 1e6}.get(unit, 1)
    agg[d['Kernel Name'][:100]][0] += 1
    agg[d['Kernel Name'][:100]][1] += v
tot = sum(v[1] for v in agg.values())
print(f"ncu launch list (gpu__time_duration.sum, --clock-control none, cold/serialised): {sys.argv[1]}")
print(f"{'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>6s}  kernel")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[0]:8d} {v[1]/1e3:12.1f} {v[1]/1e3/v[0]:10.1f} {100*v[1]/tot:5.1f}%  {k}")
PY

#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_bartlett.py -q -x --timeout 600 > $OUT/l_tests.log 2>&1; echo "rc=$?" >> $OUT/l_tests.log
for wl in c1_1d c2_2d c4_batched_2d c3_3d; do
  python bench.py --workload $wl --bartlett --steps 5 > $OUT/l_bart_$wl.json 2> $OUT/l_bart_$wl.err
done
C="python bench.py --workload c4_batched_2d --bartlett --steps 2 --warmup 3"
$C > $OUT/l_plain_bart.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 20 --csv --log-file $OUT/l_launches_bart_c4.csv $C > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_bart_cols -s 1 -c 1 -o $OUT/l_prof_cols -f $C > $OUT/l_ncu.log 2>&1
[ -f $OUT/l_prof_cols.ncu-rep ] && python scripts/ncu_summary.py $OUT/l_prof_cols.ncu-rep > $OUT/l_prof_cols.summary.txt 2>&1
[ -f $OUT/l_prof_cols.ncu-rep ] && python scripts/sass_lines.py $OUT/l_prof_cols.ncu-rep paper_1610_01050_b200/librsft.so > $OUT/l_prof_cols.lines.txt 2>&1
echo done

#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_bartlett.py -q -x --timeout 600 > $OUT/n_tests.log 2>&1; echo "rc=$?" >> $OUT/n_tests.log
for wl in c2_2d c4_batched_2d c3_3d; do
  python bench.py --workload $wl --bartlett --steps 5 > $OUT/n_bart_$wl.json 2> $OUT/n_bart_$wl.err
done
C="python bench.py --workload c4_batched_2d --bartlett --steps 2 --warmup 3"
$C > $OUT/n_plain_bart.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 20 --csv --log-file $OUT/n_launches_bart_c4.csv $C > /dev/null 2>&1
C4="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$C4 > $OUT/n_plain_c4.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 -o $OUT/n_prof_fused -f $C4 > $OUT/n_ncu_fused.log 2>&1
[ -f $OUT/n_prof_fused.ncu-rep ] && python scripts/sass_lines.py $OUT/n_prof_fused.ncu-rep paper_1610_01050_b200/librsft.so 40 > $OUT/n_prof_fused.lines.txt 2>&1
[ -f $OUT/n_prof_fused.ncu-rep ] && python scripts/ncu_summary.py $OUT/n_prof_fused.ncu-rep > $OUT/n_prof_fused.summary.txt 2>&1
echo done

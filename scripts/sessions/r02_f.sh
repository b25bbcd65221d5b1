#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu -x --timeout 900 -k "3d or c3 or 1d or c1 or c4_full or compaction or variant_b or segment" > $OUT/f_pytest.log 2>&1; echo "rc=$?" >> $OUT/f_pytest.log
python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e > $OUT/f_c1.json 2> $OUT/f_c1.err
python bench.py --workload c3_3d --frames 256 --steps 10 --no-cpu --no-e2e > $OUT/f_c3.json 2> $OUT/f_c3.err
C3="python bench.py --workload c3_3d --frames 256 --steps 2 --warmup 3 --no-cpu --no-e2e"
$C3 > $OUT/f_plain_c3.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/f_launches_c3.csv $C3 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_split_fold -s 1 -c 1 -o $OUT/f_prof_c3 -f $C3 > $OUT/f_ncu_c3.log 2>&1
C1="python bench.py --workload c1_1d --frames 131072 --steps 2 --warmup 3 --no-cpu --no-e2e"
$C1 > $OUT/f_plain_c1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/f_launches_c1.csv $C1 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_vote1d -s 1 -c 1 -o $OUT/f_prof_v1 -f $C1 > $OUT/f_ncu_v1.log 2>&1
for r in $OUT/f_prof_c3 $OUT/f_prof_v1; do
  [ -f $r.ncu-rep ] && python scripts/ncu_summary.py $r.ncu-rep > $r.summary.txt 2>&1
done
echo done

#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_bartlett.py tests/test_gpu_montecarlo.py -q -x -s --timeout 600 > $OUT/k_tests.log 2>&1; echo "rc=$?" >> $OUT/k_tests.log
for wl in c1_1d c2_2d c4_batched_2d c3_3d; do
  python bench.py --workload $wl --bartlett --steps 5 > $OUT/k_bart_$wl.json 2> $OUT/k_bart_$wl.err
  python bench.py --workload $wl --segments --steps 5 > $OUT/k_seg_$wl.json 2> $OUT/k_seg_$wl.err
done
C="python bench.py --workload c4_batched_2d --bartlett --steps 2 --warmup 3"
$C > $OUT/k_plain_bart.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 20 --csv --log-file $OUT/k_launches_bart_c4.csv $C > /dev/null 2>&1
C="python bench.py --workload c3_3d --segments --steps 2 --warmup 3"
$C > $OUT/k_plain_seg.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/k_launches_seg_c3.csv $C > /dev/null 2>&1
echo done

#!/bin/bash
# Bartlett two-pass with transpose-form warp FFTs (no shuffle stages), 4-warp column CTAs with next-segment prefetch
set -u
OUT=gpurun_out/bh; mkdir -p $OUT
timeout 900 python -m pytest tests/test_bartlett.py -x -q --timeout 600 > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for wl in c4_batched_2d c2_2d c3_3d; do
  python bench.py --workload $wl --bartlett --steps 5 > $OUT/bart_$wl.json 2> $OUT/bart_$wl.err
done
for wl in c4_batched_2d c2_2d; do
  CMD="python bench.py --workload $wl --bartlett --steps 2 --warmup 3"
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.sum --clock-control none -c 30 --csv --log-file $OUT/launches_bart_$wl.csv $CMD > /dev/null 2>&1
done
echo done

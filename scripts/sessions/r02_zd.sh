#!/bin/bash
set -u
OUT=gpurun_out/zd; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "2d or c4 or c2" > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
for i in 1 2; do
python bench.py --steps 10 --no-cpu --no-e2e > $OUT/c4_$i.json 2> $OUT/c4_$i.err
python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e > $OUT/c2_$i.json 2> $OUT/c2_$i.err
done
RSFT_VOTE2S=0 python bench.py --steps 10 --no-cpu --no-e2e > $OUT/c4_old.json 2> $OUT/c4_old.err
RSFT_VOTE2S=0 python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e > $OUT/c2_old.json 2> $OUT/c2_old.err
for wl in c4_batched_2d:4096 c2_2d:8192; do
  w=${wl%%:*}; f=${wl##*:}
  CMD="python bench.py --workload $w --frames $f --steps 2 --warmup 3 --no-cpu --no-e2e"
  $CMD > $OUT/plain_$w.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_$w.csv $CMD > /dev/null 2>&1
done
echo done

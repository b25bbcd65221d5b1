#!/bin/bash
set -u
OUT=gpurun_out/za; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "3d or c3 or vote3d" > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
for i in 1 2; do
python bench.py --workload c3_3d --frames 256 --steps 10 --no-cpu --no-e2e > $OUT/c3_$i.json 2> $OUT/c3_$i.err
done
C3="python bench.py --workload c3_3d --frames 256 --steps 2 --warmup 3 --no-cpu --no-e2e"
$C3 > $OUT/plain_c3.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c3.csv $C3 > /dev/null 2>&1
echo done

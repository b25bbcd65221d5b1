#!/bin/bash
set -u
OUT=gpurun_out/z; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_montecarlo.py -q -x --timeout 600 -k "1d or c1 or host or T50 or fixed_schedule" > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
for i in 1 2; do
python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e > $OUT/c1_$i.json 2> $OUT/c1_$i.err
python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e --run > $OUT/c1_run_$i.json 2> $OUT/c1_run_$i.err
done
C1="python bench.py --workload c1_1d --frames 131072 --steps 2 --warmup 3 --no-cpu --no-e2e"
$C1 > $OUT/plain_c1.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c1.csv $C1 > /dev/null 2>&1
echo done

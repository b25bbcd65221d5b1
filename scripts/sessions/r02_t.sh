#!/bin/bash
set -u
OUT=gpurun_out/t; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "3d or c3 or c5 or segment" > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
RSFT_VOTE3D=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "3d_mma or c5_full or variant_b_c5" > $OUT/tests_v3.log 2>&1; echo "rc=$?" >> $OUT/tests_v3.log
python bench.py --workload c3_3d --frames 256 --steps 10 --no-cpu --no-e2e > $OUT/c3.json 2> $OUT/c3.err
python bench.py --workload c5_cube --no-cpu --no-e2e > $OUT/c5.json 2> $OUT/c5.err
RSFT_VOTE3D=1 python bench.py --workload c5_cube --no-cpu --no-e2e > $OUT/c5_v3.json 2> $OUT/c5_v3.err
for v in 0 1; do
C="python bench.py --workload c5_cube --steps 2 --warmup 3 --no-cpu --no-e2e"
RSFT_VOTE3D=$v $C > $OUT/plain_$v.log 2>&1 && RSFT_VOTE3D=$v ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file $OUT/launches_c5_$v.csv $C > /dev/null 2>&1
done
C3="python bench.py --workload c3_3d --frames 256 --steps 2 --warmup 3 --no-cpu --no-e2e"
$C3 > $OUT/plain_c3.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c3.csv $C3 > /dev/null 2>&1
echo done

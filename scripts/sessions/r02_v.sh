#!/bin/bash
set -u
OUT=gpurun_out/v; mkdir -p $OUT
RSFT_VOTE1D_OCC=6 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "1d or c1" > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
for i in 1 2; do
python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e > $OUT/c1_$i.json 2> $OUT/c1_$i.err
RSFT_VOTE1D_OCC=6 python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e > $OUT/c1_occ_$i.json 2> $OUT/c1_occ_$i.err
done
C1="python bench.py --workload c1_1d --frames 131072 --steps 2 --warmup 3 --no-cpu --no-e2e"
RSFT_VOTE1D_OCC=6 $C1 > $OUT/plain_c1.log 2>&1 && RSFT_VOTE1D_OCC=6 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c1_occ.csv $C1 > /dev/null 2>&1
echo done

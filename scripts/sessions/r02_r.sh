#!/bin/bash
set -u
OUT=gpurun_out/r; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "2d or 1d or c2 or c1 or smoke" > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e > $OUT/c2.json 2> $OUT/c2.err
RSFT_F2_STAGES=2 python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e > $OUT/c2_s2.json 2> $OUT/c2_s2.err
python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e > $OUT/c1.json 2> $OUT/c1.err
python bench.py --no-cpu --no-e2e > $OUT/c4.json 2> $OUT/c4.err
C1="python bench.py --workload c1_1d --frames 131072 --steps 2 --warmup 3 --no-cpu --no-e2e"
$C1 > $OUT/plain_c1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c1.csv $C1 > /dev/null 2>&1
echo done

#!/bin/bash
set -u
OUT=gpurun_out/zf; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_montecarlo.py -q --timeout 900 -k "1d or c1 or segment or T50" > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e > $OUT/c1.json 2> $OUT/c1.err
python bench.py --workload c1_1d --segments --steps 5 > $OUT/seg_c1.json 2> $OUT/seg_c1.err
echo done

#!/bin/bash
set -u
OUT=gpurun_out/y; mkdir -p $OUT
for v in 8 10 12; do
RSFT_G1_VOTE_WARPS=$v timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "1d_g_c1like or 1d_v or c1" > $OUT/tests_$v.log 2>&1; echo "rc=$?" >> $OUT/tests_$v.log
RSFT_G1_VOTE_WARPS=$v python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e --run > $OUT/c1_run_v$v.json 2> $OUT/c1_run_v$v.err
done
echo done

#!/bin/bash
set -u
OUT=gpurun_out/zg; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 -k "1d_B128_full" > $OUT/t1.log 2>&1; echo "rc=$?" >> $OUT/t1.log
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 -k "1d_B256_eq_N" > $OUT/t2.log 2>&1; echo "rc=$?" >> $OUT/t2.log
timeout 300 python -m pytest tests/test_gpu_parity.py -q --timeout 120 -k "segment_mode" > $OUT/t3.log 2>&1; echo "rc=$?" >> $OUT/t3.log
timeout 120 python bench.py --workload c1_1d --segments --steps 5 > $OUT/seg_c1.json 2> $OUT/seg_c1.err
echo done

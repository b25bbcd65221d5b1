#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_bartlett.py -q -x --timeout 600 > $OUT/p_tests.log 2>&1; echo "rc=$?" >> $OUT/p_tests.log
python bench.py --workload c1_1d --bartlett --steps 5 > $OUT/p_bart_c1.json 2> $OUT/p_bart_c1.err
echo done

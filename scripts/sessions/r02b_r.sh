#!/bin/bash
# Bartlett 1-D N = 4096 (c1) with the transpose-form four-step kernel vs the shuffle form
set -u
OUT=gpurun_out/br; mkdir -p $OUT
timeout 600 python -m pytest tests/test_bartlett.py -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
RSFT_BART_1D_SHFL=1 timeout 600 python -m pytest tests/test_bartlett.py -x -q -k "4096" > $OUT/pytest_shfl.log 2>&1; echo "rc=$?" >> $OUT/pytest_shfl.log
python bench.py --workload c1_1d --bartlett --steps 5 > $OUT/bart_c1.json 2> $OUT/bart_c1.err
RSFT_BART_1D_SHFL=1 python bench.py --workload c1_1d --bartlett --steps 5 > $OUT/bart_c1_shfl.json 2> $OUT/bart_c1_shfl.err
echo done

#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x --timeout 600 -k "1d or c1" > $OUT/d_pytest.log 2>&1; echo "rc=$?" >> $OUT/d_pytest.log
for c in 1 2; do
  RSFT_G1_CTAS=$c python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e > $OUT/d_c1_$c.json 2> $OUT/d_c1_$c.err
done
echo done

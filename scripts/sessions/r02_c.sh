#!/bin/bash
# Round 2, session C: k_gather1d bulk-copy chunk size sweep at c1 + 1-D parity.
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x --timeout 600 -k "1d or c1" > $OUT/c_pytest.log 2>&1; echo "rc=$?" >> $OUT/c_pytest.log
for k in 32768 16384 8192 4096 2048; do
  for c in 2 1; do
    RSFT_G1_CTAS=$c RSFT_G1_CHUNK=$k python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e > $OUT/c_c1_${k}_$c.json 2> $OUT/c_c1_${k}_$c.err
  done
done
echo done

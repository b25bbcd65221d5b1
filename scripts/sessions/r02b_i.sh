#!/bin/bash
# Bartlett column pass variants: warps per CTA (4 / 8) x next-segment register prefetch (on / off)
set -u
OUT=gpurun_out/bi; mkdir -p $OUT
for v in "" _cw4pf0 _cw8pf0 _cw8pf1; do
  for wl in c4_batched_2d c2_2d c3_3d; do
    RSFT_LIB=$PWD/paper_1610_01050_b200/librsft$v.so python bench.py --workload $wl --bartlett --steps 5 > $OUT/bart_$wl$v.json 2> $OUT/bart_$wl$v.err
  done
done
RSFT_LIB=$PWD/paper_1610_01050_b200/librsft_cw8pf0.so timeout 600 python -m pytest tests/test_bartlett.py -x -q > $OUT/pytest_cw8pf0.log 2>&1; echo "rc=$?" >> $OUT/pytest_cw8pf0.log
echo done

#!/bin/bash
set -u
OUT=gpurun_out/zb; mkdir -p $OUT
for g in 148 144 140 136 132 128 120 112; do
  RSFT_FUSED_SMS=$g python bench.py --steps 10 --no-cpu --no-e2e > $OUT/c4_$g.json 2> $OUT/c4_$g.err
done
echo done

#!/bin/bash
# fused c1 kernel: nanosleep back-off for the vote warps' bfull wait and the producer's empty wait
set -u
OUT=gpurun_out/bn; mkdir -p $OUT
for v in "" _sl100 _sl400 _sl1500; do
  for r in 1 2; do
    RSFT_LIB=$PWD/paper_1610_01050_b200/librsft$v.so python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e > $OUT/c1$v.$r.json 2> $OUT/c1$v.$r.err
  done
done
echo done

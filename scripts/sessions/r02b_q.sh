#!/bin/bash
# c5 vote occupancy: k_vote built for 4 (default) / 6 / 8 CTAs per SM
set -u
OUT=gpurun_out/bq; mkdir -p $OUT
for v in "" _vc6 _vc8; do
  for r in 1 2; do
    RSFT_LIB=$PWD/paper_1610_01050_b200/librsft$v.so python bench.py --workload c5_cube --no-cpu --no-e2e > $OUT/c5$v.$r.json 2> $OUT/c5$v.$r.err
  done
  CMD="python bench.py --workload c5_cube --steps 2 --warmup 3 --no-cpu --no-e2e"
  RSFT_LIB=$PWD/paper_1610_01050_b200/librsft$v.so ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c5$v.csv $CMD > /dev/null 2>&1
done
echo done

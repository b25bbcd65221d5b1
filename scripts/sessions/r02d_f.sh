#!/bin/bash
# c5: k_split_mma X-ring depth variants (RSFT_MMA_SX = 8 / 12 / 16, build/var); c1: bulk-copy chunk 16384 (new
# default) vs 8192 / 32768 on rsft_run and on the two-call path; GPU suite on the new default.
set -u
OUT=gpurun_out/df; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu --timeout 1200 > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
for rep in 1 2; do
  for v in default sx8 sx12; do
    so=build/var/librsft_$v.so; [ $v = default ] && so=paper_1610_01050_b200/librsft.so
    RSFT_LIB=$so python bench.py --workload c5_cube --steps 50 --no-cpu --no-e2e > $OUT/c5_${v}_$rep.json 2> $OUT/c5_${v}_$rep.err
  done
done
C1="python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e"
$C1 > $OUT/bench_c1.json 2> $OUT/bench_c1.err
$C1 --two-calls > $OUT/bench_c1_two.json 2> $OUT/bench_c1_two.err
for k in 8192 32768; do
  RSFT_G1_CHUNK=$k $C1 > $OUT/sweep_c1_chunk$k.json 2> $OUT/sweep_c1_chunk$k.err
  RSFT_G1_CHUNK=$k $C1 --two-calls > $OUT/sweep_c1_two_chunk$k.json 2> $OUT/sweep_c1_two_chunk$k.err
done
CMD="$C1 --steps 2 --warmup 3"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
  --log-file $OUT/launches_c1_1d.csv $CMD > /dev/null 2>&1
echo done

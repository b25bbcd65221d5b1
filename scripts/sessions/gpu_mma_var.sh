#!/bin/bash
# k_split_mma variants (default, no operand work, no TMA): launch list per variant.
mkdir -p gpurun_out
CMD5="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --workload c5_cube"
for so in ${VARS:-paper_1610_01050_b200/librsft.so build/var/librsft_mmadbg1.so build/var/librsft_mmadbg2.so}; do
  n=$(basename $so .so)
  RSFT_LIB=$so $CMD5 > /dev/null 2>&1 && RSFT_LIB=$so ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_split -c 5 --csv --log-file gpurun_out/mv_$n.csv $CMD5 > /dev/null 2>&1
  echo "== $n"; python scripts/launches.py gpurun_out/mv_$n.csv | head -3
done

#!/bin/bash
# Split-fold tuning: parity of the split path with the default build, then c5 bench per variant.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -x -k "split or 3d or c3 or determinism or loop_range or c5" --timeout 600 > gpurun_out/v_parity.log 2>&1; tail -3 gpurun_out/v_parity.log
for so in paper_1610_01050_b200/librsft.so build/var/librsft_*.so; do
  echo "== $so" >> gpurun_out/v_bench.txt
  RSFT_LIB=$so python bench.py --workload c5_cube --steps 20 --warmup 5 --no-cpu --no-e2e >> gpurun_out/v_bench.txt 2>&1
done
CMD5="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --workload c5_cube"
$CMD5 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/v_launches_c5.csv $CMD5 > /dev/null 2>&1
echo done

#!/bin/bash
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/n_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 -o gpurun_out/prof_fused2 -f $CMD > gpurun_out/n_full.log 2>&1
CMD5="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --workload c5_cube"
$CMD5 > gpurun_out/n_plain5.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_split_fold -s 1 -c 1 -o gpurun_out/prof_split -f $CMD5 > gpurun_out/n_full5.log 2>&1
echo done

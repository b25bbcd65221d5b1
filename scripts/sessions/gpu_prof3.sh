#!/bin/bash
mkdir -p gpurun_out
CMDS5="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --workload c5_cube"
$CMDS5 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_split_fold" -s 4 -c 1 -o gpurun_out/prof_split3 -f $CMDS5 > gpurun_out/n_split3.log 2>&1
CMDS="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$CMDS > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_region_write" -s 3 -c 1 -o gpurun_out/prof_rw -f $CMDS > gpurun_out/n_rw.log 2>&1
echo done

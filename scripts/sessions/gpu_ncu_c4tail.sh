#!/bin/bash
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_region_write|k_vote" -s 2 -c 2 -o gpurun_out/prof_c4tail -f $CMD > gpurun_out/c4tail_ncu.log 2>&1
echo done

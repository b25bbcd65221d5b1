#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-vote}
WL=${2:-c4_batched_2d}
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --workload $WL"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_vote -s 1 -c 1 -o gpurun_out/prof_${TAG} -f $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo done

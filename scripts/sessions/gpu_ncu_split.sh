#!/bin/bash
# ncu --set full of the split fold kernel (c5) for the given library variant (default build).
mkdir -p gpurun_out
TAG=${1:-split}
CMD5="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --workload c5_cube"
$CMD5 > gpurun_out/${TAG}_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_split_fold -s 1 -c 1 -o gpurun_out/prof_${TAG} -f $CMD5 > gpurun_out/${TAG}_ncu.log 2>&1
echo done

#!/bin/bash
# ncu --set full of one kernel (regex $2) of a bench workload ($3, default c5_cube), tag $1.
mkdir -p gpurun_out
TAG=${1:-k}; K=${2:-k_split}; WL=${3:-c5_cube}
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --workload $WL"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/prof_${TAG} -f $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo done

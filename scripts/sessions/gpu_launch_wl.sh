#!/bin/bash
# launch lists for the batched c1/c2/c3 variants
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -c 40 --csv --log-file gpurun_out/ll_c1.csv python bench.py --workload c1_1d --frames 131072 --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -c 40 --csv --log-file gpurun_out/ll_c3.csv python bench.py --workload c3_3d --frames 256 --pool 16 --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -c 40 --csv --log-file gpurun_out/ll_c2.csv python bench.py --workload c2_2d --frames 8192 --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
echo done

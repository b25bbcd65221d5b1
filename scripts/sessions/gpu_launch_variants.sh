#!/bin/bash
# Per-variant ncu launch list (kernel durations) for c5: tuning experiments.
mkdir -p gpurun_out
for so in build/var/librsft_*.so; do
  b=$(basename $so .so)
  RSFT_LIB=$so ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -c 12 --csv --log-file gpurun_out/vl_$b.csv python bench.py --workload ${1:-c5_cube} --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
echo done

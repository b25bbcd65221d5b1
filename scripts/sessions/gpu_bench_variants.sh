#!/bin/bash
# c5 bench per library variant in build/var (tuning experiments; no parity).
mkdir -p gpurun_out
WL=${1:-c5_cube}
for so in build/var/librsft_*.so; do
  echo "== $so" >> gpurun_out/vb_bench.txt
  RSFT_LIB=$so python bench.py --workload $WL --steps 20 --warmup 5 --no-cpu --no-e2e >> gpurun_out/vb_bench.txt 2>&1
done
echo done

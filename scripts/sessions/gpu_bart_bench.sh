#!/bin/bash
mkdir -p gpurun_out
for wl in c1_1d c2_2d c4_batched_2d c3_3d; do
  python bench.py --bartlett --workload $wl --steps 5 > gpurun_out/bart_$wl.json 2> gpurun_out/bart_$wl.err
done
python bench.py --workload c2_2d --frames 8192 --no-cpu --no-e2e > gpurun_out/rsft_c2.json 2>/dev/null
for wl in c1_1d c2_2d c4_batched_2d c3_3d; do
  python bench.py --segments --workload $wl --steps 5 > gpurun_out/seg_$wl.json 2> gpurun_out/seg_$wl.err
done
echo done

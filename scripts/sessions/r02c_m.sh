#!/bin/bash
# Round-2c re-entry check of HEAD: GPU tests, smoke, default bench, c3/c5 bench lines.
set -u
OUT=gpurun_out/m; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for wl in c5_cube c3_3d c1_1d c2_2d; do
  timeout 600 python bench.py --workload $wl --steps 20 --no-cpu --no-e2e > $OUT/bench_$wl.json 2> $OUT/bench_$wl.err
done
echo done

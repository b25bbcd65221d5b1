#!/bin/bash
# Re-entry check of HEAD: smoke, full GPU tests, default bench + the other bench lines.
set -u
OUT=gpurun_out/x; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $OUT/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 1200 > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
python bench.py > $OUT/bench_c4.json 2> $OUT/bench_c4.err
python bench.py --workload c5_cube --no-cpu --no-e2e > $OUT/bench_c5.json 2> $OUT/bench_c5.err
python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e --run > $OUT/bench_c1run.json 2> $OUT/bench_c1run.err
python bench.py --workload c3_3d --frames 256 --steps 10 --no-cpu --no-e2e > $OUT/bench_c3.json 2> $OUT/bench_c3.err
echo done

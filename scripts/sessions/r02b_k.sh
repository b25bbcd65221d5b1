#!/bin/bash
# branch-free packed lane DIF (warp_dif): full GPU suite + the bench lines it touches
set -u
OUT=gpurun_out/bk; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 1200 > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
python bench.py --no-cpu --no-e2e > $OUT/bench_c4.json 2> $OUT/bench_c4.err
python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e > $OUT/bench_c1.json 2> $OUT/bench_c1.err
python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e > $OUT/bench_c2.json 2> $OUT/bench_c2.err
python bench.py --workload c3_3d --frames 256 --steps 10 --no-cpu --no-e2e > $OUT/bench_c3.json 2> $OUT/bench_c3.err
python bench.py --workload c5_cube --no-cpu --no-e2e > $OUT/bench_c5.json 2> $OUT/bench_c5.err
echo done

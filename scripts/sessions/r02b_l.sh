#!/bin/bash
set -u
OUT=gpurun_out/bl; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "1d or c1 or determinism" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for r in 1 2; do python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e > $OUT/bench_c1.$r.json 2> $OUT/bench_c1.$r.err; done
python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e --two-calls > $OUT/bench_c1_two.json 2> $OUT/bench_c1_two.err
echo done

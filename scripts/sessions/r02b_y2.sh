#!/bin/bash
set -u
OUT=gpurun_out/y2; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "2d or c4 or c2 or persistent or zero or gamma or compaction or determinism or host" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for ne in 4 8; do
RSFT_F2V_EPI=$ne python bench.py --no-cpu --no-e2e --run > $OUT/bench_c4run_$ne.json 2> $OUT/bench_c4run_$ne.err
RSFT_F2V_EPI=$ne python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e --run > $OUT/bench_c2run_$ne.json 2> $OUT/bench_c2run_$ne.err
done
python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e > $OUT/bench_c2.json 2> $OUT/bench_c2.err
echo done

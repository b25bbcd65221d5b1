#!/bin/bash
# fused2v (D = 2 rsft_run with fold + epilogue/vote warps): parity on every D = 2 fused case, c4 / c2 bench lines
set -u
OUT=gpurun_out/y; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "2d or c4 or c2 or persistent or zero or gamma or compaction or determinism or host" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
python bench.py --no-cpu --no-e2e --run > $OUT/bench_c4run.json 2> $OUT/bench_c4run.err
python bench.py --no-cpu --no-e2e > $OUT/bench_c4.json 2> $OUT/bench_c4.err
python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e --run > $OUT/bench_c2run.json 2> $OUT/bench_c2run.err
CMD="python bench.py --no-cpu --no-e2e --run --steps 2 --warmup 3"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c4run.csv $CMD > /dev/null 2>&1
echo done

#!/bin/bash
# k_split_fft_w64 (B_0 = 64 outer grids, c5): parity on the 3-D cases + c5 cube, c5 bench (+ vote3d at c5), launch list
set -u
OUT=gpurun_out/bc; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q --timeout 900 -k "3d or c5 or variant" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
python bench.py --workload c5_cube --no-cpu --no-e2e > $OUT/bench_c5.json 2> $OUT/bench_c5.err
RSFT_VOTE3D=1 python bench.py --workload c5_cube --no-cpu --no-e2e > $OUT/bench_c5_v3.json 2> $OUT/bench_c5_v3.err
CMD="python bench.py --workload c5_cube --steps 2 --warmup 3 --no-cpu --no-e2e"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c5.csv $CMD > /dev/null 2>&1
RSFT_VOTE3D=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c5_v3.csv $CMD > /dev/null 2>&1
echo done

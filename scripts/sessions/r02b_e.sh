#!/bin/bash
# c5 tail: register-form outer FFT (k_split_fft_w64) + bitmap vote with empty-slab plane test (k_vote3s)
set -u
OUT=gpurun_out/be; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q --timeout 900 -k "3d or c5 or c3 or variant" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
python bench.py --workload c5_cube --no-cpu --no-e2e > $OUT/bench_c5.json 2> $OUT/bench_c5.err
RSFT_FFT_WARP=0 python bench.py --workload c5_cube --no-cpu --no-e2e > $OUT/bench_c5_ctafft.json 2> $OUT/bench_c5_ctafft.err
RSFT_VOTE3S=0 python bench.py --workload c5_cube --no-cpu --no-e2e > $OUT/bench_c5_novs.json 2> $OUT/bench_c5_novs.err
python bench.py --workload c3_3d --frames 256 --steps 10 --no-cpu --no-e2e > $OUT/bench_c3.json 2> $OUT/bench_c3.err
RSFT_VOTE3S=0 python bench.py --workload c3_3d --frames 256 --steps 10 --no-cpu --no-e2e > $OUT/bench_c3_novs.json 2> $OUT/bench_c3_novs.err
CMD="python bench.py --workload c5_cube --steps 2 --warmup 3 --no-cpu --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c5.csv $CMD > /dev/null 2>&1
CMD="python bench.py --workload c3_3d --frames 256 --steps 2 --warmup 3 --no-cpu --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c3.csv $CMD > /dev/null 2>&1
echo done

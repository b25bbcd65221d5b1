#!/bin/bash
# w64/w32 outer FFT load hoisting (c5, c3); k_fused2v variants (weights from global, Ffull back-off) at c4 / c2
set -u
OUT=gpurun_out/bd; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "3d_w or c5_full or c3" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
python bench.py --workload c5_cube --no-cpu --no-e2e > $OUT/bench_c5.json 2> $OUT/bench_c5.err
python bench.py --workload c3_3d --frames 256 --steps 10 --no-cpu --no-e2e > $OUT/bench_c3.json 2> $OUT/bench_c3.err
CMD="python bench.py --workload c5_cube --steps 2 --warmup 3 --no-cpu --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c5.csv $CMD > /dev/null 2>&1
CMD="python bench.py --workload c3_3d --frames 256 --steps 2 --warmup 3 --no-cpu --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c3.csv $CMD > /dev/null 2>&1
for v in "" _gw _sl; do
  for rep in 1 2; do
  RSFT_LIB=$PWD/paper_1610_01050_b200/librsft$v.so python bench.py --no-cpu --no-e2e > $OUT/bench_c4$v.$rep.json 2> $OUT/bench_c4$v.$rep.err
  done
  RSFT_LIB=$PWD/paper_1610_01050_b200/librsft$v.so python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e > $OUT/bench_c2$v.json 2> $OUT/bench_c2$v.err
done
echo done

#!/bin/bash
# k_fused2v: one epilogue warp per loop (gather, free the slot, then FFT); 1 vs 2 residue-sum slots (FB), ring depth
set -u
OUT=gpurun_out/bf; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "2d or c4 or c2 or persistent or zero or gamma or compaction or determinism or fused2v" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
RSFT_LIB=$PWD/paper_1610_01050_b200/librsft_fb1.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "2d_fused or c4 or c2 or persistent or fused2v" > $OUT/pytest_fb1.log 2>&1; echo "rc=$?" >> $OUT/pytest_fb1.log
for rep in 1 2; do
  python bench.py --no-cpu --no-e2e > $OUT/bench_c4_fb2.$rep.json 2> $OUT/bench_c4_fb2.$rep.err
  RSFT_LIB=$PWD/paper_1610_01050_b200/librsft_fb1.so python bench.py --no-cpu --no-e2e > $OUT/bench_c4_fb1.$rep.json 2> $OUT/bench_c4_fb1.$rep.err
  RSFT_F2V_STAGES=4 RSFT_LIB=$PWD/paper_1610_01050_b200/librsft_fb1.so python bench.py --no-cpu --no-e2e > $OUT/bench_c4_fb1s4.$rep.json 2> $OUT/bench_c4_fb1s4.$rep.err
done
python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e > $OUT/bench_c2_fb2.json 2> $OUT/bench_c2_fb2.err
RSFT_LIB=$PWD/paper_1610_01050_b200/librsft_fb1.so python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e > $OUT/bench_c2_fb1.json 2> $OUT/bench_c2_fb1.err
echo done

#!/bin/bash
# register-form outer FFT for B_0 = 32 (c3) vs the direct-DFT warp form; new fused2v corner cases
set -u
OUT=gpurun_out/bp; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "3d or c3 or c5 or f2v" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for r in 1 2; do
python bench.py --workload c3_3d --frames 256 --steps 10 --no-cpu --no-e2e > $OUT/c3.$r.json 2> $OUT/c3.$r.err
RSFT_FFT_W32DFT=1 python bench.py --workload c3_3d --frames 256 --steps 10 --no-cpu --no-e2e > $OUT/c3_dft.$r.json 2> $OUT/c3_dft.$r.err
done
python bench.py --workload c5_cube --no-cpu --no-e2e > $OUT/c5.json 2> $OUT/c5.err
CMD="python bench.py --workload c3_3d --frames 256 --steps 2 --warmup 3 --no-cpu --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c3.csv $CMD > /dev/null 2>&1
echo done

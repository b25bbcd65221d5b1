#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_montecarlo.py -q -s -x --timeout 600 > $OUT/j_mc.log 2>&1; echo "rc=$?" >> $OUT/j_mc.log
timeout 900 python tests/study_next2.py > $OUT/j_study.log 2>&1; echo "rc=$?" >> $OUT/j_study.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "2d_frame_vote or c2_shape" > $OUT/j_v2.log 2>&1; echo "rc=$?" >> $OUT/j_v2.log
python bench.py --workload c3_3d --frames 256 --steps 10 --no-cpu --no-e2e > $OUT/j_c3.json 2> $OUT/j_c3.err
python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e > $OUT/j_c2.json 2> $OUT/j_c2.err
echo done

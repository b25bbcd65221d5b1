#!/bin/bash
set -u
OUT=gpurun_out/ze; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -k "2d or c4 or c2" > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:k_vote2s -s 1 -c 1 -o $OUT/prof_c4_vote2s -f $CMD > $OUT/ncu.log 2>&1
python scripts/ncu_summary.py $OUT/prof_c4_vote2s.ncu-rep > $OUT/prof_c4_vote2s.summary.txt 2>&1
python scripts/sass_lines.py $OUT/prof_c4_vote2s.ncu-rep paper_1610_01050_b200/librsft.so 40 > $OUT/prof_c4_vote2s.lines.txt 2>&1
echo done

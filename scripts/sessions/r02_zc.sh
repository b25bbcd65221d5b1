#!/bin/bash
set -u
OUT=gpurun_out/zc; mkdir -p $OUT
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$CMD > $OUT/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_vote -s 1 -c 1 -o $OUT/prof_c4_vote -f $CMD > $OUT/ncu.log 2>&1
python scripts/ncu_summary.py $OUT/prof_c4_vote.ncu-rep > $OUT/prof_c4_vote.summary.txt 2>&1
python scripts/sass_lines.py $OUT/prof_c4_vote.ncu-rep paper_1610_01050_b200/librsft.so 40 > $OUT/prof_c4_vote.lines.txt 2>&1
echo done

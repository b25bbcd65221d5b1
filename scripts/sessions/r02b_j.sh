#!/bin/bash
# Bartlett with per-shape column CTAs (tests + bench lines); c1 fused rsft_run kernel source-line profile
set -u
OUT=gpurun_out/bj; mkdir -p $OUT
timeout 900 python -m pytest tests/test_bartlett.py -x -q --timeout 600 > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for wl in c4_batched_2d c2_2d c3_3d c1_1d; do
  python bench.py --workload $wl --bartlett --steps 5 > $OUT/bart_$wl.json 2> $OUT/bart_$wl.err
done
CMD="python bench.py --workload c1_1d --frames 131072 --steps 2 --warmup 3 --no-cpu --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:k_gather1d -s 1 -c 1 -o $OUT/prof_c1_run -f $CMD > $OUT/ncu_c1.log 2>&1
if [ -f $OUT/prof_c1_run.ncu-rep ]; then
  python scripts/ncu_summary.py $OUT/prof_c1_run.ncu-rep > $OUT/prof_c1_run.summary.txt 2>&1
  python scripts/sass_lines.py $OUT/prof_c1_run.ncu-rep paper_1610_01050_b200/librsft.so 50 > $OUT/prof_c1_run.lines.txt 2>&1
  rm -f $OUT/prof_c1_run.ncu-rep
fi
echo done

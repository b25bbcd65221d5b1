#!/bin/bash
set -u
OUT=gpurun_out/s; mkdir -p $OUT
RSFT_MMA_MBAR=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "mma or variant_b or determinism or c5" > $OUT/tests_mbar.log 2>&1; echo "rc=$?" >> $OUT/tests_mbar.log
for i in 1 2; do
python bench.py --workload c5_cube --no-cpu --no-e2e > $OUT/c5_bar_$i.json 2> $OUT/c5_bar_$i.err
RSFT_MMA_MBAR=1 python bench.py --workload c5_cube --no-cpu --no-e2e > $OUT/c5_mbar_$i.json 2> $OUT/c5_mbar_$i.err
done
C5="python bench.py --workload c5_cube --steps 2 --warmup 3 --no-cpu --no-e2e"
RSFT_MMA_MBAR=1 $C5 > $OUT/plain.log 2>&1 && \
RSFT_MMA_MBAR=1 ncu --set full --clock-control none --import-source on -k regex:k_split_mma -s 1 -c 1 -o $OUT/prof_mma -f $C5 > $OUT/ncu.log 2>&1
[ -f $OUT/prof_mma.ncu-rep ] && python scripts/ncu_summary.py $OUT/prof_mma.ncu-rep > $OUT/prof_mma.summary.txt 2>&1
[ -f $OUT/prof_mma.ncu-rep ] && python scripts/sass_lines.py $OUT/prof_mma.ncu-rep paper_1610_01050_b200/librsft.so 30 > $OUT/prof_mma.lines.txt 2>&1
rm -f $OUT/prof_mma.ncu-rep
echo done

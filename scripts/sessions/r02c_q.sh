#!/bin/bash
# k_vote3d offsets in registers (no per-lookup branch) + k_vote double-buffered E copies: 3-D parity, c3/c5 bench, launch lists, ncu.
set -u
OUT=gpurun_out/q; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "3d or vote or c3 or cube" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
C3="python bench.py --workload c3_3d --frames 256 --steps 2 --warmup 3 --no-cpu --no-e2e"
C5="python bench.py --workload c5_cube --steps 2 --warmup 3 --no-cpu --no-e2e"
timeout 300 python bench.py --workload c3_3d --frames 256 --steps 20 --no-cpu --no-e2e > $OUT/c3.json 2> $OUT/c3.err
timeout 300 python bench.py --workload c5_cube --steps 50 --no-cpu --no-e2e > $OUT/c5.json 2> $OUT/c5.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c3.csv $C3 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c5.csv $C5 > /dev/null 2>&1
python scripts/launches.py $OUT/launches_c3.csv $OUT/launches_c5.csv > $OUT/launches.txt 2>&1
for k in k_vote3d; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o $OUT/prof_$k -f $C3 > $OUT/ncu_$k.log 2>&1
  [ -f $OUT/prof_$k.ncu-rep ] && python scripts/ncu_summary.py $OUT/prof_$k.ncu-rep > $OUT/prof_$k.summary.txt 2>&1
  [ -f $OUT/prof_$k.ncu-rep ] && python scripts/sass_lines.py $OUT/prof_$k.ncu-rep paper_1610_01050_b200/librsft.so > $OUT/prof_$k.lines.txt 2>&1
done



echo done
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_vote -s 1 -c 1 -o $OUT/prof_kvote_c5 -f $C5 > $OUT/ncu_kvote_c5.log 2>&1
[ -f $OUT/prof_kvote_c5.ncu-rep ] && python scripts/ncu_summary.py $OUT/prof_kvote_c5.ncu-rep > $OUT/prof_kvote_c5.summary.txt 2>&1
[ -f $OUT/prof_kvote_c5.ncu-rep ] && python scripts/sass_lines.py $OUT/prof_kvote_c5.ncu-rep paper_1610_01050_b200/librsft.so > $OUT/prof_kvote_c5.lines.txt 2>&1
echo done2

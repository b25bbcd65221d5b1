#!/bin/bash
# c5: k_split_mma X ring of 20 stages (build/var/librsft_sx20.so) vs 16; c1 with one bulk copy per frame
# (default): GPU suite, smoke, final c1 line + launch list; final c5 / c3 lines.
set -u
OUT=gpurun_out/dg; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -q -m gpu --timeout 1200 > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
for rep in 1 2; do
  for v in default sx20; do
    so=build/var/librsft_$v.so; [ $v = default ] && so=paper_1610_01050_b200/librsft.so
    RSFT_LIB=$so python bench.py --workload c5_cube --steps 50 --no-cpu --no-e2e > $OUT/c5_${v}_$rep.json 2> $OUT/c5_${v}_$rep.err
  done
done
RSFT_LIB=build/var/librsft_sx20.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "c5 or mma or cube" --timeout 500 > $OUT/pytest_sx20.log 2>&1; echo "rc=$?" >> $OUT/pytest_sx20.log
C1="python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e"
$C1 > $OUT/bench_c1.json 2> $OUT/bench_c1.err
$C1 --two-calls > $OUT/bench_c1_two.json 2> $OUT/bench_c1_two.err
python bench.py --no-cpu --no-e2e > $OUT/bench_c4_rep.json 2> $OUT/bench_c4_rep.err
CMD="$C1 --steps 2 --warmup 3"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
  --log-file $OUT/launches_c1_1d.csv $CMD > /dev/null 2>&1
timeout 500 ncu --set full --clock-control none --import-source on -k regex:k_gather1d -s 1 -c 1 -o $OUT/prof_c1_k_gather1d_run -f $CMD > $OUT/ncu_c1.log 2>&1
if [ -f $OUT/prof_c1_k_gather1d_run.ncu-rep ]; then
  python scripts/ncu_summary.py $OUT/prof_c1_k_gather1d_run.ncu-rep > $OUT/prof_c1_k_gather1d_run.summary.txt 2>&1
  python scripts/sass_lines.py $OUT/prof_c1_k_gather1d_run.ncu-rep paper_1610_01050_b200/librsft.so 30 > $OUT/prof_c1_k_gather1d_run.lines.txt 2>&1
  rm -f $OUT/prof_c1_k_gather1d_run.ncu-rep
fi
echo done

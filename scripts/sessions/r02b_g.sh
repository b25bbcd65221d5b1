#!/bin/bash
# Bartlett baseline analysis: launch lists (time + DRAM bytes) and ncu captures of the two passes (c4, c2)
set -u
OUT=gpurun_out/bg; mkdir -p $OUT
for wl in c4_batched_2d c2_2d; do
  python bench.py --workload $wl --bartlett --steps 5 > $OUT/bart_$wl.json 2> $OUT/bart_$wl.err
  CMD="python bench.py --workload $wl --bartlett --steps 2 --warmup 3"
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 30 --csv --log-file $OUT/launches_bart_$wl.csv $CMD > /dev/null 2>&1
done
prof() {
  CMD="python bench.py --workload $2 --bartlett --steps 2 --warmup 3"
  ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 -o $OUT/prof_$1 -f $CMD > $OUT/ncu_$1.log 2>&1
  if [ -f $OUT/prof_$1.ncu-rep ]; then
    python scripts/ncu_summary.py $OUT/prof_$1.ncu-rep > $OUT/prof_$1.summary.txt 2>&1
    python scripts/sass_lines.py $OUT/prof_$1.ncu-rep paper_1610_01050_b200/librsft.so 30 > $OUT/prof_$1.lines.txt 2>&1
    rm -f $OUT/prof_$1.ncu-rep
  fi
}
prof c4_rows c4_batched_2d k_bart_rows
prof c4_cols c4_batched_2d k_bart_cols
echo done

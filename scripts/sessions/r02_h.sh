#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python bench.py --workload c3_3d --frames 256 --steps 10 --no-cpu --no-e2e > $OUT/h_c3.json 2> $OUT/h_c3.err
for t in 64 128 256 512; do
  RSFT_FFT_THREADS=$t python bench.py --workload c3_3d --frames 256 --steps 10 --no-cpu --no-e2e > $OUT/h_c3_t$t.json 2> $OUT/h_c3_t$t.err
done
RSFT_NO_VOTE2D=1 python bench.py --no-cpu --no-e2e > $OUT/h_c4_old.json 2> $OUT/h_c4_old.err
C4="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$C4 > $OUT/h_plain_c4.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_vote2d -s 1 -c 1 -o $OUT/h_prof_v2 -f $C4 > $OUT/h_ncu_v2.log 2>&1
C1="python bench.py --workload c1_1d --frames 131072 --steps 2 --warmup 3 --no-cpu --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:k_vote1d -s 1 -c 1 -o $OUT/h_prof_v1 -f $C1 > $OUT/h_ncu_v1.log 2>&1
for r in $OUT/h_prof_v2 $OUT/h_prof_v1; do
  [ -f $r.ncu-rep ] && python scripts/ncu_summary.py $r.ncu-rep > $r.summary.txt 2>&1
done
echo done

#!/bin/bash
set -u
OUT=gpurun_out/w; mkdir -p $OUT
prof() {   # name workload frames kernel-regex
  CMD="python bench.py --workload $2 --frames $3 --steps 2 --warmup 3 --no-cpu --no-e2e"
  $CMD > $OUT/plain_$1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$4 -s 1 -c 1 -o $OUT/prof_$1 -f $CMD > $OUT/ncu_$1.log 2>&1
  if [ -f $OUT/prof_$1.ncu-rep ]; then
    python scripts/ncu_summary.py $OUT/prof_$1.ncu-rep > $OUT/prof_$1.summary.txt 2>&1
    python scripts/sass_lines.py $OUT/prof_$1.ncu-rep paper_1610_01050_b200/librsft.so 40 > $OUT/prof_$1.lines.txt 2>&1
    rm -f $OUT/prof_$1.ncu-rep
  fi
}
prof c3_k_vote3d c3_3d 256 k_vote3d
prof c1_k_vote1d c1_1d 131072 k_vote1d
prof c3_k_split_fft c3_3d 256 k_split_fft
echo done

#!/bin/bash
# fused2v: full GPU suite, ncu captures of k_fused2v at c4 and c2 (source-line attribution)
set -u
OUT=gpurun_out/z; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 1200 > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
prof() {   # name workload frames kernel-regex extra
  CMD="python bench.py --workload $2 --frames $3 --steps 2 --warmup 3 --no-cpu --no-e2e --run"
  $CMD > $OUT/plain_$1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$4 -s 1 -c 1 -o $OUT/prof_$1 -f $CMD > $OUT/ncu_$1.log 2>&1
  if [ -f $OUT/prof_$1.ncu-rep ]; then
    python scripts/ncu_summary.py $OUT/prof_$1.ncu-rep > $OUT/prof_$1.summary.txt 2>&1
    python scripts/sass_lines.py $OUT/prof_$1.ncu-rep paper_1610_01050_b200/librsft.so 40 > $OUT/prof_$1.lines.txt 2>&1
    rm -f $OUT/prof_$1.ncu-rep
  fi
}
prof c4_k_fused2v c4_batched_2d 4096 k_fused2v
prof c2_k_fused2v c2_2d 8192 k_fused2v
echo done

#!/bin/bash
# c5 tail kernels: launch list + ncu source-line captures of k_split_fft, k_etab, k_vote; k_fused2v at c4
set -u
OUT=gpurun_out/bb; mkdir -p $OUT
prof() {   # name workload frames kernel-regex
  CMD="python bench.py --workload $2 --frames $3 --steps 2 --warmup 3 --no-cpu --no-e2e"
  ncu --set full --clock-control none --import-source on -k regex:$4 -s 1 -c 1 -o $OUT/prof_$1 -f $CMD > $OUT/ncu_$1.log 2>&1
  if [ -f $OUT/prof_$1.ncu-rep ]; then
    python scripts/ncu_summary.py $OUT/prof_$1.ncu-rep > $OUT/prof_$1.summary.txt 2>&1
    python scripts/sass_lines.py $OUT/prof_$1.ncu-rep paper_1610_01050_b200/librsft.so 40 > $OUT/prof_$1.lines.txt 2>&1
    rm -f $OUT/prof_$1.ncu-rep
  fi
}
python bench.py --workload c5_cube --no-cpu --no-e2e > $OUT/bench_c5.json 2> $OUT/bench_c5.err
CMD="python bench.py --workload c5_cube --steps 2 --warmup 3 --no-cpu --no-e2e"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c5.csv $CMD > /dev/null 2>&1
prof c5_k_split_fft c5_cube 1 k_split_fft
prof c5_k_etab c5_cube 1 k_etab
prof c5_k_vote c5_cube 1 'k_vote<'
prof c4_k_fused2v c4_batched_2d 4096 k_fused2v
echo done

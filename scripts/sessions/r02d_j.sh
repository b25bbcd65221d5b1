#!/bin/bash
# k_fused2v with 16-row (8-KiB) TMA boxes and 2 ring stages by default: smoke, GPU suite, final c4 (full line) and
# c2 lines, launch lists, ncu captures.
set -u
OUT=gpurun_out/dj; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests/ -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
python bench.py > $OUT/bench_c4.json 2> $OUT/bench_c4.err
python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e > $OUT/bench_c2.json 2> $OUT/bench_c2.err
for wl in c4_batched_2d:4096 c2_2d:8192; do
  w=${wl%%:*}; f=${wl##*:}
  CMD="python bench.py --workload $w --frames $f --steps 2 --warmup 3 --no-cpu --no-e2e"
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
    --log-file $OUT/launches_$w.csv $CMD > /dev/null 2>&1
done
prof() {   # name workload frames kernel-regex
  CMD="python bench.py --workload $2 --frames $3 --steps 2 --warmup 3 --no-cpu --no-e2e"
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$4 -s 1 -c 1 -o $OUT/prof_$1 -f $CMD > $OUT/ncu_$1.log 2>&1
  if [ -f $OUT/prof_$1.ncu-rep ]; then
    python scripts/ncu_summary.py $OUT/prof_$1.ncu-rep > $OUT/prof_$1.summary.txt 2>&1
    python scripts/sass_lines.py $OUT/prof_$1.ncu-rep paper_1610_01050_b200/librsft.so 30 > $OUT/prof_$1.lines.txt 2>&1
    rm -f $OUT/prof_$1.ncu-rep
  fi
}
prof c4_k_fused2v c4_batched_2d 4096 k_fused2v
prof c2_k_fused2v c2_2d 8192 k_fused2v
echo done

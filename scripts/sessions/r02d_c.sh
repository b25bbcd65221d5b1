#!/bin/bash
# k_region_scan_write<WPR> (4 warps per region list for large frames): GPU suite, c4 / c2 A/B against the
# two-pass scan + writer (RSFT_NO_SCANWRITE=1), clean c3 line, launch lists, ncu capture of the writer.
set -u
OUT=gpurun_out/dc; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu --timeout 1200 > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
for rep in 1 2; do
  python bench.py --no-cpu --no-e2e > $OUT/bench_c4_$rep.json 2> $OUT/bench_c4_$rep.err
  RSFT_NO_SCANWRITE=1 python bench.py --no-cpu --no-e2e > $OUT/bench_c4_old_$rep.json 2> $OUT/bench_c4_old_$rep.err
  python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e > $OUT/bench_c2_$rep.json 2> $OUT/bench_c2_$rep.err
  RSFT_NO_SCANWRITE=1 python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e > $OUT/bench_c2_old_$rep.json 2> $OUT/bench_c2_old_$rep.err
done
python bench.py > $OUT/bench_c4.json 2> $OUT/bench_c4.err
python bench.py --two-calls --no-cpu --no-e2e > $OUT/bench_c4_two.json 2> $OUT/bench_c4_two.err
python bench.py --workload c3_3d --frames 256 --steps 20 --no-cpu --no-e2e > $OUT/bench_c3.json 2> $OUT/bench_c3.err
for wl in c4_batched_2d:4096 c2_2d:8192; do
  w=${wl%%:*}; f=${wl##*:}
  CMD="python bench.py --workload $w --frames $f --steps 2 --warmup 3 --no-cpu --no-e2e"
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
    --log-file $OUT/launches_$w.csv $CMD > /dev/null 2>&1
done
python scripts/launches.py $OUT/launches_c4_batched_2d.csv $OUT/launches_c2_2d.csv > $OUT/launches.txt 2>&1
CMD="python bench.py --workload c4_batched_2d --frames 4096 --steps 2 --warmup 3 --no-cpu --no-e2e"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_region_scan_write -s 1 -c 1 -o $OUT/prof_c4_k_region_scan_write -f $CMD > $OUT/ncu_rsw.log 2>&1
if [ -f $OUT/prof_c4_k_region_scan_write.ncu-rep ]; then
  python scripts/ncu_summary.py $OUT/prof_c4_k_region_scan_write.ncu-rep > $OUT/prof_c4_k_region_scan_write.summary.txt 2>&1
  python scripts/sass_lines.py $OUT/prof_c4_k_region_scan_write.ncu-rep paper_1610_01050_b200/librsft.so 20 > $OUT/prof_c4_k_region_scan_write.lines.txt 2>&1
  rm -f $OUT/prof_c4_k_region_scan_write.ncu-rep
fi
echo done

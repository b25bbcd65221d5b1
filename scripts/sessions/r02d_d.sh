#!/bin/bash
# Final lines on the final code: GPU suite, smoke, every bench line, launch lists with DRAM bytes,
# k_fused2v ring-depth sweep (RSFT_F2V_STAGES), ncu captures of k_fused2v and the one-launch writer.
set -u
OUT=gpurun_out/dd; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $OUT/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -q -m gpu --timeout 1200 > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
python bench.py > $OUT/bench_c4.json 2> $OUT/bench_c4.err
python bench.py --impl reference --steps 2 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
python bench.py --workload c5_cube --steps 50 --no-cpu --no-e2e > $OUT/bench_c5.json 2> $OUT/bench_c5.err
python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e > $OUT/bench_c1.json 2> $OUT/bench_c1.err
python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e > $OUT/bench_c2.json 2> $OUT/bench_c2.err
python bench.py --workload c3_3d --frames 256 --steps 20 --no-cpu --no-e2e > $OUT/bench_c3.json 2> $OUT/bench_c3.err
python bench.py --two-calls --no-cpu --no-e2e > $OUT/bench_c4_two.json 2> $OUT/bench_c4_two.err
for s in 2 3; do
  RSFT_F2V_STAGES=$s python bench.py --no-cpu --no-e2e > $OUT/sweep_c4_stages$s.json 2> $OUT/sweep_c4_stages$s.err
  RSFT_F2V_STAGES=$s python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e > $OUT/sweep_c2_stages$s.json 2> $OUT/sweep_c2_stages$s.err
done
for wl in c4_batched_2d:4096 c1_1d:131072 c3_3d:256 c2_2d:8192 c5_cube:1; do
  w=${wl%%:*}; f=${wl##*:}
  CMD="python bench.py --workload $w --frames $f --steps 2 --warmup 3 --no-cpu --no-e2e"
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
    --log-file $OUT/launches_$w.csv $CMD > /dev/null 2>&1
done
prof() {   # name workload frames kernel-regex
  CMD="python bench.py --workload $2 --frames $3 --steps 2 --warmup 3 --no-cpu --no-e2e"
  timeout 500 ncu --set full --clock-control none --import-source on -k regex:$4 -s 1 -c 1 -o $OUT/prof_$1 -f $CMD > $OUT/ncu_$1.log 2>&1
  if [ -f $OUT/prof_$1.ncu-rep ]; then
    python scripts/ncu_summary.py $OUT/prof_$1.ncu-rep > $OUT/prof_$1.summary.txt 2>&1
    python scripts/sass_lines.py $OUT/prof_$1.ncu-rep paper_1610_01050_b200/librsft.so 30 > $OUT/prof_$1.lines.txt 2>&1
    rm -f $OUT/prof_$1.ncu-rep
  fi
}
prof c4_k_fused2v c4_batched_2d 4096 k_fused2v
prof c4_k_region_scan_write c4_batched_2d 4096 k_region_scan_write
prof c2_k_fused2v c2_2d 8192 k_fused2v
prof c2_k_region_scan_write c2_2d 8192 k_region_scan_write
echo done

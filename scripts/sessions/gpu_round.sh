#!/bin/bash
# Full GPU session: smoke, full parity, bench (+e2e, cpu baseline), c5 benches, reference arm,
# launch lists (c4, c5), ncu --set full of the dominant kernels (k_fused at c4, k_split_mma at c5).
set -u
mkdir -p gpurun_out
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $OUT/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
python -m pytest tests -q -m gpu --timeout 1500 > $OUT/parity_full.log 2>&1; echo "pytest rc=$?" >> $OUT/parity_full.log
python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
python bench.py --workload c5_cube --no-cpu --no-e2e > $OUT/bench_c5.json 2> $OUT/bench_c5.err
python bench.py --workload c5_cube --no-cpu --no-e2e --c5-variant A > $OUT/bench_c5A.json 2> $OUT/bench_c5A.err
python bench.py --impl reference --steps 2 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e > $OUT/bench_c1.json 2> $OUT/bench_c1.err
python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e > $OUT/bench_c2.json 2> $OUT/bench_c2.err
python bench.py --workload c3_3d --frames 256 --steps 10 --no-cpu --no-e2e > $OUT/bench_c3.json 2> $OUT/bench_c3.err
for wl in c4_batched_2d c5_cube; do
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --workload $wl"
  $CMD > $OUT/plain_$wl.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -c 60 --csv \
      --log-file $OUT/launches_$wl.csv $CMD > $OUT/ncu_launches_$wl.log 2>&1
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 -o $OUT/prof_k_fused -f $CMD > $OUT/ncu_full_c4.log 2>&1
CMD5="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --workload c5_cube"
ncu --set full --clock-control none --import-source on -k regex:k_split_mma -s 1 -c 1 -o $OUT/prof_k_split_mma -f $CMD5 > $OUT/ncu_full_c5.log 2>&1
RSFT_NO_MMA=1 ncu --set full --clock-control none --import-source on -k regex:k_split_fold -s 1 -c 1 -o $OUT/prof_k_split_fold -f $CMD5 > $OUT/ncu_full_c5_ffma.log 2>&1

# keep the copy-back under the 64 MiB limit: summaries on the box, full reports only if small
for r in $OUT/prof_k_fused $OUT/prof_k_split_mma $OUT/prof_k_split_fold; do
  [ -f $r.ncu-rep ] && python scripts/ncu_summary.py $r.ncu-rep > $r.summary.txt 2>&1
done
rm -f $OUT/prof_k_split_fold.ncu-rep $OUT/prof_k_fused.ncu-rep
echo done

#!/bin/bash
# Full GPU session: smoke, full parity, bench (+e2e, cpu baseline), launch list, ncu capture.
set -u
mkdir -p gpurun_out
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $OUT/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
python -m pytest tests -q -m gpu --timeout 1500 > $OUT/parity_full.log 2>&1; echo "pytest rc=$?" >> $OUT/parity_full.log
python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
python bench.py --workload c5_cube --no-cpu --no-e2e > $OUT/bench_c5.json 2> $OUT/bench_c5.err
python bench.py --impl reference --steps 2 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$CMD > $OUT/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
$CMD > $OUT/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 -o $OUT/prof_fused_r01 -f $CMD > $OUT/ncu_full.log 2>&1
CMD5="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --workload c5_cube"
$CMD5 > $OUT/plain5.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c5.csv $CMD5 > $OUT/ncu_launches5.log 2>&1
echo done

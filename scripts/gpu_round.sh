#!/bin/bash
# One GPU session: smoke, bench, ncu launch list + full capture of the top kernel, full-size parity.
set -u
mkdir -p gpurun_out
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$CMD > $OUT/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
$CMD > $OUT/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 -o $OUT/prof_fused $CMD > $OUT/ncu_full.log 2>&1
python -m pytest tests/test_gpu_parity.py -q -k "c4 or c5" --timeout 900 > $OUT/full_parity.log 2>&1
echo done

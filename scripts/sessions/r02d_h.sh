#!/bin/bash
# Final check with the driver's own commands on the final code: smoke, pytest -m gpu -x, bench.py (default),
# bench.py --impl reference, then the ncu launch list of the default bench command.
set -u
OUT=gpurun_out/dh; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests/ -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
python bench.py > $OUT/bench_c4.json 2> $OUT/bench_c4.err
python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e > $OUT/bench_c2.json 2> $OUT/bench_c2.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches_default_bench.csv python bench.py --no-cpu > $OUT/ncu_default.log 2>&1
python scripts/launches.py $OUT/launches_default_bench.csv > $OUT/launches_default_bench.txt 2>&1
echo done

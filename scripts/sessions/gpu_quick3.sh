#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x --timeout 1500 > gpurun_out/q3_parity.log 2>&1; tail -2 gpurun_out/q3_parity.log
python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e > gpurun_out/q3_bench_c1.json 2> gpurun_out/q3_bench_c1.err
ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -c 40 --csv --log-file gpurun_out/q3_ll_c1.csv python bench.py --workload c1_1d --frames 131072 --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
echo done

#!/bin/bash
# quick loop: CI parity + bench (no CPU/e2e) + launch list
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -x -k "not c5 and not c4" --timeout 300 > gpurun_out/q_parity.log 2>&1; tail -3 gpurun_out/q_parity.log
CMD="python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/q_launches.csv $CMD > /dev/null 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --workload c5_cube > gpurun_out/q_bench_c5.json 2> gpurun_out/q_bench_c5.err
echo done

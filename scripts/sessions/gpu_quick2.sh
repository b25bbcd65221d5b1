#!/bin/bash
# full GPU parity + c4/c5 launch lists + short benches (no CPU baseline / e2e)
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x --timeout 1500 > gpurun_out/q2_parity.log 2>&1; tail -2 gpurun_out/q2_parity.log
python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/q2_bench_c4.json 2> gpurun_out/q2_bench_c4.err
python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --workload c5_cube > gpurun_out/q2_bench_c5.json 2> gpurun_out/q2_bench_c5.err
python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --workload c5_cube --c5-variant A > gpurun_out/q2_bench_c5A.json 2> gpurun_out/q2_bench_c5A.err
for wl in c4_batched_2d c5_cube; do
  ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -c 40 --csv --log-file gpurun_out/q2_launches_$wl.csv python bench.py --workload $wl --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
echo done

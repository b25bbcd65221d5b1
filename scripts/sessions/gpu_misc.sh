#!/bin/bash
# sanitizers on small cases + bench lines of c1/c2/c3 batched variants + refreshed c4 bench
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_cases.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_summary.txt
done
python bench.py --workload c2_2d --frames 8192 --no-cpu --no-e2e > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --workload c1_1d --frames 131072 --no-cpu --no-e2e > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
python bench.py --workload c3_3d --frames 256 --pool 16 --no-cpu --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo done

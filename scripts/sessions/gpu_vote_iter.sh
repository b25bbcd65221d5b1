#!/bin/bash
# Vote iteration: GPU tests, c4 bench line, c4 + c5 launch lists.
mkdir -p gpurun_out
TAG=${1:-v}
python -m pytest tests -q -m gpu -x --timeout 1500 > gpurun_out/${TAG}_parity.log 2>&1; tail -1 gpurun_out/${TAG}_parity.log
python bench.py --steps 10 --no-cpu --no-e2e > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}_c4.err
python -c "import json;d=json.load(open('gpurun_out/${TAG}_c4.json'));print('c4', d['value'], d['ms_per_step'])"
for wl in c4_batched_2d c5_cube; do
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --workload $wl"
  ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/${TAG}_ll_$wl.csv $CMD > /dev/null 2>&1
  python scripts/launches.py gpurun_out/${TAG}_ll_$wl.csv | head -6
done

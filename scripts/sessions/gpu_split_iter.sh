#!/bin/bash
# Split-mode iteration: parity of every GPU test, then the c5 bench line and a launch list.
mkdir -p gpurun_out
TAG=${1:-it}
python -m pytest tests -q -m gpu -x --timeout 1500 > gpurun_out/${TAG}_parity.log 2>&1; tail -3 gpurun_out/${TAG}_parity.log
python bench.py --workload c5_cube --steps 20 --no-cpu > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.err
python -c "import json;d=json.load(open('gpurun_out/${TAG}_c5.json'));print(d['value'],d['ms_per_step'],d['roofline'])"
ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/${TAG}_ll_c5.csv python bench.py --workload c5_cube --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
python scripts/launches.py gpurun_out/${TAG}_ll_c5.csv | head -12

#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/e_smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/e_smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 900 > $OUT/e_pytest.log 2>&1; echo "rc=$?" >> $OUT/e_pytest.log
python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e > $OUT/e_c1.json 2> $OUT/e_c1.err
python bench.py --workload c3_3d --frames 256 --steps 10 --no-cpu --no-e2e > $OUT/e_c3.json 2> $OUT/e_c3.err
python bench.py --no-cpu --no-e2e > $OUT/e_c4.json 2> $OUT/e_c4.err
C1="python bench.py --workload c1_1d --frames 131072 --steps 2 --warmup 3 --no-cpu --no-e2e"
$C1 > $OUT/e_plain_c1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/e_launches_c1.csv $C1 > /dev/null 2>&1
C3="python bench.py --workload c3_3d --frames 256 --steps 2 --warmup 3 --no-cpu --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/e_launches_c3.csv $C3 > /dev/null 2>&1
echo done

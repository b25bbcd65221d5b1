#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/g_smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/g_smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 900 > $OUT/g_pytest.log 2>&1; echo "rc=$?" >> $OUT/g_pytest.log
python bench.py --no-cpu --no-e2e > $OUT/g_c4.json 2> $OUT/g_c4.err
python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e > $OUT/g_c1.json 2> $OUT/g_c1.err
python bench.py --workload c3_3d --frames 256 --steps 10 --no-cpu --no-e2e > $OUT/g_c3.json 2> $OUT/g_c3.err
python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e > $OUT/g_c2.json 2> $OUT/g_c2.err
python bench.py --workload c5_cube --no-cpu --no-e2e > $OUT/g_c5.json 2> $OUT/g_c5.err
for wl in c1_1d:131072 c3_3d:256 c4_batched_2d:4096 c2_2d:8192; do
  w=${wl%%:*}; f=${wl##*:}
  CMD="python bench.py --workload $w --frames $f --steps 2 --warmup 3 --no-cpu --no-e2e"
  $CMD > $OUT/g_plain_$w.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/g_launches_$w.csv $CMD > /dev/null 2>&1
done
echo done

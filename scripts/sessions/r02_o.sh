#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "c4_full or compaction or run_host" > $OUT/o_tests.log 2>&1; echo "rc=$?" >> $OUT/o_tests.log
RSFT_COMPACT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "c4_full or compaction or 2d_fused or c2_shape" > $OUT/o_tests_compact.log 2>&1; echo "rc=$?" >> $OUT/o_tests_compact.log
python bench.py --no-cpu --no-e2e > $OUT/o_c4.json 2> $OUT/o_c4.err
RSFT_COMPACT=1 python bench.py --no-cpu --no-e2e > $OUT/o_c4_compact.json 2> $OUT/o_c4_compact.err
C4="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
RSFT_COMPACT=1 $C4 > $OUT/o_plain_c4.log 2>&1 && \
  RSFT_COMPACT=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/o_launches_c4_compact.csv $C4 > /dev/null 2>&1
for wl in c2_2d:8192 c3_3d:256 c1_1d:131072; do
  w=${wl%%:*}; f=${wl##*:}
  RSFT_COMPACT=1 python bench.py --workload $w --frames $f --steps 10 --no-cpu --no-e2e > $OUT/o_${w}_compact.json 2> $OUT/o_${w}_compact.err
  python bench.py --workload $w --frames $f --steps 10 --no-cpu --no-e2e > $OUT/o_${w}.json 2> $OUT/o_${w}.err
done
python bench.py --workload c5_cube --no-cpu --no-e2e > $OUT/o_c5.json 2> $OUT/o_c5.err
echo done

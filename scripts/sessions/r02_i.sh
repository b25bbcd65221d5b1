#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 1800 python -m pytest tests -q -m gpu -x --timeout 1200 > $OUT/i_pytest.log 2>&1; echo "rc=$?" >> $OUT/i_pytest.log
RSFT_VOTE2D=1 python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e > $OUT/i_c2_v2.json 2> $OUT/i_c2_v2.err
python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e > $OUT/i_c2.json 2> $OUT/i_c2.err
C3="python bench.py --workload c3_3d --frames 256 --steps 2 --warmup 3 --no-cpu --no-e2e"
$C3 > $OUT/i_plain_c3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_split_fft -s 1 -c 1 -o $OUT/i_prof_fft -f $C3 > $OUT/i_ncu_fft.log 2>&1
[ -f $OUT/i_prof_fft.ncu-rep ] && python scripts/ncu_summary.py $OUT/i_prof_fft.ncu-rep > $OUT/i_prof_fft.summary.txt 2>&1
echo done

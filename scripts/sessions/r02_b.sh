#!/bin/bash
# Round 2, session B: D = 1 gather-form kernel (k_gather1d): parity, c1 bench, launch list, ncu.
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/b_smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/b_smoke.log
timeout 900 python -m pytest tests -q -m gpu -x --timeout 600 -k "1d or c1 or smoke" > $OUT/b_pytest.log 2>&1; echo "rc=$?" >> $OUT/b_pytest.log
for cfg in "2 0" "1 0" "2 2" "2 4" "1 6"; do
  set -- $cfg
  RSFT_G1_CTAS=$1 RSFT_G1_STAGES=$2 python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e > $OUT/b_c1_$1_$2.json 2> $OUT/b_c1_$1_$2.err
done
C1="python bench.py --workload c1_1d --frames 131072 --steps 2 --warmup 3 --no-cpu --no-e2e"
$C1 > $OUT/b_plain_c1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/b_launches_c1.csv $C1 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_gather1d -s 1 -c 1 -o $OUT/b_prof_c1 -f $C1 > $OUT/b_ncu_c1.log 2>&1
[ -f $OUT/b_prof_c1.ncu-rep ] && python scripts/ncu_summary.py $OUT/b_prof_c1.ncu-rep > $OUT/b_prof_c1.summary.txt 2>&1
echo done

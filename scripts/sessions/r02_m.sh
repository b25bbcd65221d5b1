#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_bartlett.py -q -x --timeout 600 > $OUT/m_tests.log 2>&1; echo "rc=$?" >> $OUT/m_tests.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "segment" > $OUT/m_seg.log 2>&1; echo "rc=$?" >> $OUT/m_seg.log
for wl in c2_2d c4_batched_2d c3_3d; do
  python bench.py --workload $wl --bartlett --steps 5 > $OUT/m_bart_$wl.json 2> $OUT/m_bart_$wl.err
  python bench.py --workload $wl --segments --steps 5 > $OUT/m_seg_$wl.json 2> $OUT/m_seg_$wl.err
done
C="python bench.py --workload c4_batched_2d --bartlett --steps 2 --warmup 3"
$C > $OUT/m_plain_bart.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 20 --csv --log-file $OUT/m_launches_bart_c4.csv $C > /dev/null 2>&1
C="python bench.py --workload c3_3d --segments --steps 2 --warmup 3"
$C > $OUT/m_plain_seg.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/m_launches_seg_c3.csv $C > /dev/null 2>&1
C4="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$C4 > $OUT/m_plain_c4.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_vote -s 1 -c 1 -o $OUT/m_prof_vote -f $C4 > $OUT/m_ncu_vote.log 2>&1
[ -f $OUT/m_prof_vote.ncu-rep ] && python scripts/sass_lines.py $OUT/m_prof_vote.ncu-rep paper_1610_01050_b200/librsft.so 40 > $OUT/m_prof_vote.lines.txt 2>&1
[ -f $OUT/m_prof_vote.ncu-rep ] && python scripts/ncu_summary.py $OUT/m_prof_vote.ncu-rep > $OUT/m_prof_vote.summary.txt 2>&1
echo done

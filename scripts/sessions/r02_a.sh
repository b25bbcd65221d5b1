#!/bin/bash
# Round 2, session A: new parity tests, smoke (incl. k_split_mma), bench default, the
# multi-GPU code path on a 1-GPU lease (1-rank NCCL group), c1/c3 baselines + ncu captures.
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1200 python -m pytest tests -q -m gpu -x --timeout 900 -k "c4_full or c2_shape or mma or variant_b" > $OUT/pytest_new.log 2>&1; echo "rc=$?" >> $OUT/pytest_new.log
python bench.py > $OUT/bench.json 2> $OUT/bench.err
NCCL_DEBUG=INFO python bench.py --force-collectives --no-cpu --no-e2e > $OUT/bench_pg.json 2> $OUT/bench_pg.err
python bench.py --workload c5_cube --no-cpu --no-e2e > $OUT/c5_nopg.json 2> $OUT/c5_nopg.err
NCCL_DEBUG=INFO python bench.py --workload c5_cube --no-cpu --no-e2e --force-collectives --c5-variant A > $OUT/c5A_pg.json 2> $OUT/c5A_pg.err
NCCL_DEBUG=INFO python bench.py --workload c5_cube --no-cpu --no-e2e --force-collectives --c5-variant B > $OUT/c5B_pg.json 2> $OUT/c5B_pg.err
python bench.py --gpus 1 --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e > $OUT/bench_c1.json 2> $OUT/bench_c1.err
python bench.py --workload c3_3d --frames 256 --steps 10 --no-cpu --no-e2e > $OUT/bench_c3.json 2> $OUT/bench_c3.err
C1="python bench.py --workload c1_1d --frames 131072 --steps 2 --warmup 3 --no-cpu --no-e2e"
$C1 > $OUT/plain_c1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c1.csv $C1 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 -o $OUT/prof_c1_k_fused -f $C1 > $OUT/ncu_c1.log 2>&1
C3="python bench.py --workload c3_3d --frames 256 --steps 2 --warmup 3 --no-cpu --no-e2e"
$C3 > $OUT/plain_c3.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c3.csv $C3 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_split_fold -s 1 -c 1 -o $OUT/prof_c3_k_split_fold -f $C3 > $OUT/ncu_c3.log 2>&1
for r in $OUT/prof_c1_k_fused $OUT/prof_c3_k_split_fold; do
  [ -f $r.ncu-rep ] && python scripts/ncu_summary.py $r.ncu-rep > $r.summary.txt 2>&1
done
echo done

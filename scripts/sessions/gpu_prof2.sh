#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -x -k "not c5 and not c4" --timeout 300 > gpurun_out/q_parity.log 2>&1; tail -1 gpurun_out/q_parity.log
CMD="python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/q_launches.csv $CMD > /dev/null 2>&1
CMD5="python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --workload c5_cube"
$CMD5 > gpurun_out/q_bench_c5.json 2> gpurun_out/q_bench_c5.err
CMDS="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$CMDS > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_vote|k_compact" -s 2 -c 2 -o gpurun_out/prof_vote -f $CMDS > gpurun_out/n_vote.log 2>&1
CMDS5="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --workload c5_cube"
$CMDS5 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_split" -s 4 -c 2 -o gpurun_out/prof_split2 -f $CMDS5 > gpurun_out/n_split.log 2>&1
echo done

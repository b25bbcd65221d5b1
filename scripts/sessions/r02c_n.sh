#!/bin/bash
# k_vote3d with a cp.async double-buffered prefetch of the next region's E blocks: parity + c3 bench + launch list.
set -u
OUT=gpurun_out/n; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "3d or vote or c3 or seg or cube" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
C3="python bench.py --workload c3_3d --frames 256 --steps 20 --no-cpu --no-e2e"
timeout 300 $C3 > $OUT/c3.json 2> $OUT/c3.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c3.csv python bench.py --workload c3_3d --frames 256 --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
python scripts/launches.py $OUT/launches_c3.csv > $OUT/launches_c3.txt 2>&1
echo done

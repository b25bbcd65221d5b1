#!/bin/bash
# Round-2 final evidence on HEAD: smoke, full GPU suite, every bench line, Bartlett / segment lines,
# 1-rank NCCL collectives, launch lists with DRAM bytes, ncu --set full captures of the dominant kernels.
set -u
OUT=gpurun_out/da; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $OUT/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -q -m gpu --timeout 1200 > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
python bench.py > $OUT/bench_c4.json 2> $OUT/bench_c4.err
python bench.py --impl reference --steps 2 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
python bench.py --workload c5_cube --no-cpu --no-e2e > $OUT/bench_c5.json 2> $OUT/bench_c5.err
python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e > $OUT/bench_c1.json 2> $OUT/bench_c1.err
python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e > $OUT/bench_c2.json 2> $OUT/bench_c2.err
python bench.py --workload c3_3d --frames 256 --steps 10 --no-cpu --no-e2e > $OUT/bench_c3.json 2> $OUT/bench_c3.err
python bench.py --two-calls --no-cpu --no-e2e > $OUT/bench_c4_two.json 2> $OUT/bench_c4_two.err
for wl in c1_1d c2_2d c4_batched_2d c3_3d; do
  python bench.py --workload $wl --bartlett --steps 5 > $OUT/bart_$wl.json 2> $OUT/bart_$wl.err
  python bench.py --workload $wl --segments --steps 5 > $OUT/seg_$wl.json 2> $OUT/seg_$wl.err
done
NCCL_DEBUG=INFO python bench.py --force-collectives --no-cpu --no-e2e > $OUT/coll_c4.json 2> $OUT/coll_c4.err
NCCL_DEBUG=INFO python bench.py --force-collectives --workload c5_cube --c5-variant A --no-cpu --no-e2e > $OUT/coll_c5A.json 2> $OUT/coll_c5A.err
NCCL_DEBUG=INFO python bench.py --force-collectives --workload c5_cube --c5-variant B --no-cpu --no-e2e > $OUT/coll_c5B.json 2> $OUT/coll_c5B.err
for wl in c4_batched_2d:4096 c1_1d:131072 c3_3d:256 c2_2d:8192 c5_cube:1; do
  w=${wl%%:*}; f=${wl##*:}
  CMD="python bench.py --workload $w --frames $f --steps 2 --warmup 3 --no-cpu --no-e2e"
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
    --log-file $OUT/launches_$w.csv $CMD > /dev/null 2>&1
done
prof() {   # name workload frames kernel-regex [extra bench args]
  CMD="python bench.py --workload $2 --frames $3 --steps 2 --warmup 3 --no-cpu --no-e2e ${5:-}"
  timeout 500 ncu --set full --clock-control none --import-source on -k regex:$4 -s 1 -c 1 -o $OUT/prof_$1 -f $CMD > $OUT/ncu_$1.log 2>&1
  if [ -f $OUT/prof_$1.ncu-rep ]; then
    python scripts/ncu_summary.py $OUT/prof_$1.ncu-rep > $OUT/prof_$1.summary.txt 2>&1
    python scripts/sass_lines.py $OUT/prof_$1.ncu-rep paper_1610_01050_b200/librsft.so 30 > $OUT/prof_$1.lines.txt 2>&1
    rm -f $OUT/prof_$1.ncu-rep
  fi
}
prof c4_k_fused2v c4_batched_2d 4096 k_fused2v
prof c3_k_split_fold c3_3d 256 k_split_fold
prof c3_k_split_fft_wr c3_3d 256 k_split_fft_wr
prof c3_k_vote3d c3_3d 256 k_vote3d
prof c5_k_split_mma c5_cube 1 k_split_mma
prof c5_k_vote c5_cube 1 "k_vote<"
CB="python bench.py --workload c1_1d --bartlett --steps 2 --warmup 3"
timeout 500 ncu --set full --clock-control none --import-source on -k regex:k_bart -s 1 -c 1 -o $OUT/prof_c1_bart -f $CB > $OUT/ncu_c1_bart.log 2>&1
if [ -f $OUT/prof_c1_bart.ncu-rep ]; then
  python scripts/ncu_summary.py $OUT/prof_c1_bart.ncu-rep > $OUT/prof_c1_bart.summary.txt 2>&1
  rm -f $OUT/prof_c1_bart.ncu-rep
fi
echo done

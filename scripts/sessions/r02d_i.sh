#!/bin/bash
# k_fused2v TMA box size: tuning builds with 4-row (2-KiB) and 16-row (8-KiB) boxes (build/var, -DRSFT_F2V_U)
# against the default 8 rows, each at several ring depths; c4 and c2 lines (digests must equal the default's).
set -u
OUT=gpurun_out/di; mkdir -p $OUT
run() {  # tag lib stages
  RSFT_LIB=$2 RSFT_F2V_STAGES=$3 python bench.py --no-cpu --no-e2e --steps 10 > $OUT/c4_$1_s$3.json 2> $OUT/c4_$1_s$3.err
  RSFT_LIB=$2 RSFT_F2V_STAGES=$3 python bench.py --workload c2_2d --frames 8192 --steps 10 --no-cpu --no-e2e > $OUT/c2_$1_s$3.json 2> $OUT/c2_$1_s$3.err
}
run u8 paper_1610_01050_b200/librsft.so 3
run u16 build/var/librsft_u16.so 2
run u16 build/var/librsft_u16.so 3
run u4 build/var/librsft_u4.so 4
run u4 build/var/librsft_u4.so 5
run u4 build/var/librsft_u4.so 6
run u8 paper_1610_01050_b200/librsft.so 3
echo done

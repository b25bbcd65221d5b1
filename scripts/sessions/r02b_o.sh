#!/bin/bash
# c1: is the fused kernel bound by its loop warps (one CTA per SM) or by the vote warps?
set -u
OUT=gpurun_out/bo; mkdir -p $OUT
RSFT_G1_CTAS=1 python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e --two-calls > $OUT/c1_two_cta1.json 2> $OUT/c1_two_cta1.err
python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e --two-calls > $OUT/c1_two_cta2.json 2> $OUT/c1_two_cta2.err
for nv in 4 8 12 16; do
  RSFT_G1_VOTE_WARPS=$nv python bench.py --workload c1_1d --frames 131072 --steps 10 --no-cpu --no-e2e > $OUT/c1_nv$nv.json 2> $OUT/c1_nv$nv.err
done
echo done

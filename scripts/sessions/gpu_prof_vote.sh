#!/bin/bash
mkdir -p gpurun_out
python scripts/vote_variants.py > gpurun_out/vv.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_vote|k_compact" -s 3 -c 3 -o gpurun_out/prof_vote3 -f python scripts/vote_variants.py > gpurun_out/n_vote.log 2>&1
echo done

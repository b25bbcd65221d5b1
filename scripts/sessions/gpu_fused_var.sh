#!/bin/bash
# k_fused ring variants at c4: bench line (k_fused avg launch from the bench's CUDA events) per library.
mkdir -p gpurun_out
for so in ${VARS}; do
  n=$(basename $so .so)
  RSFT_LIB=$so python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/fv_$n.json 2> gpurun_out/fv_$n.err
  python -c "import json;d=json.load(open('gpurun_out/fv_$n.json'));r=d['roofline'];print('$n', round(d['value']), round(d['ms_per_step'],4), round(r['avg_launch_ms'],4), round(r['frac'],4))" 2>/dev/null || (echo "$n failed"; tail -2 gpurun_out/fv_$n.err)
done

for so in paper_1610_01050_b200/librsft.so build/var/librsft_vote3.so build/var/librsft_vote5.so; do
  RSFT_LIB=$so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_vote -c 8 --csv --log-file gpurun_out/vv_$(basename $so .so).csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
  echo "== $so"; python scripts/launches.py gpurun_out/vv_$(basename $so .so).csv | head -2
done

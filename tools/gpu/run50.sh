for r in 1 2; do for v in bl256 bl512 bl1024; do
  L=build_var/$v/libamppi_b200.so
  AMPPI_ABI_LENIENT=1 AMPPI_LIB_PATH=$L python bench.py --workload c4 --steps 10 --warmup 3 --cpu-seconds 1 > gpurun_out/r50_${v}_$r.log 2>&1
  grep -o '"ms_per_step": [0-9.]*' gpurun_out/r50_${v}_$r.log | head -1 | sed "s/^/$v rep=$r /"
done; done

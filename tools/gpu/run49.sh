for r in 1 2; do for v in cur bl64 bl128 bl256; do
  if [ $v = cur ]; then L=paper_2509_17340_b200/libamppi_b200.so; else L=build_var/$v/libamppi_b200.so; fi
  AMPPI_ABI_LENIENT=1 AMPPI_LIB_PATH=$L python bench.py --workload c4 --steps 10 --warmup 3 --cpu-seconds 1 > gpurun_out/r49_${v}_$r.log 2>&1
  grep -o '"ms_per_step": [0-9.]*' gpurun_out/r49_${v}_$r.log | head -1 | sed "s/^/$v rep=$r /"
done; done

for r in 1 2; do for v in ppt8 ppt4 ppt2 ppt1; do
  if [ $v = ppt8 ]; then L=paper_2509_17340_b200/libamppi_b200.so; else L=build_var/$v/libamppi_b200.so; fi
  AMPPI_LIB_PATH=$L python bench.py --steps 2 --warmup 3 --cpu-seconds 1 --no-e2e --latency-cycles 2000 > gpurun_out/r78_${v}_$r.log 2>&1
  AMPPI_LIB_PATH=$L python bench.py --workload c3 --steps 20 --warmup 3 --cpu-seconds 1 > gpurun_out/r78_c3_${v}_$r.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/r78_${v}_$r.log').read().strip().splitlines()[-1]); l=d['latency']
c=json.loads(open('gpurun_out/r78_c3_${v}_$r.log').read().strip().splitlines()[-1]); k=c.get('kernels',{}).get('k_key_points',{})
print('$v', $r, 'c1 p50', round(l['p50_ms'],4), 'c3', round(c['ms_per_step'],4), 'c3 keying', round(k.get('ms_total',0)/max(k.get('launches',1),1)*1000,1))"
done; done

python -m pytest tests/test_plan_parity.py tests/test_dmax_boundary.py tests/test_gpu_loop.py tests/test_closed_loop_replay.py tests/test_shim.py tests/test_config_sizes.py -q > gpurun_out/r81_pytest.log 2>&1; echo pytest rc=$?
for r in 1 2 3; do for v in old new; do
  if [ $v = new ]; then L=paper_2509_17340_b200/libamppi_b200.so; else L=build_var/nohint/libamppi_b200.so; fi
  AMPPI_LIB_PATH=$L python bench.py --steps 2 --warmup 3 --cpu-seconds 1 --no-e2e --latency-cycles 2000 > gpurun_out/r81_${v}_$r.log 2>&1
  AMPPI_LIB_PATH=$L python bench.py --workload c3 --steps 20 --warmup 3 --cpu-seconds 1 > gpurun_out/r81_c3_${v}_$r.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/r81_${v}_$r.log').read().strip().splitlines()[-1]); l=d['latency']
c=json.loads(open('gpurun_out/r81_c3_${v}_$r.log').read().strip().splitlines()[-1]); k=c.get('kernels',{}).get('k_stage1_warp32',{})
print('$v', $r, 'c1 p50', round(l['p50_ms'],4), 'paper', round(l['paper_default']['p50_ms'],4), 'c3', round(c['ms_per_step'],4), 'c3 stage1', round(k.get('ms_total',0)/max(k.get('launches',1),1)*1000,1))"
done; done

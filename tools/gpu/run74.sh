python -m pytest tests/test_snapshot_parity.py tests/test_plan_parity.py tests/test_config_sizes.py tests/test_gpu_loop.py tests/test_closed_loop_replay.py tests/test_shim.py -q > gpurun_out/r74_pytest.log 2>&1; echo pytest rc=$?
for r in 1 2 3; do for v in old new; do
  if [ $v = new ]; then L=paper_2509_17340_b200/libamppi_b200.so; else L=build_var/cloold/libamppi_b200.so; fi
  AMPPI_LIB_PATH=$L python bench.py --steps 2 --warmup 3 --cpu-seconds 1 --no-e2e --latency-cycles 2000 > gpurun_out/r74_${v}_$r.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/r74_${v}_$r.log').read().strip().splitlines()[-1]); l=d['latency']; print('$v', $r, round(l['p50_ms'],4), round(l['paper_default']['p50_ms'],4))"
  AMPPI_LIB_PATH=$L python bench.py --workload c3 --steps 20 --warmup 3 --cpu-seconds 1 > gpurun_out/r74_c3_${v}_$r.log 2>&1
  grep -o '"ms_per_step": [0-9.]*' gpurun_out/r74_c3_${v}_$r.log | head -1 | sed "s/^/c3 $v $r /"
done; done

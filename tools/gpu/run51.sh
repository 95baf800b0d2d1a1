python -m pytest tests/test_config_sizes.py tests/test_sample_sharding.py tests/test_plan_parity.py tests/test_dist_gloo.py -q > gpurun_out/r51_pytest.log 2>&1; echo pytest rc=$?
for r in 1 2 3; do python bench.py --workload c4 --steps 10 --warmup 3 --cpu-seconds 1 > gpurun_out/r51_c4_$r.log 2>&1; grep -o '"ms_per_step": [0-9.]*' gpurun_out/r51_c4_$r.log | head -1; done
python bench.py --steps 10 --warmup 3 --no-latency --cpu-seconds 1 --no-e2e > gpurun_out/r51_c5.log 2>&1; grep -o '"ms_per_step": [0-9.]*' gpurun_out/r51_c5.log | head -1

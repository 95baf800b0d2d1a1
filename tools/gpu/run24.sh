cat /dev/null
python -m pytest tests/test_plan_parity.py tests/test_gpu_loop.py tests/test_closed_loop_replay.py tests/test_shim.py tests/test_sample_sharding.py tests/test_dmax_boundary.py -x -q > gpurun_out/r24_pytest.log 2>&1; echo pytest rc=$?
python bench.py --steps 10 --warmup 3 --no-e2e --cpu-seconds 1 > gpurun_out/r24_c5.log 2>&1; echo c5 rc=$?

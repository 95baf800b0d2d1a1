python tools/diag_keying.py > gpurun_out/r14_diag.log 2>&1; echo diag rc=$?
python -m pytest tests/test_snapshot_parity.py tests/test_batch_ragged.py tests/test_plan_parity.py tests/test_config_sizes.py tests/test_gpu_loop.py tests/test_shim.py tests/test_io.py -x -q > gpurun_out/r14_pytest.log 2>&1; echo pytest rc=$?
timeout 300 python bench.py --workload c3 --steps 5 --warmup 2 > gpurun_out/r14_c3.log 2>&1; echo c3 rc=$?
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --cpu-seconds 1 > gpurun_out/r14_c5.log 2>&1; echo c5 rc=$?

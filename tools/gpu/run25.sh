python -m pytest tests/test_snapshot_parity.py tests/test_batch_ragged.py tests/test_plan_parity.py tests/test_batch_parity.py tests/test_gpu_loop.py tests/test_config_sizes.py -x -q > gpurun_out/r25_pytest.log 2>&1; echo pytest rc=$?
python tools/ab.py bitonic:build_var/bitonic/libamppi_b200.so count:paper_2509_17340_b200/libamppi_b200.so 3 > gpurun_out/r25_ab.log 2>&1; echo ab rc=$?
python bench.py --steps 10 --warmup 3 --no-e2e --cpu-seconds 1 > gpurun_out/r25_c5.log 2>&1; echo c5 rc=$?

cat gpurun_out/r15_c3.log > /dev/null 2>&1
python -m pytest tests/test_plan_parity.py tests/test_batch_parity.py tests/test_batch_ragged.py tests/test_gpu_loop.py tests/test_config_sizes.py tests/test_sample_sharding.py -x -q > gpurun_out/r16_pytest.log 2>&1; echo pytest rc=$?
python tools/ab.py old:build_var/warpcol/libamppi_b200.so new:paper_2509_17340_b200/libamppi_b200.so 3 > gpurun_out/r16_ab.log 2>&1; echo ab rc=$?

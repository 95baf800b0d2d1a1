python -m pytest tests/test_snapshot_parity.py tests/test_batch_ragged.py tests/test_batch_parity.py tests/test_plan_parity.py tests/test_config_sizes.py -q > gpurun_out/r73_pytest.log 2>&1; echo pytest rc=$?
python tools/ab.py nodefer:build_var/nodefer/libamppi_b200.so defer:paper_2509_17340_b200/libamppi_b200.so 3 > gpurun_out/r73_ab.log 2>&1; echo ab rc=$?

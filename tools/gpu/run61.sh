python -m pytest tests/test_plan_parity.py tests/test_batch_parity.py tests/test_config_sizes.py tests/test_screen_drift.py tests/test_dmax_boundary.py -q -x > gpurun_out/r61_pytest.log 2>&1; echo pytest rc=$?
python tools/ab.py noreach:build_var/noreach/libamppi_b200.so reach:paper_2509_17340_b200/libamppi_b200.so 3 > gpurun_out/r61_ab.log 2>&1; echo ab rc=$?

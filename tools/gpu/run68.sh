python -m pytest tests/test_snapshot_parity.py tests/test_batch_parity.py tests/test_plan_parity.py tests/test_config_sizes.py tests/test_screen_drift.py -q > gpurun_out/r68_pytest.log 2>&1; echo pytest rc=$?
python tools/ab.py leafd:build_var/leafd/libamppi_b200.so leaff:paper_2509_17340_b200/libamppi_b200.so 3 > gpurun_out/r68_ab.log 2>&1; echo ab rc=$?

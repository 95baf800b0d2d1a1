python -m pytest tests/test_plan_parity.py tests/test_config_sizes.py tests/test_batch_parity.py tests/test_dmax_boundary.py tests/test_sample_sharding.py -q > gpurun_out/r36_pytest.log 2>&1; echo pytest rc=$?
python tools/ab.py nocas:build_var/nocascade/libamppi_b200.so cas:paper_2509_17340_b200/libamppi_b200.so 3 > gpurun_out/r36_ab.log 2>&1; echo ab rc=$?

AMPPI_LIB_PATH=build_var/colpts/libamppi_b200.so python -m pytest tests/test_plan_parity.py tests/test_config_sizes.py tests/test_batch_parity.py -q -x > gpurun_out/r46_pytest_colpts.log 2>&1; echo pytest colpts rc=$?
AMPPI_LIB_PATH=build_var/repackpop/libamppi_b200.so python -m pytest tests/test_plan_parity.py tests/test_config_sizes.py tests/test_batch_parity.py -q -x > gpurun_out/r46_pytest_repack.log 2>&1; echo pytest repack rc=$?
python -m pytest tests/test_plan_parity.py tests/test_batch_parity.py -q -x > gpurun_out/r46_pytest.log 2>&1; echo pytest rc=$?
python tools/ab.py cur:paper_2509_17340_b200/libamppi_b200.so colpts:build_var/colpts/libamppi_b200.so repackpop:build_var/repackpop/libamppi_b200.so 3 > gpurun_out/r46_ab.log 2>&1; echo ab rc=$?

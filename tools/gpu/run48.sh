AMPPI_LIB_PATH=build_var/repackhit/libamppi_b200.so python -m pytest tests/test_plan_parity.py tests/test_batch_parity.py -q -x > gpurun_out/r48_pytest.log 2>&1; echo pytest rc=$?
python tools/ab.py cur:paper_2509_17340_b200/libamppi_b200.so hit:build_var/repackhit/libamppi_b200.so 3 > gpurun_out/r48_ab.log 2>&1; echo ab rc=$?

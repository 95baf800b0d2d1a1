python -m pytest tests/test_plan_parity.py tests/test_batch_parity.py -q -x > gpurun_out/r71_pytest.log 2>&1; echo pytest rc=$?
python tools/ab.py bw1:build_var/bw1/libamppi_b200.so bw4m10:paper_2509_17340_b200/libamppi_b200.so bw4m8:build_var/bw4m8/libamppi_b200.so bw2m16:build_var/bw2m16/libamppi_b200.so 3 > gpurun_out/r71_ab.log 2>&1; echo ab rc=$?

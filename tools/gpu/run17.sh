python -m pytest tests/test_plan_parity.py tests/test_batch_parity.py tests/test_gpu_loop.py -x -q > gpurun_out/r17_pytest.log 2>&1; echo pytest rc=$?
python tools/ab.py old:build_var/warpcol/libamppi_b200.so run4:paper_2509_17340_b200/libamppi_b200.so run1:build_var/colrun1/libamppi_b200.so run8:build_var/colrun8/libamppi_b200.so 3 > gpurun_out/r17_ab.log 2>&1; echo ab rc=$?

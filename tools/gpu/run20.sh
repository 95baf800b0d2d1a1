python -m pytest tests/test_plan_parity.py tests/test_batch_parity.py tests/test_gpu_loop.py -x -q > gpurun_out/r20_pytest.log 2>&1; echo pytest rc=$?
python tools/ab.py old:build_var/warpcol/libamppi_b200.so new:paper_2509_17340_b200/libamppi_b200.so 3 > gpurun_out/r20_ab.log 2>&1; echo ab rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/r20_c5.log 2>&1; echo c5 rc=$?

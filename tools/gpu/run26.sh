python -m pytest tests/test_batch_parity.py tests/test_batch_ragged.py tests/test_abi.py -x -q > gpurun_out/r26_pytest.log 2>&1; echo pytest rc=$?
python bench.py --steps 20 --warmup 5 --cpu-seconds 2 > gpurun_out/r26_c5.log 2>&1; echo c5 rc=$?

python -m pytest tests/test_batch_parity.py -q -k precision64 > gpurun_out/r83_pytest.log 2>&1; echo pytest rc=$?

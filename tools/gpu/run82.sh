python -m pytest tests/test_batch_parity.py -q -k two_iterations > gpurun_out/r82_pytest.log 2>&1; echo pytest rc=$?

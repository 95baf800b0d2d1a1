python tools/diag_keying.py > gpurun_out/r15_diag.log 2>&1; echo diag rc=$?
python -m pytest tests/test_snapshot_parity.py tests/test_batch_ragged.py -x -q > gpurun_out/r15_pytest.log 2>&1; echo pytest rc=$?
timeout 300 python bench.py --workload c3 --steps 5 --warmup 2 > gpurun_out/r15_c3.log 2>&1; echo c3 rc=$?

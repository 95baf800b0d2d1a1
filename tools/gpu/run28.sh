set -x
python -m pytest tests/test_snapshot_parity.py tests/test_batch_ragged.py tests/test_batch_parity.py tests/test_plan_parity.py tests/test_config_sizes.py -x -q > gpurun_out/r28_pytest.log 2>&1; echo pytest rc=$?
python tools/ab.py base:build_var/noprefilter/libamppi_b200.so pre:paper_2509_17340_b200/libamppi_b200.so 3 > gpurun_out/r28_ab.log 2>&1; echo ab rc=$?
python bench.py --workload c3 --steps 10 --warmup 3 > gpurun_out/r28_c3.log 2>&1; echo c3 rc=$?

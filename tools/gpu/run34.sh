python -m pytest tests/test_screen_drift.py tests/test_plan_parity.py tests/test_config_sizes.py tests/test_batch_parity.py tests/test_dmax_boundary.py tests/test_snapshot_parity.py tests/test_gpu_loop.py tests/test_closed_loop_replay.py -q > gpurun_out/r34_pytest.log 2>&1; echo pytest rc=$?
python tools/ab.py base:build_var/noprefilter/libamppi_b200.so f64box:build_var/f64box/libamppi_b200.so cur:paper_2509_17340_b200/libamppi_b200.so 3 > gpurun_out/r34_ab.log 2>&1; echo ab rc=$?
timeout 300 python tools/screen_drift.py 4096 1 > gpurun_out/r34_drift.log 2>&1; echo drift rc=$?

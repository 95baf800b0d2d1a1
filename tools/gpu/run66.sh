python -m pytest tests/test_snapshot_parity.py tests/test_batch_ragged.py tests/test_batch_parity.py tests/test_plan_parity.py tests/test_config_sizes.py tests/test_gpu_loop.py -q > gpurun_out/r66_pytest.log 2>&1; echo pytest rc=$?
AMPPI_LIB_PATH=build_stats/libamppi_b200.so python tools/snap_phases_c5.py > gpurun_out/r66_phases.log 2>&1; echo ph rc=$?
python tools/ab.py smem:build_var/sortsmem/libamppi_b200.so regs:paper_2509_17340_b200/libamppi_b200.so 3 > gpurun_out/r66_ab.log 2>&1; echo ab rc=$?

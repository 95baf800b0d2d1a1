AMPPI_LIB_PATH=build_stats/libamppi_b200.so python tools/snap_phases_c5.py > gpurun_out/r39_phases_new.log 2>&1; echo ph rc=$?
AMPPI_LIB_PATH=build_var/stats_scan/libamppi_b200.so python tools/snap_phases_c5.py > gpurun_out/r39_phases_scan.log 2>&1; echo ph rc=$?
python -m pytest tests/test_snapshot_parity.py tests/test_batch_ragged.py tests/test_batch_parity.py tests/test_plan_parity.py -q > gpurun_out/r39_pytest.log 2>&1; echo pytest rc=$?
python tools/ab.py scan:build_var/leafscan/libamppi_b200.so par:paper_2509_17340_b200/libamppi_b200.so 3 > gpurun_out/r39_ab.log 2>&1; echo ab rc=$?

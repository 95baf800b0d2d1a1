set -x
timeout 300 python tools/screen_drift.py 4096 1 > gpurun_out/r32_drift.log 2>&1; echo drift rc=$?
AMPPI_LIB_PATH=build_var/nolog/libamppi_b200.so timeout 300 python tools/screen_drift.py 4096 1 > gpurun_out/r32_drift_nolog.log 2>&1; echo drift rc=$?
AMPPI_LIB_PATH=build_var/world/libamppi_b200.so timeout 300 python -m pytest tests/test_screen_drift.py tests/test_plan_parity.py -q -k "far_from" > gpurun_out/r32_world_far.log 2>&1; echo worldfar rc=$?
python -m pytest tests/test_screen_drift.py tests/test_plan_parity.py tests/test_config_sizes.py tests/test_batch_parity.py tests/test_dmax_boundary.py -q > gpurun_out/r32_pytest.log 2>&1; echo pytest rc=$?
python tools/ab.py world:build_var/world/libamppi_b200.so local:paper_2509_17340_b200/libamppi_b200.so 3 > gpurun_out/r32_ab.log 2>&1; echo ab rc=$?

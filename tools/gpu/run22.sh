AMPPI_LIB_PATH=build_var/hintkey/libamppi_b200.so python -m pytest tests/test_plan_parity.py -x -q > gpurun_out/r22_pytest.log 2>&1; echo pytest rc=$?
python tools/ab.py base:build_var/base/libamppi_b200.so hint:build_var/hintkey/libamppi_b200.so 3 > gpurun_out/r22_ab.log 2>&1; echo ab rc=$?

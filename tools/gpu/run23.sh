AMPPI_LIB_PATH=build_var/groups2/libamppi_b200.so python -m pytest tests/test_plan_parity.py -x -q > gpurun_out/r23_pytest.log 2>&1; echo pytest rc=$?
python tools/ab.py base:build_var/base/libamppi_b200.so g2:build_var/groups2/libamppi_b200.so g3:build_var/groups3/libamppi_b200.so 3 > gpurun_out/r23_ab.log 2>&1; echo ab rc=$?

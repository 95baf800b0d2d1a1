AMPPI_LIB_PATH=build_var/bound8/libamppi_b200.so python -m pytest tests/test_plan_parity.py tests/test_batch_parity.py -x -q > gpurun_out/r11_pytest8.log 2>&1; echo pytest8 rc=$?
python tools/ab.py base:build_var/base/libamppi_b200.so b8:build_var/bound8/libamppi_b200.so b16:build_var/bound16/libamppi_b200.so b4:build_var/bound4/libamppi_b200.so 3 > gpurun_out/r11_ab.log 2>&1; echo ab rc=$?

AMPPI_LIB_PATH=build_var/driftdbg/libamppi_b200.so timeout 300 python tools/screen_drift.py 96 1 > gpurun_out/r30_drift.log 2>&1; echo drift rc=$?

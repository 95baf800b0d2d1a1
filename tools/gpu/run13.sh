python tools/diag_keying.py > gpurun_out/r13_diag.log 2>&1; echo diag rc=$?
AMPPI_LIB_PATH=build_var/nodsmem/libamppi_b200.so python tools/diag_keying.py > gpurun_out/r13_diag_nodsmem.log 2>&1; echo diag2 rc=$?

for r in 1 2; do AMPPI_LIB_PATH=build_stats/libamppi_b200.so python tools/snap_phases_c5.py; done > gpurun_out/r65_phases.log 2>&1; echo ph rc=$?

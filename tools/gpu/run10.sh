python tools/ab.py base:build_var/base/libamppi_b200.so new:paper_2509_17340_b200/libamppi_b200.so split6:build_var/leafsplit6/libamppi_b200.so 3 > gpurun_out/r10_ab.log 2>&1; echo ab rc=$?

python tools/ab.py w64:paper_2509_17340_b200/libamppi_b200.so w48:build_var/w48/libamppi_b200.so w40:build_var/w40/libamppi_b200.so 3 > gpurun_out/r54_ab.log 2>&1; echo ab rc=$?

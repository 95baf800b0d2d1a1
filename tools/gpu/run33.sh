python tools/ab.py base:build_var/noprefilter/libamppi_b200.so nolog:build_var/nolog/libamppi_b200.so cur:paper_2509_17340_b200/libamppi_b200.so 3 > gpurun_out/r33_ab.log 2>&1; echo ab rc=$?

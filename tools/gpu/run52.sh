python tools/ab.py cur:paper_2509_17340_b200/libamppi_b200.so ideal:build_var/idealbound/libamppi_b200.so 2 > gpurun_out/r52_ab.log 2>&1; echo ab rc=$?

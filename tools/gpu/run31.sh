set -x
timeout 300 python tools/screen_drift.py 4096 1 > gpurun_out/r31_drift.log 2>&1; echo drift rc=$?
python -m pytest tests -m gpu -x -q > gpurun_out/r31_pytest.log 2>&1; echo pytest rc=$?
python tools/ab.py base:build_var/noprefilter/libamppi_b200.so local:paper_2509_17340_b200/libamppi_b200.so 3 > gpurun_out/r31_ab.log 2>&1; echo ab rc=$?

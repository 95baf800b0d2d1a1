set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest.log 2>&1; echo pytest rc=$?
make -C paper_2509_17340_b200/csrc stats -j8 > /dev/null 2>&1; echo stats build rc=$?
AMPPI_LIB_PATH=build_stats/libamppi_b200.so timeout 600 python tools/query_stats.py > gpurun_out/r2_query_stats.json 2>&1; echo qs rc=$?

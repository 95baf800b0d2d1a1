set -x
python -m pytest tests/test_shim.py -x -q > gpurun_out/r3_shim.log 2>&1; echo shim rc=$?
AMPPI_LIB_PATH=build_stats/libamppi_b200.so timeout 600 python tools/query_stats.py > gpurun_out/r3_query_stats.json 2>&1; echo qs rc=$?

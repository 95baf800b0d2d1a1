python -m pytest tests -m gpu -x -q > gpurun_out/r60_pytest.log 2>&1; echo pytest rc=$?
python bench.py --steps 10 --warmup 3 --no-latency --cpu-seconds 1 --no-e2e > gpurun_out/r60_c5.log 2>&1; grep -o '"ms_per_step": [0-9.]*' gpurun_out/r60_c5.log | head -1
AMPPI_LIB_PATH=build_stats/libamppi_b200.so python tools/query_stats.py > gpurun_out/r60_qstats.log 2>&1; echo qs rc=$?

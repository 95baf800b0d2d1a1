set -x
python -m pytest tests/test_plan_parity.py tests/test_batch_parity.py tests/test_config_sizes.py tests/test_batch_ragged.py -x -q > gpurun_out/r8_pytest.log 2>&1; echo pytest rc=$?
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-latency --cpu-seconds 1 > gpurun_out/r8_bench.log 2>&1; echo bench rc=$?
AMPPI_LIB_PATH=build_stats/libamppi_b200.so timeout 600 python tools/query_stats.py > gpurun_out/r8_query_stats.json 2>&1; echo qs rc=$?

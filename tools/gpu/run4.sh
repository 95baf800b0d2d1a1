set -x
python -m pytest tests/test_config_sizes.py -x -q -s > gpurun_out/r4_sizes.log 2>&1; echo sizes rc=$?
python bench.py --steps 10 --warmup 3 --no-e2e --latency-cycles 10 --cpu-seconds 1 > gpurun_out/r4_bench.log 2>&1; echo bench rc=$?

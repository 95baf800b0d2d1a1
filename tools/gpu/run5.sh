set -x
python -m pytest tests/test_lidar.py tests/test_sample_sharding.py -x -q > gpurun_out/r5_lidar.log 2>&1; echo lidar rc=$?
python -m pytest tests -m gpu -q > gpurun_out/r5_pytest.log 2>&1; echo pytest rc=$?

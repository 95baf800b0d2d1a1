set -x
python -m pytest tests/test_screen_drift.py -x -q > gpurun_out/r29_pytest.log 2>&1; echo pytest rc=$?
timeout 600 python tools/screen_drift.py 4096 1 > gpurun_out/r29_drift.log 2>&1; echo drift rc=$?

set -x
python -m pytest tests/test_plan_parity.py tests/test_snapshot_parity.py tests/test_batch_parity.py tests/test_dmax_boundary.py -x -q > gpurun_out/r9_pytest.log 2>&1; echo pytest rc=$?
AMPPI_LIB_PATH=build_var/leafsplit6/libamppi_b200.so python -m pytest tests/test_plan_parity.py tests/test_batch_parity.py -x -q > gpurun_out/r9_pytest6.log 2>&1; echo pytest6 rc=$?
for v in default leafsplit6 leafsplit3; do
  if [ $v = default ]; then unset AMPPI_LIB_PATH; else export AMPPI_LIB_PATH=build_var/$v/libamppi_b200.so; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-latency --cpu-seconds 1 > gpurun_out/r9_bench_$v.log 2>&1; echo bench $v rc=$?
done

set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/r1_pytest.log 2>&1; echo pytest rc=$?
python bench.py --steps 5 --warmup 3 > gpurun_out/r1_bench.log 2>&1; echo bench rc=$?
export AMPPI_DEVICE_CHUNKS=1
CMD="python bench.py --steps 1 --warmup 3 --latency-cycles 10 --cpu-seconds 1 --no-e2e"
$CMD > gpurun_out/r1_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_stage1_f32c" -c 1 -o gpurun_out/r1_main $CMD > gpurun_out/r1_ncu.log 2>&1; echo ncu rc=$?

set -x
python -m pytest tests -m gpu -q > gpurun_out/r19_pytest.log 2>&1; echo pytest rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/r19_c5.log 2>&1; echo c5 rc=$?
CMD="python bench.py --steps 1 --warmup 3 --latency-cycles 10 --cpu-seconds 1 --no-e2e --device-chunks 1"
$CMD > gpurun_out/r19_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r19_launches.csv $CMD > gpurun_out/r19_ncu_launch.log 2>&1; echo launches rc=$?
$CMD > gpurun_out/r19_plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_stage1_f32|k_snapshot_scene|k_col_query" -c 5 -o gpurun_out/r19_full $CMD > gpurun_out/r19_ncu_full.log 2>&1; echo full rc=$?
CMD3="python bench.py --workload c3 --steps 1 --warmup 1"
$CMD3 > gpurun_out/r19_plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_key_points|k_finalize" -c 2 -o gpurun_out/r19_c3 $CMD3 > gpurun_out/r19_ncu_c3.log 2>&1; echo c3ncu rc=$?

set -x
python -m pytest tests -m gpu -q > gpurun_out/r76_pytest.log 2>&1; echo pytest rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/r76_c5.log 2>&1; echo c5 rc=$?
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r76_ref_c5.log 2>&1; echo refc5 rc=$?
python bench.py --workload c4 --steps 10 --warmup 3 > gpurun_out/r76_c4.log 2>&1; echo c4 rc=$?
python bench.py --workload c3 --steps 10 --warmup 3 > gpurun_out/r76_c3.log 2>&1; echo c3 rc=$?
python bench.py --workload c2 --steps 3 --warmup 1 > gpurun_out/r76_c2.log 2>&1; echo c2 rc=$?
python bench.py --impl reference --workload c4 --steps 2 --warmup 1 > gpurun_out/r76_ref_c4.log 2>&1; echo refc4 rc=$?
python bench.py --impl reference --workload c3 --steps 3 --warmup 1 > gpurun_out/r76_ref_c3.log 2>&1; echo refc3 rc=$?
python bench.py --gpus 2 --steps 5 --warmup 2 --no-latency --cpu-seconds 2 > gpurun_out/r76_c5_g2.log 2>&1; echo c5g2 rc=$?
python bench.py --gpus 2 --workload c4 --steps 3 --warmup 1 > gpurun_out/r76_c4_g2.log 2>&1; echo c4g2 rc=$?
CMD="python bench.py --steps 1 --warmup 3 --latency-cycles 10 --cpu-seconds 1 --no-e2e --device-chunks 1"
$CMD > gpurun_out/r76_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r76_launches.csv $CMD > gpurun_out/r76_ncu_launch.log 2>&1; echo launches rc=$?
$CMD > gpurun_out/r76_plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_stage1_f32|k_snapshot_scene|k_col_query|k_col_classify" -c 6 -o gpurun_out/r76_full $CMD > gpurun_out/r76_ncu_full.log 2>&1; echo full rc=$?
python tools/c1_once.py 20 > gpurun_out/r76_c1plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r76_c1_launches.csv python tools/c1_once.py 20 > gpurun_out/r76_c1ncu.log 2>&1; echo c1 rc=$?

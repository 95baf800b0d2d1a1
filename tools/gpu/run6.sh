set -x
python -m pytest tests/test_lidar.py -x -q > gpurun_out/r6_lidar.log 2>&1; echo lidar rc=$?
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r6_c5.log 2>&1; echo c5 rc=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r6_ref_c5.log 2>&1; echo refc5 rc=$?
timeout 300 python bench.py --workload c4 --steps 5 --warmup 2 > gpurun_out/r6_c4.log 2>&1; echo c4 rc=$?
timeout 300 python bench.py --workload c3 --steps 5 --warmup 2 > gpurun_out/r6_c3.log 2>&1; echo c3 rc=$?
timeout 300 python bench.py --workload c2 --steps 2 --warmup 1 > gpurun_out/r6_c2.log 2>&1; echo c2 rc=$?
timeout 300 python bench.py --impl reference --workload c4 --steps 2 --warmup 1 > gpurun_out/r6_ref_c4.log 2>&1; echo refc4 rc=$?
timeout 300 python bench.py --impl reference --workload c3 --steps 2 --warmup 1 > gpurun_out/r6_ref_c3.log 2>&1; echo refc3 rc=$?
timeout 600 python bench.py --gpus 2 --steps 5 --warmup 2 --no-latency --cpu-seconds 2 > gpurun_out/r6_c5_g2.log 2>&1; echo c5g2 rc=$?
timeout 300 python bench.py --gpus 2 --workload c4 --steps 3 --warmup 1 > gpurun_out/r6_c4_g2.log 2>&1; echo c4g2 rc=$?

python bench.py --gpus 2 --steps 5 --warmup 2 --no-latency --cpu-seconds 2 > gpurun_out/r64_c5_g2.log 2>&1; echo c5g2 rc=$?
tail -c 600 gpurun_out/r64_c5_g2.log

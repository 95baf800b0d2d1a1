python -m pytest tests -m gpu -x -q > gpurun_out/r55_pytest.log 2>&1; echo pytest rc=$?
for r in 1 2; do python bench.py --workload c4 --steps 10 --warmup 3 --cpu-seconds 1 > gpurun_out/r55_c4_$r.log 2>&1; grep -o '"ms_per_step": [0-9.]*' gpurun_out/r55_c4_$r.log | head -1; done
python bench.py --steps 5 --warmup 3 --cpu-seconds 1 --no-e2e > gpurun_out/r55_c5.log 2>&1; grep -o '"p50_ms": [0-9.]*' gpurun_out/r55_c5.log | head -2

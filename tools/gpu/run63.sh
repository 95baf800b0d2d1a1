python -m pytest tests/test_batch_parity.py -q -x -k streaming > gpurun_out/r63_pytest.log 2>&1; echo pytest rc=$?
for r in 1 2; do python bench.py --steps 10 --warmup 3 --no-latency --cpu-seconds 1 > gpurun_out/r63_c5_$r.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r63_c5_$r.log').read().strip().splitlines()[-1]); print('value ms', round(d['ms_per_step'],3), 'e2e ms', round(d['e2e']['ms_per_step'],3))"; done

for r in 1 2 3; do for v in cur envnopre; do
  if [ $v = cur ]; then L=paper_2509_17340_b200/libamppi_b200.so; else L=build_var/$v/libamppi_b200.so; fi
  AMPPI_LIB_PATH=$L python bench.py --steps 2 --warmup 3 --cpu-seconds 1 --no-e2e --latency-cycles 2000 > gpurun_out/r57_${v}_$r.log 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/r57_${v}_$r.log').read().strip().splitlines()[-1]); l=d['latency']; print('$v', $r, round(l['p50_ms'],4), round(l['p99_ms'],4), round(l['paper_default']['p50_ms'],4))"
done; done
python tools/c1_once.py 20 > /dev/null 2>&1; AMPPI_LIB_PATH=build_var/envnopre/libamppi_b200.so ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r57_c1_envnopre.csv python tools/c1_once.py 20 > /dev/null 2>&1; echo ncu rc=$?

set -x
for v in "$@"; do
  AMPPI_LIB_PATH=build_var/$v/libamppi_b200.so timeout 300 python bench.py --steps 5 --warmup 3 --latency-cycles 200 --cpu-seconds 0.5 --no-e2e > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  python - "$v" <<'PY'
import json,sys
d=json.load(open(f"gpurun_out/var_{sys.argv[1]}.json"))
print(sys.argv[1], round(d["ms_per_step"],3), d["latency"]["p50_ms"], {k:round(v["ms_total"]/v["launches"],3) for k,v in d["kernels"].items()})
PY
done

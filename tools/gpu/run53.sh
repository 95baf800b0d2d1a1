for f in 0 45056 49152 53248; do timeout 900 python tools/c5_full_parity.py 4096 $f 2>&1 | tail -2; done > gpurun_out/r53_parity.log 2>&1; echo parity rc=$?

for f in 0 57344; do timeout 900 python tools/c5_full_parity.py 4096 $f 2>&1 | tail -1; done > gpurun_out/r79_parity.log 2>&1; echo parity rc=$?

for f in 61440 65536 69632 73728; do timeout 900 python tools/c5_full_parity.py 4096 $f 2>&1 | tail -1; done > gpurun_out/r85_parity.log 2>&1; echo parity rc=$?

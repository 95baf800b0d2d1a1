for r in 1 2; do python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/r77_pytest_$r.log 2>&1; echo pytest$r rc=$?; done

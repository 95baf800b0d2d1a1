python -m pytest tests -m gpu -q > gpurun_out/r84_pytest.log 2>&1; echo pytest rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r84_smoke.log 2>&1; echo smoke rc=$?

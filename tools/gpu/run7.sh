set -x
python -m pytest tests -m gpu -q > gpurun_out/r7_pytest.log 2>&1; echo pytest rc=$?
python tools/sanitize_case.py > gpurun_out/r7_plain.log 2>&1 && timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_case.py > gpurun_out/r7_racecheck.log 2>&1; echo racecheck rc=$?

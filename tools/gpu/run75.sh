( time python bench.py ) > gpurun_out/r75_default.log 2>&1; echo default rc=$?
( time python bench.py --impl reference ) > gpurun_out/r75_ref.log 2>&1; echo ref rc=$?

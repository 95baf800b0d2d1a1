python tools/pipe_trace.py 6:1.2 1:1.0 4:1.2 8:1.1 12:1.0 > gpurun_out/r21_trace.log 2>&1; echo trace rc=$?

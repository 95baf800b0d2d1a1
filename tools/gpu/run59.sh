python tools/c1_profile.py > gpurun_out/r59_c1_profile.log 2>&1; echo prof rc=$?

python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r62_smoke.log 2>&1; echo smoke rc=$?

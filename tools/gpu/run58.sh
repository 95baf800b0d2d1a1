python tools/c1_once.py 5 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_anchors|k_finalize_scene|k_refine_fused_w|k_stage1_warp32|k_stage2_fused_w" -c 5 -o gpurun_out/r58_c1 python tools/c1_once.py 3 > gpurun_out/r58_ncu.log 2>&1; echo ncu rc=$?

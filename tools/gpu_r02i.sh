timeout 300 python tools/matvec_probe.py > gpurun_out/mv_probe.log 2>&1
REDVE_MATVEC=generic timeout 300 python tools/matvec_probe.py >> gpurun_out/mv_probe.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_cg_matvec_ct|k_normal_matvec_p" -s 2 -c 1 -o gpurun_out/prof_mv -f python tools/matvec_probe.py 8332 8192 3 > gpurun_out/ncu_mv.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_mv.log

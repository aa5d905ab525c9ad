timeout 300 python tools/step_probe.py 64 256 fp 2 > gpurun_out/sp.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_col|k_row_inv" -s 10 -c 4 -o gpurun_out/prof_pers -f python tools/step_probe.py 64 256 fp 2 > gpurun_out/ncu_pers.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_pers.log

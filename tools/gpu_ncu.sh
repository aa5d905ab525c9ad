# full ncu capture of the hot kernels (plain run first, same command line)
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_short.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_row_fwd|k_col|k_row_inv|k_cost|k_gram|k_combine" -s 40 -c 6 -o gpurun_out/prof -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_full.log

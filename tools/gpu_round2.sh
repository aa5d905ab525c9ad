# round 2 measurement pass on one box: bench FIRST (fresh-box behaviour), then
# tests, smoke, reference arm, every config, launch list, ncu captures
O=${O:-gpurun_out/r02f}; mkdir -p $O

nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,clocks.max.mem --format=csv > $O/smi.txt 2>&1
timeout 600 python bench.py > $O/bench_first.log 2>&1; echo "rc=$?" >> $O/bench_first.log
timeout 900 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
timeout 900 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo "rc=$?" >> $O/bench_ref.log
for c in 0 2 3 4; do timeout 900 python bench.py --config $c > $O/bench_c$c.log 2>&1; echo "rc=$?" >> $O/bench_c$c.log; done
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/bench_short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_row_fwd|k_col|k_row_inv|k_cost_fp|k_gram|k_combine" -s 60 -c 6 -o $O/prof_c1 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_c1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cg_matvec_ct|k_pw_sweep" -s 2 -c 3 -o $O/prof_sr -f python tools/matvec_probe.py 8332 8192 3 > $O/ncu_sr.log 2>&1
echo done

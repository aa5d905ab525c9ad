# final pass of a round: bench first (fresh-box behaviour), tests, smoke, reference arm, every config
O=${O:-gpurun_out/final}; mkdir -p $O
timeout 600 python bench.py > $O/bench_first.log 2>&1; echo "rc=$?" >> $O/bench_first.log
timeout 1500 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
timeout 900 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo "rc=$?" >> $O/bench_ref.log
for c in 0 2 3 4; do timeout 900 python bench.py --config $c > $O/bench_c$c.log 2>&1; echo "rc=$?" >> $O/bench_c$c.log; done
timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_gpus2.log 2>&1; echo "rc=$?" >> $O/bench_gpus2.log
tail -2 $O/gpu_tests.log; tail -1 $O/smoke.log
for f in bench_first bench bench_c0 bench_c2 bench_c3 bench_c4 bench_gpus2; do echo $f; python tools/show_bench.py $O/$f.log 2>&1 | head -1; done

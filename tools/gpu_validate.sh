# validation pass: GPU tests, smoke, headline bench, reference arm (O = output dir)
O=${O:-gpurun_out/val}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
tail -3 $O/gpu_tests.log; tail -1 $O/smoke.log; tail -2 $O/bench.log

# quick A/B pass: Fourier-route parity tests, then the headline bench twice (O = output dir)
O=${O:-gpurun_out/ab}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config_scale.py tests/test_gpu_persistent.py -m gpu -q -x --tb=short -p no:cacheprovider > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
tail -3 $O/tests.log
for i in 1 2; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$i.log 2>&1; echo "rc=$?" >> $O/bench_$i.log
  python tools/show_bench.py $O/bench_$i.log
done

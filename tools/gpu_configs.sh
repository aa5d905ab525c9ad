# every BASELINE.json config on one GPU, contract W >= 3 (CPU baselines included)
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c1.log
timeout 600 python bench.py --config 0 --steps 5 --warmup 3 > gpurun_out/bench_c0.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c0.log
timeout 900 python bench.py --config 2 --steps 3 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c2.log
timeout 900 python bench.py --config 3 --steps 2 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c3.log
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 > gpurun_out/bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4.log
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_c1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref_c1.log

timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --config 0 --steps 5 --warmup 3 > gpurun_out/bench_c0.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c0.log
timeout 900 python bench.py --config 2 --steps 2 --warmup 1 > gpurun_out/bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c2.log
timeout 900 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c3.log

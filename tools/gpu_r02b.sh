set -x
timeout 300 python tools/repeat_probe.py 8 > gpurun_out/repeat.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench2.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench3.log 2>&1

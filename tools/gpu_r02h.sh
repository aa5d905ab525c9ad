timeout 600 python -m pytest tests/test_gpu_matvec.py tests/test_gpu_spatial.py tests/test_gpu_config_scale.py -q --tb=short -p no:cacheprovider -x -k "matvec or config2 or spatial" > gpurun_out/gpu_mv.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_mv.log
timeout 600 python bench.py --config 4 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1

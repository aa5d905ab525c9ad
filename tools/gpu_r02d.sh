timeout 600 python -m pytest tests/test_gpu_persistent.py -q --tb=short -p no:cacheprovider -x > gpurun_out/gpu_pers.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_pers.log
for P in 0 1; do REDVE_PERSISTENT=$P timeout 300 python tools/step_probe.py 64 256 fp-ve 10 > gpurun_out/probe_p$P.log 2>&1; done
REDVE_PERSISTENT=1 PROBE_DEN=fb timeout 300 python tools/step_probe.py 128 512 fp-ve 3 > gpurun_out/probe512_p1.log 2>&1

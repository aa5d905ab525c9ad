timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config_scale.py -q --tb=short -p no:cacheprovider -x -k "FpStep or config1 or Solves" > gpurun_out/gpu_ri8.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_ri8.log
for P in 0 1; do REDVE_ROWINV8=$P timeout 300 python tools/step_probe.py 64 256 fp 5 > gpurun_out/probe_ri$P.log 2>&1; done
for P in 0 1; do REDVE_ROWINV8=$P PROBE_DEN=fb timeout 300 python tools/step_probe.py 128 512 fp 2 > gpurun_out/probe512_ri$P.log 2>&1; done

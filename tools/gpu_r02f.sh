for P in c 0; do REDVE_PERSISTENT=$P timeout 300 python tools/step_probe.py 64 256 fp 5 > gpurun_out/probe_p$P.log 2>&1; done
for P in c 0; do REDVE_PERSISTENT=$P PROBE_DEN=fb timeout 300 python tools/step_probe.py 128 512 fp 2 > gpurun_out/probe512_p$P.log 2>&1; done

for c in 0 2 3 4; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; echo "c$c rc=$?"; done

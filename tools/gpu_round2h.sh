# last pass of round 2 (after the PatchWeighted vector-sweep change): gpu_final.sh, then launch lists and
# ncu --set full captures of the PatchWeighted kernels on configs[2] / configs[4] (each after its plain run exited 0)
O=${O:-gpurun_out/r02h}; mkdir -p $O
O=$O bash tools/gpu_final.sh
for c in 2 4; do
  timeout 600 python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > $O/plain_c$c.log 2>&1 || { echo "plain c$c failed"; continue; }
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/launches_c$c.csv \
    python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_list_c$c.log 2>&1; echo "launch list c$c rc=$?"
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_pw_sweep_v|k_pw_weights_t" -s 24 -c 4 -o $O/prof_pw_c$c -f \
    python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_pw_c$c.log 2>&1; echo "ncu pw c$c rc=$?"
done
ls -la $O

# ncu --set full of the dominant kernels of the other configs and the cadence
# cost (each command first runs plain and must exit 0)
O=${O:-gpurun_out/r02f_other}; mkdir -p $O
run() {  # name, kernel regex, skip, count, bench args...
  local name=$1 rx=$2 skip=$3 cnt=$4; shift 4
  timeout 600 python bench.py "$@" --steps 1 --warmup 3 --no-cpu-baseline > $O/plain_$name.log 2>&1 || { echo "plain $name failed"; return; }
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $skip -c $cnt -o $O/prof_$name -f \
    python bench.py "$@" --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_$name.log 2>&1; echo "ncu $name rc=$?"
}
run c1cost "k_cost_fp|k_copy_view" 20 4 --config 1
run c2 "k_pw_sweep_t|k_pw_weights_t|k_cg_update" 30 5 --config 2
run c3 "k_rd_bank8w" 4 2 --config 3 --batch 64
run c0 "k_spec_run" 2 1 --config 0
ls -la $O

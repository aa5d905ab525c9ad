# solves/s of the headline workload as a function of the batch per launch (L2 residency)
O=${O:-gpurun_out/bsweep}
mkdir -p $O
for b in 8 16 24 32 48 64; do
  timeout 600 python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline > $O/b_$b.log 2>&1
  python tools/show_bench.py $O/b_$b.log | head -12
done

# run-to-run spread of the headline bench with and without the clock sampler
O=${O:-gpurun_out/rep}
mkdir -p $O
for i in 1 2 3 4 5 6; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/with_$i.log 2>&1
  REDVE_BENCH_NO_SMI=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/without_$i.log 2>&1
done
python - <<'PY'
import json, glob, os
O = os.environ.get("O", "gpurun_out/rep")
for f in sorted(glob.glob(O + "/*.log")):
    d = [json.loads(l) for l in open(f) if l.startswith("{")]
    if d:
        d = d[-1]
        print(os.path.basename(f), {k: round(v["ms_per_step"], 2) for k, v in d["methods"].items()}, "e2e", round(d["e2e"]["ms_per_step"], 2))
PY

import json, sys
lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")]
d = json.loads(lines[-1])
print("value", round(d["value"], 1), "ms/step", round(d["ms_per_step"], 2), "e2e", round(d["e2e"]["value"], 1),
      "dom", d["roofline"]["kernel"], "frac", d["roofline"]["frac"] and round(d["roofline"]["frac"], 3), "launches", d["gpu_launches"])
for k, v in d["kernels"].items():
    print(f"  {k:12s} n={v['launches']:4d} avg={v['avg_us']:8.1f}us gbs={v['gbs'] and round(v['gbs'])}")
print("clocks", d.get("clocks"))

# PatchWeighted call time, scalar vs vector sweep, over image sizes and plane widths (picks the switch-over)
O=${O:-gpurun_out/pwsizes}; mkdir -p $O
for wdt in float32 float64; do for n in 128 192 256 384 512 768 1024 2048; do for v in 0 1; do
  REDVE_PW_VEC=$v python tools/pw_probe.py $n 20 $wdt 2>/dev/null | grep patch_weighted | sed "s/^/vec=$v /"
done; done; done | tee $O/sizes.log

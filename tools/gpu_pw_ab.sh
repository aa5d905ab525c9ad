# A/B of the PatchWeighted vector sweep: parity tests, configs[4] and configs[2] (vector sweep forced), then the
# same at another launch bound (MINB = CTAs/SM of k_pw_sweep_v), rebuilt on the box (O = output dir)
O=${O:-gpurun_out/pwab}; mkdir -p $O
run() {
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spatial.py tests/test_gpu_config_scale.py -m gpu -q -x --tb=short -p no:cacheprovider -k "Patch or patch or spatial or config2" > $O/tests_$1.log 2>&1; tail -1 $O/tests_$1.log
  timeout 600 python bench.py --config 4 --no-cpu-baseline > $O/c4_$1.log 2>&1; python tools/show_bench.py $O/c4_$1.log | grep "value\|patch_w"
  REDVE_PW_VEC=1 timeout 600 python bench.py --config 2 --no-cpu-baseline > $O/c2vec_$1.log 2>&1; python tools/show_bench.py $O/c2vec_$1.log | grep "value\|patch_w"
}
run a
for mb in ${MINB:-5}; do
  sed -i "s/__launch_bounds__(256, 4)  \/\/ CTAs\/SM of the vector sweep/__launch_bounds__(256, $mb)  \/\/ CTAs\/SM of the vector sweep/" paper_1805_02158_b200/csrc/sr.cu
  (cd paper_1805_02158_b200/csrc && make -j8 > /dev/null 2>&1; grep -A2 "k_pw_sweep_vILi3EfEE" build/sr.ptxas.log | tail -2)
  run mb$mb
  sed -i "s/__launch_bounds__(256, $mb)  \/\/ CTAs\/SM of the vector sweep/__launch_bounds__(256, 4)  \/\/ CTAs\/SM of the vector sweep/" paper_1805_02158_b200/csrc/sr.cu
done

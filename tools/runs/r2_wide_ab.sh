# wide formats (warp per value): fused multiply-accumulate in the column products -- parity, then Lotkin timing A/B
timeout 1200 python -m pytest tests/test_gpu_wide.py tests/test_gpu_wide_warp.py -x -q -p no:cacheprovider > gpurun_out/r2_wide_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_wide_tests.log
tail -3 gpurun_out/r2_wide_tests.log
for rep in 1 2; do
for v in default wmul0; do
  if [ $v = default ]; then L=""; else L="MPGPU_LIB=paper_1410_1599_b200/_variants/$v/libmpgpu.so"; fi
  echo "== $v"; env $L timeout 600 python tools/lotkin_wide.py --n 128 --bits 8192 --alpha 1..1 2>&1 | tail -3
  env $L timeout 600 python tools/wide_lat.py 2>&1 | tail -6
done; done > gpurun_out/r2_wide_ab.log 2>&1
cat gpurun_out/r2_wide_ab.log

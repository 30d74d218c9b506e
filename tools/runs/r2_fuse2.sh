# fused two-level pre- and post-additions: parity, then timing A/B (MPGPU_PREADD_FUSE=0: two launches per level pair)
timeout 1500 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_fullsize_hash.py tests/test_gpu_fullsize.py tests/test_gpu_dropin.py tests/test_gpu_auto.py tests/test_gpu_host_pipe.py tests/test_gpu_lu.py -x -q -p no:cacheprovider > gpurun_out/r2_fuse2_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_fuse2_tests.log
tail -3 gpurun_out/r2_fuse2_tests.log
for rep in 1 2; do
for f in 0 32; do
  MPGPU_PREADD_FUSE=$f timeout 300 python tools/ab_leaf.py --bits 128 256 512 1024 --reps 4 --tag fuse$f
done
for v in pt16 pt64; do
  MPGPU_LIB=paper_1410_1599_b200/_variants/$v/libmpgpu.so timeout 300 python tools/ab_leaf.py --bits 256 512 1024 --reps 4 --tag $v
done; done > gpurun_out/r2_ab_fuse2.jsonl 2>&1
grep '^{' gpurun_out/r2_ab_fuse2.jsonl

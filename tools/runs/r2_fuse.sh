# fused two-level pre-additions: parity (all limb counts: MPGPU_PREADD_FUSE=32), then timing A/B
MPGPU_PREADD_FUSE=32 timeout 1200 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_fullsize_hash.py tests/test_gpu_fullsize.py tests/test_gpu_dropin.py -x -q -p no:cacheprovider > gpurun_out/r2_fuse_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_fuse_tests.log
tail -3 gpurun_out/r2_fuse_tests.log
for f in 0 8 32; do
  MPGPU_PREADD_FUSE=$f timeout 300 python tools/ab_leaf.py --bits 128 256 512 1024 --reps 4 --tag fuse$f
done > gpurun_out/r2_ab_fuse.jsonl 2>&1
grep '^{' gpurun_out/r2_ab_fuse.jsonl

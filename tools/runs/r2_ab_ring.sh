V=paper_1410_1599_b200/_variants
for t in ring noring r4tk8 ring; do L=$V/$t/libmpgpu.so; [ $t = ring ] && L=paper_1410_1599_b200/libmpgpu.so; MPGPU_LIB=$L python tools/ab_leaf.py --bits 256 --reps 5 --tag $t; done > gpurun_out/r2_ab_ring.jsonl 2>&1
python -m pytest tests/test_gpu_fullsize_hash.py tests/test_gpu_gemm.py tests/test_gpu_lu.py tests/test_gpu_auto.py -x -q -p no:cacheprovider > gpurun_out/r2_ring_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_ring_tests.log
MPGPU_LIB=$V/r4tk8/libmpgpu.so python -m pytest tests/test_gpu_fullsize_hash.py -x -q -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/r2_ring_tests.log
cat gpurun_out/r2_ab_ring.jsonl; tail -3 gpurun_out/r2_ring_tests.log

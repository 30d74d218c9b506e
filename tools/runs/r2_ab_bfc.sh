V=paper_1410_1599_b200/_variants
for t in base bfc base bfc; do L=$V/$t/libmpgpu.so; [ $t = base ] && L=paper_1410_1599_b200/libmpgpu.so; MPGPU_LIB=$L python tools/ab_leaf.py --bits 256 512 1024 --reps 5 --tag $t; done > gpurun_out/r2_ab_bfc.jsonl 2>&1
MPGPU_LIB=$V/bfc/libmpgpu.so python -m pytest tests/test_gpu_fullsize_hash.py tests/test_gpu_gemm.py -x -q -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/r2_ab_bfc.jsonl
cat gpurun_out/r2_ab_bfc.jsonl

V=paper_1410_1599_b200/_variants
for t in hoist nohoist hoist nohoist; do L=$V/$t/libmpgpu.so; [ $t = hoist ] && L=paper_1410_1599_b200/libmpgpu.so; MPGPU_LIB=$L python tools/ab_leaf.py --bits 128 256 --reps 7 --tag $t; MPGPU_LIB=$L python tools/ab_leaf.py --bits 256 --n 2048 --n-min 64 --reps 3 --tag $t; done > gpurun_out/r2_ab_hoist.jsonl 2>&1
python -m pytest tests/test_gpu_fullsize_hash.py tests/test_gpu_gemm.py tests/test_gpu_lu.py -x -q -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/r2_ab_hoist.jsonl
cat gpurun_out/r2_ab_hoist.jsonl

V=paper_1410_1599_b200/_variants
for t in base minb3 pipe_m3 pipe_m4 pipe_m3ku1; do L=$V/$t/libmpgpu.so; [ $t = base ] && L=paper_1410_1599_b200/libmpgpu.so; MPGPU_LIB=$L python tools/ab_leaf.py --bits 256 512 --reps 5 --tag $t; done > gpurun_out/r2_ab_pipe.jsonl 2>&1
for t in pipe_m3 pipe_m4; do MPGPU_LIB=$V/$t/libmpgpu.so python -m pytest tests/test_gpu_fullsize_hash.py tests/test_gpu_gemm.py -x -q -p no:cacheprovider 2>&1 | tail -2; done > gpurun_out/r2_ab_pipe_tests.log 2>&1
cat gpurun_out/r2_ab_pipe.jsonl; cat gpurun_out/r2_ab_pipe_tests.log

python -m pytest tests/test_gpu_gemm.py -x -q -p no:cacheprovider -k "zeros" > gpurun_out/r2_zero_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_zero_tests.log
for K in 32 64; do for k in winograd block simple; do echo "K=$K $k"; python tools/prof_lu.py --n 2048 --K $K --kernel $k --reps 2 | tail -1; done; done > gpurun_out/r2_lu_k.log 2>&1
for K in 32 64; do echo "K=$K winograd nola"; MPGPU_LU_LOOKAHEAD=0 python tools/prof_lu.py --n 2048 --K $K --kernel winograd --reps 2 | tail -1; done >> gpurun_out/r2_lu_k.log 2>&1
tail -2 gpurun_out/r2_zero_tests.log; cat gpurun_out/r2_lu_k.log

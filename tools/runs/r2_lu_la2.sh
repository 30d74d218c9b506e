for K in 64 128 256; do for la in 0 1; do echo "K=$K la=$la"; MPGPU_LU_LOOKAHEAD=$la MPGPU_LU_LA_GRID=32 python tools/prof_lu.py --n 2048 --K $K --kernel winograd --reps 2; done; done > gpurun_out/r2_lu_la2.log 2>&1
for g in 24 32 40; do echo "K=128 grid=$g"; MPGPU_LU_LA_GRID=$g python tools/prof_lu.py --n 2048 --K 128 --kernel winograd --reps 2; done >> gpurun_out/r2_lu_la2.log 2>&1
cat gpurun_out/r2_lu_la2.log

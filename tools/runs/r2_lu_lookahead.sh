set -x
python -m pytest tests/test_gpu_lu.py tests/test_gpu_fullsize_hash.py tests/test_gpu_dropin.py tests/test_gpu_gemm.py -x -q -p no:cacheprovider > gpurun_out/r2_lu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_lu_tests.log
for la in 0 1; do MPGPU_LU_LOOKAHEAD=$la python tools/prof_lu.py --n 2048 --K 64 --kernel winograd --reps 3; done > gpurun_out/r2_lu_la.log 2>&1
for g in 16 32 64 96 148; do echo grid=$g; MPGPU_LU_LA_GRID=$g python tools/prof_lu.py --n 2048 --K 64 --kernel winograd --reps 3; done >> gpurun_out/r2_lu_la.log 2>&1
for k in block; do MPGPU_LU_LOOKAHEAD=0 python tools/prof_lu.py --n 2048 --K 64 --kernel $k --reps 2; python tools/prof_lu.py --n 2048 --K 64 --kernel $k --reps 2; done >> gpurun_out/r2_lu_la.log 2>&1
tail -3 gpurun_out/r2_lu_tests.log; cat gpurun_out/r2_lu_la.log

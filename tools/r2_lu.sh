mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lu.py tests/test_gpu_lu_host.py tests/test_gpu_fullsize_hash.py tests/test_gpu_benchdrv.py -x -q > gpurun_out/lu_tests.log 2>&1; echo rc=$? >> gpurun_out/lu_tests.log
python tools/prof_lu.py --n 2048 --K 64 --kernel winograd --reps 3 > gpurun_out/lu_pref.log 2>&1
MPGPU_LU_TRACE=1 python tools/prof_lu.py --n 2048 --K 64 --kernel winograd --reps 2 > gpurun_out/lu_trace3.log 2>&1
cat gpurun_out/lu_pref.log; tail -2 gpurun_out/lu_tests.log

timeout 600 python -m pytest tests/test_gpu_primitives.py -x -q -p no:cacheprovider > gpurun_out/r2_prim_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_prim_tests.log
tail -3 gpurun_out/r2_prim_tests.log
for g in 16 24 32 48; do
  echo "LA_GRID=$g" ; MPGPU_LU_LA_GRID=$g timeout 300 python tools/prof_lu.py --n 2048 --K 64 --n-min 32 --kernel winograd --reps 3 | tail -1
done > gpurun_out/r2_lu_la3.log 2>&1
for s in 256 512 768 1024; do
  echo "LA_SWITCH=$s" ; MPGPU_LU_LA_SWITCH=$s timeout 300 python tools/prof_lu.py --n 2048 --K 64 --n-min 32 --kernel winograd --reps 3 | tail -1
done >> gpurun_out/r2_lu_la3.log 2>&1
cat gpurun_out/r2_lu_la3.log

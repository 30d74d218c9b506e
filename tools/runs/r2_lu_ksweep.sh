# cfg5 LU (n=2048 @256, pivoting, Winograd Schur): block size K and cutoff sweep
for cfg in "64 32" "96 32" "128 32" "128 64" "192 32" "256 32" "256 64"; do set -- $cfg
  timeout 300 python tools/prof_lu.py --n 2048 --K $1 --n-min $2 --kernel winograd --reps 3 | tail -1
done > gpurun_out/r2_lu_ksweep.log 2>&1
cat gpurun_out/r2_lu_ksweep.log

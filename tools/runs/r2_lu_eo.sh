# cfg5 LU with the carry-chained product: block size / cutoff sweep and the per-step trace
for cfg in "32 32" "48 32" "64 32" "64 16" "96 32" "128 32" "128 64"; do set -- $cfg
  timeout 300 python tools/prof_lu.py --n 2048 --K $1 --n-min $2 --kernel winograd --reps 3 | tail -1
done > gpurun_out/r2_lu_ksweep_eo.log 2>&1
cat gpurun_out/r2_lu_ksweep_eo.log
MPGPU_LU_TRACE=1 timeout 300 python tools/prof_lu.py --n 2048 --K 64 --n-min 32 --kernel winograd --reps 2 > gpurun_out/r2_lu_trace_eo.log 2>&1
tail -40 gpurun_out/r2_lu_trace_eo.log

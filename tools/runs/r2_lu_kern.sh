# cfg5 LU: Schur kernel choice (classical vs one Winograd level) per block size
for cfg in "block 64 64" "simple 64 0" "block 48 48" "block 32 32" "block 96 96" "block 128 128" "winograd 64 32" "winograd 128 32" "strassen 64 32"; do set -- $cfg
  timeout 300 python tools/prof_lu.py --n 2048 --K $2 --n-min $3 --kernel $1 --reps 3 | tail -1
done > gpurun_out/r2_lu_kern.log 2>&1
cat gpurun_out/r2_lu_kern.log
MPGPU_LU_TRACE=1 timeout 300 python tools/prof_lu.py --n 2048 --K 64 --n-min 64 --kernel block --reps 2 > gpurun_out/r2_lu_trace_block.log 2>&1

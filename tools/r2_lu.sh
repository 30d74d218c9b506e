mkdir -p gpurun_out
for sw in 0 640 896 1152 1408; do echo "switch $sw"; MPGPU_LU_LA_SWITCH=$sw python tools/prof_lu.py --n 2048 --K 64 --kernel winograd --reps 3 2>&1 | tail -2; done > gpurun_out/lu_switch.log 2>&1
cat gpurun_out/lu_switch.log

# ncu --set full of the pre-/post-addition kernels of one cfg2 product (8 pre-add + 4 post-add launches)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"preadd_kernel|postadd_kernel" -c 12 -o gpurun_out/adds_cfg2 python tools/prof_gemm.py --bits 256 --reps 1 > gpurun_out/ncu_adds_cfg2.log 2>&1
tail -2 gpurun_out/ncu_adds_cfg2.log

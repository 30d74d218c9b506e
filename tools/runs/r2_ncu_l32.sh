timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_leaf_kernel -s 1 -c 1 -o gpurun_out/leaf32_eo python tools/prof_gemm.py --bits 1024 --reps 2 > gpurun_out/ncu_leaf32_eo.log 2>&1
tail -2 gpurun_out/ncu_leaf32_eo.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_leaf_kernel -s 1 -c 1 -o gpurun_out/leaf16_eo python tools/prof_gemm.py --bits 512 --reps 2 > gpurun_out/ncu_leaf16_eo.log 2>&1

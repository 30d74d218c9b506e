timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_leaf_kernel -s 1 -c 1 -o gpurun_out/leaf8_final python tools/prof_gemm.py --bits 256 --reps 2 > gpurun_out/ncu_leaf8_final.log 2>&1
tail -2 gpurun_out/ncu_leaf8_final.log

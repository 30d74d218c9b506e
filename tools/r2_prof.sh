set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_r2t.log 2>&1; echo rc=$? >> gpurun_out/gputests_r2t.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_leaf_kernel -s 2 -c 1 -o gpurun_out/leaf8_addw python tools/prof_gemm.py --bits 256 --reps 2 > gpurun_out/ncu_leaf8_addw.log 2>&1
tail -2 gpurun_out/gputests_r2t.log

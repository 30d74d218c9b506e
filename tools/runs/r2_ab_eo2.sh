# even/odd product with the provably-zero chain carries skipped: parity, A/B, ncu of the L=8 leaf
timeout 900 python -m pytest tests/test_gpu_primitives.py tests/test_gpu_gemm.py tests/test_gpu_fullsize_hash.py -x -q -p no:cacheprovider > gpurun_out/r2_eo2_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_eo2_tests.log
tail -3 gpurun_out/r2_eo2_tests.log
AB_ARGS="--bits 256 512 1024 --reps 4" bash tools/ab_run.sh gpurun_out/r2_ab_eo2.jsonl default noskipc m7
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_leaf_kernel -s 2 -c 1 -o gpurun_out/leaf8_eo python tools/prof_gemm.py --bits 256 --reps 2 > gpurun_out/ncu_leaf8_eo.log 2>&1

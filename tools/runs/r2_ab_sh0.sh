timeout 900 python -m pytest tests/test_gpu_primitives.py tests/test_gpu_gemm.py tests/test_gpu_fullsize_hash.py tests/test_gpu_lu.py -x -q -p no:cacheprovider > gpurun_out/r2_sh0_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_sh0_tests.log
tail -3 gpurun_out/r2_sh0_tests.log
AB_ARGS="--bits 128 256 512 1024 --reps 4" bash tools/ab_run.sh gpurun_out/r2_ab_sh0b.jsonl default

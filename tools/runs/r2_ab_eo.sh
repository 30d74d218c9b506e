# even/odd carry-chained product (one IMAD.WIDE.U32.X per limb product): parity first, then leaf A/B
timeout 900 python -m pytest tests/test_gpu_primitives.py tests/test_gpu_gemm.py tests/test_gpu_fullsize_hash.py -x -q -p no:cacheprovider > gpurun_out/r2_eo_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_eo_tests.log
tail -3 gpurun_out/r2_eo_tests.log
AB_ARGS="--bits 256 512 1024 --reps 4" bash tools/ab_run.sh gpurun_out/r2_ab_eo.jsonl default noeo eo_a eo_b

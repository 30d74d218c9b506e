# warp-specialised L=8 leaf: parity first (bounded), then leaf A/B against the one-role kernel
timeout 900 python -m pytest tests/test_gpu_fullsize_hash.py tests/test_gpu_gemm.py tests/test_gpu_lu.py -x -q -p no:cacheprovider > gpurun_out/r2_ws_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_ws_tests.log
tail -3 gpurun_out/r2_ws_tests.log
AB_ARGS="--bits 256 --reps 5" bash tools/ab_run.sh gpurun_out/r2_ab_ws.jsonl default nows wsr2 wsr6
AB_ARGS="--bits 256 --reps 3 --shape 1001,777,1537 --n-min 32" bash tools/ab_run.sh gpurun_out/r2_ab_ws_cfg3.jsonl default nows

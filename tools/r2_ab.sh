set -x
MPGPU_LIB=paper_1410_1599_b200/_variants/spread/libmpgpu.so timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q -m gpu > gpurun_out/spread_tests.log 2>&1
AB_ARGS="--bits 256 512 1024 --reps 5" bash tools/ab_run.sh gpurun_out/ab_r2g.jsonl default spread
tail -1 gpurun_out/spread_tests.log

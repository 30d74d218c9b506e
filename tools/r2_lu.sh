mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lu_host.py tests/test_gpu_dropin.py tests/test_gpu_host_pipe.py -x -q > gpurun_out/lu_host_tests.log 2>&1; echo rc=$? >> gpurun_out/lu_host_tests.log
timeout 900 python bench.py --no-precision-sweep --no-cfg4 --no-configs --no-e2e --no-cpu-baseline > gpurun_out/bench_lu.json 2> gpurun_out/bench_lu.err
tail -3 gpurun_out/lu_host_tests.log

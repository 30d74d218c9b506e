set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_host_pipe.py -x -q > gpurun_out/pipe_tests.log 2>&1; echo rc=$? >> gpurun_out/pipe_tests.log
MPGPU_PIPE_TRACE=1 python tools/pipe_trace.py > gpurun_out/pipe_trace.log 2>&1
python tools/pipe_trace.py --reps 6 >> gpurun_out/pipe_trace.log 2>&1
tail -3 gpurun_out/pipe_tests.log

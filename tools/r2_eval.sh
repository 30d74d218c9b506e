set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_r2s.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_r2s.log 2>&1; echo rc=$? >> gpurun_out/gputests_r2s.log
timeout 900 python bench.py > gpurun_out/bench_r2s.json 2> gpurun_out/bench_r2s.err
tail -3 gpurun_out/gputests_r2s.log

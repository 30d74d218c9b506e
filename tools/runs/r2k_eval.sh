set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_r2k.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_r2k.log 2>&1; echo rc=$? >> gpurun_out/gputests_r2k.log
timeout 900 python bench.py > gpurun_out/bench_r2k.json 2> gpurun_out/bench_r2k.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r2k.json 2> gpurun_out/bench_ref_r2k.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2k.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-precision-sweep --no-lu --no-cfg4 --no-configs --no-e2e > gpurun_out/ncu_launch_r2k.log 2>&1
tail -3 gpurun_out/gputests_r2k.log

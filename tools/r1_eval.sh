set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_r1i.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_r1i.json 2> gpurun_out/bench_r1i.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r1i.json 2> gpurun_out/bench_ref_r1i.err
timeout 1500 python tools/run_configs.py > gpurun_out/configs_r1i.jsonl 2> gpurun_out/configs_r1i.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1i.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_r1i.log 2>&1
tail -2 gpurun_out/bench_r1i.json

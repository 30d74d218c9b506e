set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_r1f.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_r1f.json 2> gpurun_out/bench_r1f.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r1f.json 2> gpurun_out/bench_ref_r1f.err
timeout 1500 python tools/run_configs.py > gpurun_out/configs_r1f.jsonl 2> gpurun_out/configs_r1f.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1f.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_r1f.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_leaf -c 1 -o gpurun_out/prof_leaf_r1f python tools/prof_gemm.py --bits 256 --n 1024 --reps 1 > gpurun_out/ncu_full_r1f.log 2>&1
tail -2 gpurun_out/bench_r1f.json

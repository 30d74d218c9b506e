set -x
python -m pytest tests/test_gpu_fullsize_hash.py -q -p no:cacheprovider > gpurun_out/r2_hash_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_hash_tests.log
python bench.py --steps 20 --warmup 3 > gpurun_out/r2_bench_b.json 2> gpurun_out/r2_bench_b.err
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed
ncu --metrics $M --clock-control none -k regex:"preadd|postadd" --launch-skip 8 -c 8 --csv --log-file gpurun_out/r2_adds_cfg2.csv python tools/prof_gemm.py --n 1024 --bits 256 --n-min 64 > gpurun_out/r2_adds_cfg2.log 2>&1
ncu --metrics $M --clock-control none -k regex:"preadd|postadd" --launch-skip 9 -c 9 --csv --log-file gpurun_out/r2_adds_cfg4.csv python tools/prof_gemm.py --n 4096 --bits 1024 --n-min 512 > gpurun_out/r2_adds_cfg4.log 2>&1
python tools/prof_lu.py --n 2048 --K 64 --kernel winograd --reps 2 > gpurun_out/r2_lu_plain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:lu_panel_perm --launch-skip 40 -c 1 -o gpurun_out/r2_lu_panel python tools/prof_lu.py --n 2048 --K 64 --kernel winograd --reps 2 > gpurun_out/r2_ncu_lu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_lu.csv python tools/prof_lu.py --n 2048 --K 64 --kernel winograd --reps 1 > /dev/null 2>&1
tail -3 gpurun_out/r2_hash_tests.log

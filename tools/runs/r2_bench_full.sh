python tools/ref_cfg4_extrapolate.py > gpurun_out/r2_ref_cfg4_extrapolated.json 2> gpurun_out/r2_ref_cfg4.err &
CPID=$!
python bench.py > gpurun_out/r2_bench_d.json 2> gpurun_out/r2_bench_d.err
echo bench_rc=$?
python bench.py --impl reference > gpurun_out/r2_bench_ref_d.json 2>&1
wait $CPID
echo ref_rc=$?
tail -c 400 gpurun_out/r2_bench_d.err

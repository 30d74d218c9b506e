set -x
AB_ARGS="--bits 256 --reps 5" bash tools/ab_run.sh gpurun_out/ab_r2d.jsonl default tm8tk12 tm8tk10 tm4tk6 tk20m4

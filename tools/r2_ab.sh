set -x
AB_ARGS="--bits 256 512 1024 --reps 5" bash tools/ab_run.sh gpurun_out/ab_r2h.jsonl default xor8 imad16 imad32

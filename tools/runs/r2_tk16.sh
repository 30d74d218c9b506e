timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_fullsize_hash.py tests/test_gpu_lu.py tests/test_gpu_dropin.py tests/test_gpu_shard.py tests/test_gpu_group.py -x -q -p no:cacheprovider 2>&1 | tail -2
for r in 1 2; do for v in default m6; do if [ $v = default ]; then E=""; else E="MPGPU_LIB=paper_1410_1599_b200/_variants/$v/libmpgpu.so"; fi
 env $E timeout 300 python tools/ab_leaf.py --bits 256 --reps 4 --n-min 64 --tag $v-nmin64
 env $E timeout 300 python tools/ab_leaf.py --bits 256 --reps 4 --n-min 32 --tag $v-nmin32
 env $E timeout 300 python tools/prof_lu.py --n 2048 --K 64 --n-min 32 --kernel winograd --reps 3 | tail -1
done; done

#!/bin/bash
# A/B leaf timings of library variants (tools/build_variants.sh) against the default build.
# usage: tools/ab_run.sh OUT.jsonl VARIANT [VARIANT ...]   ("default" = paper_1410_1599_b200/libmpgpu.so)
out=$1; shift
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = default ]; then
      env -u MPGPU_LIB timeout 300 python tools/ab_leaf.py --tag $v $AB_ARGS
    else
      MPGPU_LIB=paper_1410_1599_b200/_variants/$v/libmpgpu.so timeout 300 python tools/ab_leaf.py --tag $v $AB_ARGS
    fi
  done
done > $out 2>&1
grep '^{' $out

#!/bin/bash
# tools/ab_multi.sh CONFIG LIB... : interleaved c2_detail runs over several library builds
cfg=$1; shift
for r in 1 2; do for v in "$@"; do
  echo -n "$v "; FL1_LIB=paper_1812_06635_b200/_build/ab/lib$v.so python tools/c2_detail.py $cfg 2>&1 | grep dev_ms | cut -c1-100
done; done

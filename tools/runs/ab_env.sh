#!/bin/bash
# tools/ab_env.sh VAR "v1 v2" CONFIG... : interleaved c2_detail runs under an env toggle
var=$1; vals=$2; shift 2
for r in 1 2; do for c in "$@"; do for v in $vals; do
  echo -n "$var=$v "; env $var=$v python tools/c2_detail.py $c 2>&1 | grep dev_ms | cut -c1-110
done; done; done

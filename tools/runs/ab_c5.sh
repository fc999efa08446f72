#!/bin/bash
# tools/runs/ab_c5.sh VARIANT... : interleaved c5 bench lines over library builds in _build/ab/lib<V>.so
for r in 1 2; do for v in "$@"; do
  FL1_LIB=paper_1812_06635_b200/_build/ab/lib$v.so timeout 300 python tools/ab_lib.py --config c5 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$v.json 2>> gpurun_out/ab.err
  python -c "import json; d=json.loads(open('gpurun_out/ab_$v.json').read()); print('$v c5', round(d['ms_per_step'],3), 'lockstep ms', round(d['roofline']['launch_ms'],2), d['clocks']['sm_mhz'])"
done; done

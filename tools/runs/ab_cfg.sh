#!/bin/bash
# tools/runs/ab_cfg.sh CONFIG STEPS VARIANT... : interleaved bench lines of one config over library builds
cfg=$1; steps=$2; shift 2
for r in 1 2; do for v in "$@"; do
  FL1_LIB=paper_1812_06635_b200/_build/ab/lib$v.so timeout 600 python tools/ab_lib.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline > gpurun_out/ab_$v.json 2>> gpurun_out/ab.err
  python -c "import json; d=json.loads(open('gpurun_out/ab_$v.json').read()); print('$v $cfg', round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d.get('phase_ms'))"
done; done

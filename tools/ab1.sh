bash tools/ab_env.sh FL1_SERPENTINE "0 1" c2 c1 > gpurun_out/t_serp.log 2>&1
for v in 0 1; do echo -n "c3 serp=$v "; FL1_SERPENTINE=$v python bench.py --config c3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value']*1e3, d.get('phase_ms'))"; done >> gpurun_out/t_serp.log 2>&1
for v in 0 1; do echo -n "c4 serp=$v "; FL1_SERPENTINE=$v python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value']*1e3, d['roofline'].get('frac'))"; done >> gpurun_out/t_serp.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/t_tests.log 2>&1; tail -2 gpurun_out/t_tests.log

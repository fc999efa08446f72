bash tools/ab_env.sh FL1_LD_ALIGN "4 16" c2 c1 > gpurun_out/t_align.log 2>&1
for v in 4 16; do echo -n "c3 align=$v "; FL1_LD_ALIGN=$v python bench.py --config c3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value']*1e3, d.get('phase_ms'))"; done >> gpurun_out/t_align.log 2>&1
FL1_LD_ALIGN=16 python -m pytest tests -m gpu -x -q > gpurun_out/t_tests.log 2>&1; tail -2 gpurun_out/t_tests.log

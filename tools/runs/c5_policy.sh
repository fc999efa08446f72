for v in "2 512" "3 512" "3 256" "3 1024" "3 128" "2 512" "3 512"; do
  set -- $v
  FL1_LOCKSTEP_POLICY=$1 FL1_LOCKSTEP_HANDOFF_S=$2 timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c5p.json 2>> gpurun_out/c5p.err
  python -c "import json; d=json.loads(open('gpurun_out/c5p.json').read()); print('c5 policy=$1 S=$2', round(d['ms_per_step'],3), 'lockstep ms', round(d['roofline']['launch_ms'],2), 'steps', d['roofline']['lockstep_steps'])"
done

for v in "3 512" "0 0" "3 128" "3 64" "3 32" "3 512" "0 0"; do
  set -- $v
  FL1_LOCKSTEP_POLICY=$1 FL1_HANDOFF_S=$2 timeout 300 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/pol.json 2>> gpurun_out/pol.err
  python -c "import json; d=json.loads(open('gpurun_out/pol.json').read()); print('policy $1 S<=$2', round(d['ms_per_step'],3), 'lockstep ms', round(d['roofline']['launch_ms'],2))"
done

for cs in -2 -1 -4 -2 -1; do
  timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --concurrency $cs > gpurun_out/c5_cs.json 2>> gpurun_out/c5_cs.err
  python -c "import json; d=json.loads(open('gpurun_out/c5_cs.json').read()); print('c5 cluster', $cs, round(d['ms_per_step'],3), 'lockstep ms', round(d['roofline']['launch_ms'],2))"
done

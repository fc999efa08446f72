for r in 1 2; do for v in 256 512 768 1024; do
  FL1_HANDOFF_S=$v timeout 300 python bench.py --config c5 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/hs.json 2>> gpurun_out/hs.err
  python -c "import json; d=json.loads(open('gpurun_out/hs.json').read()); print('S<=$v', round(d['ms_per_step'],3), 'lockstep ms', round(d['roofline']['launch_ms'],2))"
done; done

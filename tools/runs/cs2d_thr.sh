for t in 4194304 1048576 2097152 262144 4194304; do
  FL1_COLSPLIT=$t timeout 900 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/cst.json 2> gpurun_out/cst.err
  python -c "import json; d=json.loads(open('gpurun_out/cst.json').read()); print('c4 thr=$t', round(d['ms_per_step'],2), round(d['phase_ms']['D_compact_apply'],1), d['clocks']['sm_mhz'])"
done
for t in 0 1 1048576 4194304 0 1; do
  FL1_COLSPLIT=$t timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cst2.json 2> gpurun_out/cst2.err
  python -c "import json; d=json.loads(open('gpurun_out/cst2.json').read()); print('c2 thr=$t', round(d['ms_per_step'],3), round(d['phase_ms']['D_compact_apply'],3))"
done
for t in 0 1 0 1; do
  FL1_COLSPLIT=$t timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cst3.json 2> gpurun_out/cst3.err
  python -c "import json; d=json.loads(open('gpurun_out/cst3.json').read()); print('c3 thr=$t', round(d['ms_per_step'],3), round(d['phase_ms']['D_compact_apply'],3))"
done

timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "batched" > gpurun_out/c5s_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/c5s_tests.log
for i in 1 2; do
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c5s.json 2>> gpurun_out/c5s.err
python -c "import json; d=json.loads(open('gpurun_out/c5s.json').read()); print('c5 default', round(d['ms_per_step'],3), 'lockstep ms', round(d['roofline']['launch_ms'],2), d['roofline']['frac'])"
done
timeout 1200 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:prefix_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/r02b_c5 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c5b.log 2>&1; echo ncu_rc=$?

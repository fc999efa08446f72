for v in 0 16 32 48 0 24; do
  FL1_SPLIT_BUDGET_MB=$v timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c5s.json 2>> gpurun_out/c5s.err
  python -c "import json; d=json.loads(open('gpurun_out/c5s.json').read()); print('c5 budget=$v MB', round(d['ms_per_step'],3), 'lockstep ms', round(d['roofline']['launch_ms'],2))"
done
for v in 0 32; do
FL1_SPLIT_BUDGET_MB=$v timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:prefix_kernel --launch-skip 3 --launch-count 1 --csv python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -E "dram__bytes|gpu__time" | sed "s/^/budget=$v /"
done

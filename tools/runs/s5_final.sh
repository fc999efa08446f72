# session-5 final: GPU suite (parity records), smoke, the driver's two arms on c4, c1-c3 / c5 lines, c4 launch list and ncu capture
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
FL1_PARITY_OUT=gpurun_out/s5f_parity.json timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s5f_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/s5f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5f_smoke.log 2>&1; echo smoke_rc=$?; cat gpurun_out/s5f_smoke.log
bash tools/runs/driver_like.sh
for c in c1 c2 c3 c5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/s5f_bench_$c.json 2> gpurun_out/s5f_bench_$c.err; echo bench_${c}_rc=$?; python -c "
import json;a=json.loads(open('gpurun_out/s5f_bench_$c.json').read().strip().splitlines()[-1]);print(a['ms_per_step'],a['e2e']['value'],a['roofline']['frac'])"
done
# c4: DRAM bytes of the 10 solve launches of one path (one ncu pass, three metrics)
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off -k regex:engine_kernel --csv --log-file gpurun_out/s5f_ncu_c4_all.csv python tools/c4_lambda.py > gpurun_out/s5f_c4_lambda.json 2> gpurun_out/s5f_c4_lambda.err; echo ncu_c4_rc=$?

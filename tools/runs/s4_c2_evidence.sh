# session 4: c2 evidence -- per-phase timeline, power phase in isolation (sub-phase times + ncu), whole-solve ncu capture
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
FL1_SINGLE_CLUSTER=0 timeout 300 python tools/timeline_c1.py c2 > gpurun_out/s4_timeline_c2.txt 2>&1; echo timeline_rc=$?; tail -3 gpurun_out/s4_timeline_c2.txt
for s in 2876 1500 600; do FL1_UTIL_LOG=1 timeout 300 python tools/c2_power_probe.py $s; done > gpurun_out/s4_power_probe.txt 2>&1; echo probe_rc=$?; cat gpurun_out/s4_power_probe.txt
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:engine_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/s4_c2_power python tools/c2_power_probe.py 2876 > gpurun_out/s4_ncu_power.log 2>&1; echo ncu_power_rc=$?
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:engine_kernel --launch-skip 6 --launch-count 1 -o gpurun_out/s4_c2 python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s4_ncu_c2.log 2>&1; echo ncu_c2_rc=$?
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file gpurun_out/s4_launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s4_ncu_c2_launches.log 2>&1; echo ncu_launches_rc=$?

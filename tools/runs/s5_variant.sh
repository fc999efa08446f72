# two-instance engine build: the fused switch tests, parity probe, c4, and the same-box A/B against the HEAD build
FL1_SINGLE_CLUSTER=0 FL1_FUSED_POWER_MB=1 timeout 300 python tools/probes/fused_power_parity.py > gpurun_out/s5v_parity.txt 2>&1; echo parity_rc=$?; tail -4 gpurun_out/s5v_parity.txt
timeout 900 python -m pytest tests/test_switches_gpu.py -q -x > gpurun_out/s5v_switch.log 2>&1; echo switch_rc=$?; tail -1 gpurun_out/s5v_switch.log
for mb in 0 192; do
  FL1_FUSED_POWER_MB=$mb timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s5v_c4_$mb.json 2>/dev/null; python -c "
import json;a=json.loads(open('gpurun_out/s5v_c4_$mb.json').read().strip().splitlines()[-1]);print('c4', $mb, a['ms_per_step'], a.get('phase_ms'))"
done
bash tools/runs/s5_ab_head.sh 2>&1 | grep -E "^c[0-9]" | cut -c1-60

# L2 prefetch depth of the single-read power pass: parity with the route forced, then c4 A/B over the depth
FL1_SINGLE_CLUSTER=0 FL1_FUSED_POWER_MB=1 timeout 300 python tools/probes/fused_power_parity.py > gpurun_out/s5p_parity.txt 2>&1; echo parity_rc=$?; tail -4 gpurun_out/s5p_parity.txt
for pf in 0 1 2 3; do
  FL1_FUSED_PREFETCH=$pf timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s5p_c4_$pf.json 2>/dev/null; python -c "
import json;a=json.loads(open('gpurun_out/s5p_c4_$pf.json').read().strip().splitlines()[-1]);print('c4 prefetch', $pf, a['ms_per_step'], a.get('phase_ms'))"
done
FL1_FUSED_POWER_MB=0 timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s5p_c4_off.json 2>/dev/null; python -c "
import json;a=json.loads(open('gpurun_out/s5p_c4_off.json').read().strip().splitlines()[-1]);print('c4 two-pass', a['ms_per_step'], a.get('phase_ms'))"

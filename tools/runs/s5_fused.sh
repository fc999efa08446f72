# single-read (fused) power steps: parity on tall dictionaries with the route forced, then c4 A/B
FL1_SINGLE_CLUSTER=0 FL1_FUSED_POWER_MB=1 timeout 300 python tools/probes/fused_power_parity.py > gpurun_out/s5_fused_parity.txt 2>&1; echo parity_rc=$?; tail -5 gpurun_out/s5_fused_parity.txt
for mb in 0 192; do
  FL1_FUSED_POWER_MB=$mb timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s5_fused_c4_$mb.json 2> gpurun_out/s5_fused_c4_$mb.err; echo c4_${mb}_rc=$?
  python -c "
import json;a=json.loads(open('gpurun_out/s5_fused_c4_$mb.json').read().strip().splitlines()[-1]);print($mb, a['ms_per_step'], a['roofline']['frac'], a.get('phase_ms'), a['clocks'])"
done

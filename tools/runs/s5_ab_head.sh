# same-box A/B of the session-5 build against the previous HEAD build (FL1_LIB) on c1-c3 and c5, two rounds
for rnd in 1 2; do for c in ${AB_CONFIGS:-c1 c2 c3 c5}; do for lib in head new; do
  L=paper_1812_06635_b200/libfl1cuda.so; [ $lib = head ] && L=paper_1812_06635_b200/_build/libfl1cuda_head.so
  FL1_LIB=$L timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_$c.json 2>/dev/null
  python -c "
import json;a=json.loads(open('gpurun_out/ab_$c.json').read().strip().splitlines()[-1]);print('$c $lib', round(a['ms_per_step'],4), a.get('phase_ms'))"
done; done; done

# cluster-mode A^T r passes through the bulk ring (FL1_BULK_A) x ring depth (FL1_BULK_STAGES): c1, c5
for r in 1 2; do for v in "0 2" "1 2" "1 4" "1 6"; do
  set -- $v
  for c in c1 c5; do
    FL1_BULK_A=$1 FL1_BULK_STAGES=$2 timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ba.json 2>> gpurun_out/ba.err
    python -c "import json; d=json.loads(open('gpurun_out/ba.json').read()); print('bulk_a=$1 stages=$2 $c', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"
  done
done; done
FL1_BULK_A=1 FL1_BULK_STAGES=4 timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "batched or lockstep or config5 or config1 or c1" > gpurun_out/ba_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/ba_tests.log

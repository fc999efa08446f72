# session 4: GPU suite (with the bounded random sweep) + long randomised GPU-vs-oracle parity sweeps, three seeds
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s4_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/s4_tests.log
for seed in 1 2 3; do
  timeout 900 python tools/fuzz_parity.py 150 $seed > gpurun_out/s4_fuzz_$seed.txt 2>&1; echo fuzz_${seed}_rc=$?; tail -1 gpurun_out/s4_fuzz_$seed.txt
  grep -c "^FAIL" gpurun_out/s4_fuzz_$seed.txt
done

# session 5: randomised GPU-vs-oracle sweeps -- SuKro sequences with ragged factor shapes (new), dense with new seeds
for seed in 11 12; do
  timeout 1200 python tools/fuzz_parity.py 250 $seed sukro > gpurun_out/s5_fuzz_sukro_$seed.txt 2>&1; echo fuzz_sukro_${seed}_rc=$?; tail -1 gpurun_out/s5_fuzz_sukro_$seed.txt
  grep -c "^FAIL" gpurun_out/s5_fuzz_sukro_$seed.txt
done
for seed in 4 5; do
  timeout 1200 python tools/fuzz_parity.py 200 $seed > gpurun_out/s5_fuzz_dense_$seed.txt 2>&1; echo fuzz_dense_${seed}_rc=$?; tail -1 gpurun_out/s5_fuzz_dense_$seed.txt
  grep -c "^FAIL" gpurun_out/s5_fuzz_dense_$seed.txt
done

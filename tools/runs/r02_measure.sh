set -x
nproc; free -g | head -2
FL1_PARITY_MEASURE=1 FL1_PARITY_OUT=gpurun_out/parity_measure.json FL1_C4_PATH_OUT=gpurun_out/c4_path.npz timeout 2400 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/pytest_measure.log 2>&1
echo pytest_rc=$?
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
echo bench_rc=$?

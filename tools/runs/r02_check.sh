# round-2 check: GPU suite (asserting), default bench line (c4), reference arm (c4)
FL1_PARITY_OUT=gpurun_out/parity_r02.json timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_r02.log 2>&1
echo pytest_rc=$?
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo bench_rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo ref_rc=$?

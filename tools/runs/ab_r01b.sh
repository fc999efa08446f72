timeout 900 python -m pytest tests/test_switches_gpu.py -q -x -k "COMPACT or EARLY" > gpurun_out/ab_r01b_tests.log 2>&1; echo tests_rc=$?
bash tools/runs/ab_r01.sh

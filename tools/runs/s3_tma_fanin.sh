timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "batched or lockstep or config5" > gpurun_out/tmaf_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/tmaf_tests.log
for f in 2 4; do
FL1_SK_FANIN=$f timeout 180 python tools/step_log.py > gpurun_out/tmaf_steplog_$f.txt 2>&1; echo fanin=$f rc=$?; tail -8 gpurun_out/tmaf_steplog_$f.txt
done

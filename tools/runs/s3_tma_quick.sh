timeout 180 python tools/step_log.py > gpurun_out/tmaq_steplog.txt 2>&1; echo steplog_rc=$?; tail -9 gpurun_out/tmaq_steplog.txt
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "batched or lockstep or config5" > gpurun_out/tmaq_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/tmaq_tests.log

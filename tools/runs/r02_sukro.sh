timeout 900 python -m pytest tests -m gpu -q -x -k "sukro or sweep or ingestion or harness or kronecker or golden or kats" --durations=8 > gpurun_out/pytest_sukro.log 2>&1
echo pytest_rc=$?
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off -k regex:engine_kernel --csv --log-file gpurun_out/ncu_c4_all.csv python tools/c4_lambda.py > gpurun_out/c4_lambda.json 2> gpurun_out/c4_lambda.err
echo ncu1_rc=$?
timeout 1200 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:engine_kernel -o gpurun_out/r02_c4_l9 python tools/c4_lambda.py --lams 9 > gpurun_out/c4_l9.json 2> gpurun_out/c4_l9.err
echo ncu2_rc=$?

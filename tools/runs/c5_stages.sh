for v in 2 3 2 3; do
  if [ $v = 3 ]; then L=FL1_LIB=paper_1812_06635_b200/_build/libfl1cuda_s3.so; else L=; fi
  env $L timeout 600 python tools/ab_lib.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c5st.json 2>> gpurun_out/c5st.err
  python -c "import json; d=json.loads(open('gpurun_out/c5st.json').read()); print('c5 stages=$v', round(d['ms_per_step'],3), 'lockstep ms', round(d['roofline']['launch_ms'],2))"
done

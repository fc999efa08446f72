set -x
python -m pytest tests -m gpu -x -q > gpurun_out/re_tests.log 2>&1; tail -2 gpurun_out/re_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/re_smoke.log 2>&1; tail -1 gpurun_out/re_smoke.log
for c in c2 c1 c3 c5; do python bench.py --config $c > gpurun_out/re_bench_$c.json 2> gpurun_out/re_bench_$c.err; tail -c 300 gpurun_out/re_bench_$c.json; echo; done
python bench.py --config c4 --steps 2 --warmup 3 > gpurun_out/re_bench_c4.json 2> gpurun_out/re_bench_c4.err; tail -c 200 gpurun_out/re_bench_c4.json; echo
python bench.py --impl reference > gpurun_out/re_bench_ref.json 2> gpurun_out/re_bench_ref.err; tail -c 300 gpurun_out/re_bench_ref.json; echo
python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/re_pre_ncu.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/re_launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/re_ncu_l.log 2>&1; wc -l gpurun_out/re_launches_c2.csv

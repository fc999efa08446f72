# Round-end refresh: GPU tests, smoke, bench lines c1-c5 + reference arm, the default bench's
# launch list, and full ncu captures of the c2 engine launch and the c5 lockstep launch.
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/re_tests.log 2>&1; tail -2 gpurun_out/re_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/re_smoke.log 2>&1; tail -1 gpurun_out/re_smoke.log
for c in c2 c1 c3 c5; do python bench.py --config $c > gpurun_out/re_bench_$c.json 2> gpurun_out/re_bench_$c.err; tail -c 200 gpurun_out/re_bench_$c.json; echo; done
python bench.py --config c4 --steps 2 --warmup 3 > gpurun_out/re_bench_c4.json 2> gpurun_out/re_bench_c4.err; tail -c 200 gpurun_out/re_bench_c4.json; echo
python bench.py --impl reference > gpurun_out/re_bench_ref.json 2> gpurun_out/re_bench_ref.err; tail -c 200 gpurun_out/re_bench_ref.json; echo
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/re_pre_ncu.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/re_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/re_ncu_l.log 2>&1; wc -l gpurun_out/re_launches_c2.csv
ncu --set full --clock-control none --import-source on -k regex:engine_kernel --launch-skip 1 -c 1 -f -o gpurun_out/r01e_c2 python tools/solve_once.py c2 > gpurun_out/re_ncu_c2.log 2>&1; tail -2 gpurun_out/re_ncu_c2.log
ncu --set full --clock-control none --import-source on -k regex:prefix_kernel --launch-skip 3 -c 1 -f -o gpurun_out/r01e_c5 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/re_ncu_c5.log 2>&1; tail -2 gpurun_out/re_ncu_c5.log

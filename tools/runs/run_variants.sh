for v in paper_1812_06635_b200/_build/libfl1cuda_t*.so; do
  FL1_LIB=$v python tools/pass_bench.py 8192 65536 6 2>&1 | tail -1
  FL1_LIB=$v python tools/pass_bench.py 2500 10000 20 2>&1 | tail -1
  FL1_LIB=$v python tools/solve_once.py c2 2>&1 | tail -1
  FL1_LIB=$v python tools/solve_once.py c1 2>&1 | tail -1
done

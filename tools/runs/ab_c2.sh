#!/bin/bash
# A/B two library builds on the c2/c1 solves (interleaved, 3 rounds)
for r in 1 2 3; do for v in A B; do
  echo -n "$v "; FL1_LIB=paper_1812_06635_b200/_build/ab/lib$v.so python tools/c2_detail.py ${1:-c2} 2>&1 | grep dev_ms | cut -c1-120
done; done

#!/bin/bash
# K2a on configs 3/4 (bench_dense.py) for each library build, alternating twice
for rep in 1 2; do
  for lib in "$@"; do
    XE_LIB_LENIENT=1 XE_LIB=$PWD/$lib timeout 600 python scripts/bench_dense.py 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); k=d['k2_eval']; print('$lib', $rep, d['config'], round(k['candidates_per_s']/1e6,1), round(k['roofline']['frac'],4))"
  done
done

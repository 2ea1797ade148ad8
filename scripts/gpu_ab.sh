#!/bin/bash
# A/B timing of two builds of the same sources on one box:
#   lib/ (A) and lib_alt/ (B, XE_LIB), each bench run twice, interleaved.
mkdir -p gpurun_out
ARGS="--steps 10 --warmup 3 --skip-cpu --skip-pdhg --skip-search --skip-e2e ${BENCH_ARGS:-}"
for i in 1 2; do
  timeout 300 python bench.py $ARGS > gpurun_out/ab_A$i.json 2>/dev/null
  XE_LIB=paper_2212_09290_b200/lib_alt/libxengine_b200.so timeout 300 python bench.py $ARGS > gpurun_out/ab_B$i.json 2>/dev/null
done
for f in gpurun_out/ab_*.json; do python -c "import json,sys;d=json.load(open('$f'));print('$f', round(d['value']/1e6,1), 'M/s', round(d['roofline']['kernel_ms'],3), 'ms')"; done > gpurun_out/ab_summary.txt

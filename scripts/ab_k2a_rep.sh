#!/bin/bash
# Interleaved A/B of library builds on the K2a bench workload: each lib twice, alternating.
B="python bench.py --steps 10 --warmup 3 --skip-cpu --skip-pdhg --skip-search --skip-e2e --skip-configs"
for rep in 1 2; do
  for lib in "$@"; do
    XE_LIB_LENIENT=1 XE_LIB=$PWD/$lib timeout 600 $B 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', $rep, round(d['value']/1e6,1), round(d['roofline']['frac'],4), d['clocks'].get('sm_mhz'))"
  done
done

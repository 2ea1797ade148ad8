#!/bin/bash
# A/B of the streaming evaluator plans on the bench workload (VGG-16, 10 M candidates):
# base (8-warp CTAs, byte tables) vs wide (24 / 20-warp CTA per SM, 11-bit tables).
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --skip-cpu --skip-pdhg --skip-search --skip-e2e --skip-configs"
for rep in 1 2; do
  XE_STREAM_WIDE=0 timeout 600 $B > gpurun_out/ab_base_$rep.json 2>/dev/null
  timeout 600 $B > gpurun_out/ab_wide24_$rep.json 2>/dev/null
  XE_LIB_LENIENT=1 XE_LIB=$PWD/paper_2212_09290_b200/lib/libxengine_b200_w20.so timeout 600 $B > gpurun_out/ab_wide20_$rep.json 2>/dev/null
done
for f in gpurun_out/ab_*_[12].json; do python -c "
import json,sys; d=json.loads(open('$f').read()); print('$f', round(d['value']/1e6,1), 'M/s', round(d['roofline']['frac'],4), d['best']['obj_ms'])"; done > gpurun_out/ab_wide.txt
[ -n "$EXTRA" ] && eval "$EXTRA"
echo done

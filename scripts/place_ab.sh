# K2b A/B on config 5 (4M save-all placements per step): lib (A) vs lib_alt (B), twice each
python -m pytest tests/test_place_gpu.py -x -q 2>&1 | tail -2
for i in 1 2; do
  for L in lib lib_alt; do
    XE_LIB=paper_2212_09290_b200/$L/libxengine_b200.so timeout 300 python bench.py --workload random2000 --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L', round(d['value']/1e6,1), 'M placements/s', round(d['roofline']['frac'],4), d['best'])"
  done
done

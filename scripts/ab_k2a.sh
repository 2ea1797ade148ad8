#!/bin/bash
# A/B of two builds of the library on the bench workload (XE_LIB selects the .so),
# then a full ncu capture of the current stream kernel.
mkdir -p gpurun_out
for lib in ${LIBS:-paper_2212_09290_b200/lib/libxengine_b200.so}; do
  tag=$(basename $lib .so)
  XE_LIB_LENIENT=1 XE_LIB=$PWD/$lib timeout 600 python bench.py --steps 10 --warmup 3 --skip-cpu --skip-pdhg --skip-search --skip-e2e \
      > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
done
[ -n "$NCU" ] && timeout 600 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 3 -c 1 \
    -o gpurun_out/k_full -f python bench.py --steps 1 --warmup 3 --n 2000000 --skip-cpu --skip-e2e --skip-pdhg --skip-search \
    > gpurun_out/ncu_full.log 2>&1
[ -n "$EXTRA" ] && eval "$EXTRA"
echo done

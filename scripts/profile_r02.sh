#!/bin/bash
# ncu --set full of the round-2 kernels (one capture each) + launch lists.
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on -f"
timeout 600 $N -k regex:stream_kernel -s 3 -c 1 -o gpurun_out/r02_k2a_vgg python scripts/prof_r02.py eval_vgg > gpurun_out/ncu_k2a_vgg.log 2>&1
timeout 600 $N -k regex:stream_kernel -s 3 -c 1 -o gpurun_out/r02_k2a_resnet python scripts/prof_r02.py eval_resnet > gpurun_out/ncu_k2a_resnet.log 2>&1
timeout 600 $N -k regex:place -s 3 -c 1 -o gpurun_out/r02_k2b python scripts/prof_r02.py place > gpurun_out/ncu_k2b.log 2>&1
timeout 600 $N -k regex:round -s 3 -c 1 -o gpurun_out/r02_k4 python scripts/prof_r02.py round > gpurun_out/ncu_k4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02_launches_exact.csv python scripts/prof_r02.py exact > gpurun_out/ncu_exact.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --n 2000000 --skip-cpu --skip-e2e --skip-pdhg --skip-search --skip-configs > gpurun_out/ncu_bench.log 2>&1
[ -n "$EXTRA" ] && eval "$EXTRA"
echo done

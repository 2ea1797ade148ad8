#!/bin/bash
# ncu --set full of the round-2 kernels after the optimisation passes (one capture each).
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on -f"
timeout 600 $N -k regex:stream_kernel -s 3 -c 1 -o gpurun_out/r02b_k2a_vgg python scripts/prof_r02.py eval_vgg > gpurun_out/ncu_b1.log 2>&1
timeout 600 $N -k regex:stream_kernel -s 3 -c 1 -o gpurun_out/r02b_k2a_resnet python scripts/prof_r02.py eval_resnet > gpurun_out/ncu_b2.log 2>&1
timeout 600 $N -k regex:place_kernel -s 3 -c 1 -o gpurun_out/r02b_k2b python scripts/prof_r02.py place > gpurun_out/ncu_b3.log 2>&1
timeout 600 $N -k regex:round_batch -s 3 -c 1 -o gpurun_out/r02b_k4 python scripts/prof_r02.py round > gpurun_out/ncu_b4.log 2>&1
echo done

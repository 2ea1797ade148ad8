#!/bin/bash
# ncu --set full of the kernels changed late in round 2 (one capture each) + the bench launch list.
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on -f"
timeout 600 $N -k regex:stream_kernel -s 3 -c 1 -o gpurun_out/r02c_k2a_vgg python scripts/prof_r02.py eval_vgg > gpurun_out/ncu_c1.log 2>&1
timeout 600 $N -k regex:stream_kernel -s 3 -c 1 -o gpurun_out/r02c_k2a_resnet python scripts/prof_r02.py eval_resnet > gpurun_out/ncu_c3.log 2>&1
timeout 600 $N -k regex:primal_sell -s 300 -c 1 -o gpurun_out/r02c_k3_primal python scripts/prof_k1k3.py k3r 1024 > gpurun_out/ncu_c4.log 2>&1
timeout 600 $N -k regex:dual_sell -s 300 -c 1 -o gpurun_out/r02c_k3_dual python scripts/prof_k1k3.py k3r 1024 > gpurun_out/ncu_c5.log 2>&1
timeout 600 $N -k regex:write_kernel -s 0 -c 1 -o gpurun_out/r02c_mps python scripts/mps_timing.py > gpurun_out/ncu_c6.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02c_launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --n 2000000 --skip-cpu --skip-e2e --skip-pdhg --skip-search --skip-configs > gpurun_out/ncu_bench.log 2>&1
echo done

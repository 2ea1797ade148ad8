#!/bin/bash
# ncu evidence for profiles/: K2a (bench kernel) full set, K3 PDHG iteration
# kernels, K1 assembly kernels, and the launch list of a bench run.
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:eval_il -s 3 -c 1 -o gpurun_out/k2a_full -f \
    python bench.py --steps 1 --warmup 3 --n 2000000 --skip-cpu --skip-e2e --skip-pdhg > gpurun_out/ncu_k2a.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"primal_kernel|dual_kernel" -s 200 -c 2 -o gpurun_out/k3_full -f \
    python scripts/prof_k1k3.py k3 1024 > gpurun_out/ncu_k3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"row_fill|row_meta|col_kernel" -c 3 -o gpurun_out/k1_full -f \
    python scripts/prof_k1k3.py k1 > gpurun_out/ncu_k1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --n 2000000 --skip-cpu --skip-e2e --skip-pdhg > gpurun_out/ncu_bench.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo done

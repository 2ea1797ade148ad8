#!/bin/bash
# End-of-iteration evidence for profiles/: GPU tests + smoke, the default
# bench line, ncu (--set full) of K2a / K3 / K1 kernels and the launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:eval_il -s 3 -c 1 -o gpurun_out/k2a_full -f \
    python bench.py --steps 1 --warmup 3 --n 2000000 --skip-cpu --skip-e2e --skip-pdhg --skip-search > gpurun_out/ncu_k2a.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"primal_sell|dual_sell" -s 200 -c 2 -o gpurun_out/k3_full -f \
    python scripts/prof_k1k3.py k3 1024 > gpurun_out/ncu_k3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"row_fill|row_meta|col_kernel" -c 3 -o gpurun_out/k1_full -f \
    python scripts/prof_k1k3.py k1 > gpurun_out/ncu_k1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --n 2000000 --skip-cpu --skip-e2e --skip-pdhg --skip-search > gpurun_out/ncu_bench.log 2>&1
echo done

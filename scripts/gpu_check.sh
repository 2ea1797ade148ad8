#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench line, ncu launch list and a
# full ncu capture of the top kernel (regex $KREGEX).  Outputs under gpurun_out/.
set -x
KREGEX=${KREGEX:-eval_il}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
[ -n "$EXTRA" ] && eval "$EXTRA"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --n 2000000 --skip-cpu --skip-e2e --skip-pdhg --skip-search > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s 3 -c 1 -o gpurun_out/k_full -f \
    python bench.py --steps 1 --warmup 3 --n 2000000 --skip-cpu --skip-e2e --skip-pdhg --skip-search > gpurun_out/ncu_full.log 2>&1
echo done

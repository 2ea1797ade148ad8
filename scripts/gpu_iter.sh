#!/bin/bash
# Fast K2a iteration: eval parity tests, a short bench line, one ncu capture.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_eval_gpu.py -q -x > gpurun_out/pytest_eval.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_eval.log
timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu --skip-pdhg --skip-search ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu --skip-pdhg --skip-search --skip-e2e ${BENCH_ARGS:-} > gpurun_out/bench2.json 2>> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-eval_il} -s 3 -c 1 -o gpurun_out/k_full -f \
    python bench.py --steps 1 --warmup 3 --n 2000000 --skip-cpu --skip-e2e --skip-pdhg --skip-search > gpurun_out/ncu_full.log 2>&1
echo done

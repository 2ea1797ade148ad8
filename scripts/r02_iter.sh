#!/bin/bash
# Round-2 iteration: selected GPU tests + a short bench line (+ optional extra commands).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout ${TEST_TIMEOUT:-900} python -m pytest ${TESTS:-tests/test_eval_gpu.py tests/test_eval_property_gpu.py} -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_iter.log
timeout 600 python bench.py --steps 5 --warmup 3 --skip-cpu --skip-pdhg --skip-search ${BENCH_ARGS:-} > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err
[ -n "$EXTRA" ] && eval "$EXTRA"
echo done

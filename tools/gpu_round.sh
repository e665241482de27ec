#!/usr/bin/env bash
# One GPU pass (run under gpurun from the repo root): the GPU parity suite, the headline
# bench line, and the secondary rows; logs land in gpurun_out/.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout=900 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
tail -1 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 900 python bench.py --rows --no-cpu > gpurun_out/bench_rows.log 2>&1; tail -1 gpurun_out/bench_rows.log | cut -c1-200

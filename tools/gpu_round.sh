timeout 1200 python -m pytest tests -m gpu -q --timeout=300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -5 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 --rows > gpurun_out/bench_rows.log 2>&1; tail -1 gpurun_out/bench_rows.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log

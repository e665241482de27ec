mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_full.log
tail -4 gpurun_out/pytest_full.log
timeout 900 python bench.py --steps 5 --warmup 3 --rows --no-cpu > gpurun_out/bench_rows_new.log 2>&1
tail -c 3000 gpurun_out/bench_rows_new.log

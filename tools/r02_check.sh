mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --rows > gpurun_out/bench_rows2.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --strong --no-cpu > gpurun_out/bench_strong.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --kind 1 --no-cpu > gpurun_out/bench_rq.log 2>&1
tail -3 gpurun_out/pytest.log

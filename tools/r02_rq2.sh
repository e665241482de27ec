mkdir -p gpurun_out
KIND=1 timeout 300 python tests/tools/variant_check.py > gpurun_out/rq2.log 2>&1
KIND=0 timeout 300 python tests/tools/variant_check.py >> gpurun_out/rq2.log 2>&1
timeout 900 python tests/tools/parity_report.py gpurun_out/parity_rq2.json --only cfg1,cfg2,headline,cfg5 > gpurun_out/parity_rq2.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --kind 1 --no-cpu > gpurun_out/bench_rq2.log 2>&1
cat gpurun_out/rq2.log; tail -3 gpurun_out/pytest.log

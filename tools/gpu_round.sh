timeout 1200 python -m pytest tests -m gpu -q --timeout=300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 10 --warmup 3 --rows > gpurun_out/bench_rows.log 2>&1; tail -1 gpurun_out/bench_rows.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['e2e']['value']); print(json.dumps({k: d['rows'][k] for k in ['cfg3_train','cfg3_train_lazy','table1_query_sizes']}))"

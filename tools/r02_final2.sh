# round-2 measurement pass after the K3 rewrite (run under gpurun from the repo root)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_headline.log 2>&1
timeout 1200 python bench.py --rows --no-cpu > gpurun_out/bench_rows.log 2>&1
timeout 900 python tests/tools/parity_report.py gpurun_out/parity_gram.json --only gram > gpurun_out/parity_gram.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gram2 -s 1 -c 1 -o gpurun_out/gram2_cfg5 -f \
  python tools/gram_time.py > gpurun_out/ncu_gram5.log 2>&1
python tools/ncu_summary.py gpurun_out/gram2_cfg5.ncu-rep gpurun_out/gram2_cfg5_ncu_full.txt > /dev/null 2>&1
tail -2 gpurun_out/pytest_final.log; tail -2 gpurun_out/smoke.log; tail -c 600 gpurun_out/bench_headline.log

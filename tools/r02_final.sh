# round-2 measurement pass (run under gpurun from the repo root)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_headline.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1
timeout 1200 python bench.py --rows --no-cpu > gpurun_out/bench_rows.log 2>&1
timeout 600 python bench.py --kind 1 --no-cpu > gpurun_out/bench_rq.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 3 -c 1 \
  -o gpurun_out/score_headline -f python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_score.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 6 -c 2 \
  -o gpurun_out/score_headline_rq -f python bench.py --steps 2 --warmup 3 --no-cpu --kind 1 > gpurun_out/ncu_score_rq.log 2>&1
timeout 1500 python tests/tools/parity_report.py gpurun_out/parity.json > gpurun_out/parity.log 2>&1
tail -2 gpurun_out/pytest_final.log; tail -2 gpurun_out/smoke.log
# keep what comes back under gpurun's 64 MiB: summaries instead of the reports
for r in score_headline score_headline_rq; do
  python tools/ncu_summary.py gpurun_out/$r.ncu-rep gpurun_out/${r}_ncu_full.txt > /dev/null 2>&1
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  rm -f gpurun_out/$r.ncu-rep
done
ls -la gpurun_out

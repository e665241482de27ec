# round-2 closing measurement pass (run under gpurun from the repo root): tests, smoke, bench
# lines, launch list, ncu of the training kernel after the K5 change, parity report
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_headline.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1
timeout 1200 python bench.py --rows --no-cpu > gpurun_out/bench_rows.log 2>&1
timeout 600 python bench.py --kind 1 --no-cpu > gpurun_out/bench_rq.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:train_kernel -s 1 -c 1 \
  -o gpurun_out/train_cfg3 -f python tools/train_sweep.py 5 > gpurun_out/ncu_train.log 2>&1
python tools/ncu_summary.py gpurun_out/train_cfg3.ncu-rep gpurun_out/train_cfg3_ncu_full.txt > /dev/null 2>&1
rm -f gpurun_out/train_cfg3.ncu-rep gpurun_out/fast_pass1.ncu-rep
timeout 1500 python tests/tools/parity_report.py gpurun_out/parity.json > gpurun_out/parity.log 2>&1
tail -2 gpurun_out/pytest_final.log; tail -2 gpurun_out/smoke.log; tail -c 400 gpurun_out/bench_headline.log

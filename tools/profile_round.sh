# Refresh the committed measurements (run under gpurun from the repo root; logs and
# reports land in gpurun_out/, summaries are copied into profiles/ afterwards with
# tools/ncu_summary.py). PROFILE_SCORE=1 also captures the headline score launch.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_headline.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1
timeout 1200 python bench.py --rows --no-cpu > gpurun_out/bench_rows.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
if [ "${PROFILE_SCORE:-0}" = 1 ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 3 -c 1 \
    -o gpurun_out/score_headline -f python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_score.log 2>&1
fi
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fk_kernel -s 5 -c 1 \
  -o gpurun_out/fk_m8 -f python tools/fk_time.py > gpurun_out/ncu_fk.log 2>&1

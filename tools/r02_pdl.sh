mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
for r in 1 2; do
  ONEQ=16384 SPLITS=0 timeout 300 python tools/cfg1_sweep.py >> gpurun_out/pdl_cfg1.log 2>&1
  FASTRON_PDL=0 ONEQ=16384 SPLITS=0 timeout 300 python tools/cfg1_sweep.py | sed 's/^/nopdl /' >> gpurun_out/pdl_cfg1.log 2>&1
done
timeout 900 python bench.py --steps 5 --warmup 3 --rows --no-cpu > gpurun_out/bench_pdl.log 2>&1
FASTRON_PDL=0 timeout 900 python bench.py --steps 5 --warmup 3 --rows --no-cpu > gpurun_out/bench_nopdl.log 2>&1
tail -3 gpurun_out/pytest.log; cat gpurun_out/pdl_cfg1.log

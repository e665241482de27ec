mkdir -p gpurun_out
for r in 1 2; do
  for v in default nopf; do
    if [ "$v" = default ]; then L=""; else L="FASTRON_LIB=build/variants/lib_$v.so"; fi
    env $L TRAIN_N=5000 timeout 300 python tools/train_sweep.py 5 3 8 | sed "s/^/$v /" >> gpurun_out/train_ab.log 2>&1
    env $L TRAIN_N=8446 timeout 300 python tools/train_sweep.py 9 | sed "s/^/$v /" >> gpurun_out/train_ab.log 2>&1
  done
done
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 900 python bench.py --rows > gpurun_out/bench_rows.log 2>&1
tail -5 gpurun_out/pytest.log

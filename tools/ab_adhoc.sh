mkdir -p gpurun_out
for r in 1 2; do
for v in default nostage; do if [ $v = default ]; then L=; else L=FASTRON_LIB=build/variants/lib_$v.so; fi
  env $L timeout 300 python tools/gram_time.py >> gpurun_out/ab_gram.log 2>&1
done; done
timeout 900 python -m pytest tests -m gpu -x -q -k "gram or lazy or joint or fuzz or update or smoke" > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log

mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
for r in 1 2; do
for v in default old; do if [ $v = default ]; then L=; else L=FASTRON_LIB=build/variants/lib_$v.so; fi
  env $L timeout 300 python tools/edge_time.py >> gpurun_out/ab_edge.log 2>&1
  env $L KIND=1 timeout 300 python tools/score_time.py >> gpurun_out/ab_score.log 2>&1
  env $L WL=cfg2 timeout 300 python tools/score_time.py >> gpurun_out/ab_score.log 2>&1
done; done

mkdir -p gpurun_out
timeout 600 python tools/query_probe.py > gpurun_out/query_probe.log 2>&1
FASTRON_QUERY_FUSED=0 timeout 600 python tools/query_probe.py >> gpurun_out/query_probe.log 2>&1
for v in ${VARIANTS:-}; do
  if [ "$v" = default ]; then KIND=1 timeout 300 python tests/tools/variant_check.py >> gpurun_out/rq_ab.log 2>&1
  else FASTRON_LIB=build/variants/lib_$v.so KIND=1 timeout 300 python tests/tools/variant_check.py >> gpurun_out/rq_ab.log 2>&1; fi
done
timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
tail -5 gpurun_out/pytest.log

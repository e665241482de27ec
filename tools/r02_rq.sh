# RQ accuracy A/B (run under gpurun from the repo root): error stats + headline time per
# library variant (VARIANTS), then the GPU test suite.
mkdir -p gpurun_out
for v in ${VARIANTS:-default}; do
  if [ "$v" = default ]; then KIND=1 timeout 300 python tests/tools/variant_check.py >> gpurun_out/rq_ab.log 2>&1
  else FASTRON_LIB=build/variants/lib_$v.so KIND=1 timeout 300 python tests/tools/variant_check.py >> gpurun_out/rq_ab.log 2>&1; fi
done
KIND=0 timeout 300 python tests/tools/variant_check.py >> gpurun_out/rq_ab.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf -s > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
tail -3 gpurun_out/pytest.log

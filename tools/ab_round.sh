# A/B round (run under gpurun from the repo root): alternating variants, logs in gpurun_out/
mkdir -p gpurun_out
run() {  # run <log> <variant> <cmd...>
  local log=$1 v=$2; shift 2
  if [ "$v" = default ]; then timeout 300 "$@" >> gpurun_out/$log 2>&1
  else FASTRON_LIB=build/variants/lib_$v.so timeout 300 "$@" >> gpurun_out/$log 2>&1; fi
}
for r in 1 2; do
  for v in ${SCORE_VARIANTS:-}; do NO_ORACLE=1 run ab_score.log $v python tests/tools/variant_check.py; done
  for v in ${FK_VARIANTS:-}; do run ab_fk.log $v python tools/fk_time.py; done
  for v in ${GRAM_VARIANTS:-}; do run ab_gram.log $v python tools/gram_time.py; done
done

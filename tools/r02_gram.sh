mkdir -p gpurun_out
for r in 1 2 3; do
  for v in ${VARIANTS:-default}; do
    if [ "$v" = default ]; then timeout 300 python tools/gram_time.py >> gpurun_out/gram_ab.log 2>&1
    else FASTRON_LIB=build/variants/lib_$v.so timeout 300 python tools/gram_time.py >> gpurun_out/gram_ab.log 2>&1; fi
  done
done
cat gpurun_out/gram_ab.log

mkdir -p gpurun_out
for r in 1 2; do
for v in default g16c3 g8c3; do if [ $v = default ]; then L=; else L=FASTRON_LIB=build/variants/lib_$v.so; fi
  env $L timeout 300 python tools/gram_time.py >> gpurun_out/ab_gram.log 2>&1
done; done

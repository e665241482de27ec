# Gram probe: N sweep at M = 8, then an ncu --set full capture (with source) of the cfg3 Gram
mkdir -p gpurun_out
python tools/gram_sweep.py > gpurun_out/gram_sweep.log 2>&1
FASTRON_GRAM_T=1 NS=20000 python tools/gram_sweep.py >> gpurun_out/gram_sweep.log 2>&1
python tools/gram_time.py >> gpurun_out/gram_sweep.log 2>&1
cat gpurun_out/gram_sweep.log
NS=5000 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gram_kernel -s 1 -c 1 \
  -o gpurun_out/gram_cfg3_src -f python tools/gram_sweep.py > gpurun_out/gram_ncu.log 2>&1
tail -3 gpurun_out/gram_ncu.log

mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gram_train.py tests/test_gpu_joint.py -q -x -rf > gpurun_out/ab11.log 2>&1; echo "rc=$?" >> gpurun_out/ab11.log
for r in 1 2 3; do python tools/gram_time.py >> gpurun_out/ab11.log 2>&1; FASTRON_LIB=build/variants/lib_gprev.so python tools/gram_time.py >> gpurun_out/ab11.log 2>&1; done
NS=2560,5000,7680,10240 python tools/gram_sweep.py >> gpurun_out/ab11.log 2>&1
FASTRON_GRAM_UH=64 NS=2560,5000,7680,10240 python tools/gram_sweep.py >> gpurun_out/ab11.log 2>&1
tail -16 gpurun_out/ab11.log

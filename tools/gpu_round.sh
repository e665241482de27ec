for n in 512 5000; do TRAIN_N=$n FASTRON_LIB=build/variants/lib_trprof.so timeout 300 python tools/train_sweep.py 1 2>&1 | grep -E "prof" | head -1; done
timeout 900 python -m pytest tests/test_gpu_gram_train.py tests/test_gpu_lazy.py tests/test_gpu_update.py -q --timeout=300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
TRAIN_N=5000 timeout 300 python tools/train_sweep.py 1 2 4 2>&1 | tail -3

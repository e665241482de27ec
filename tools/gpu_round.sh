timeout 900 python -m pytest tests/test_gpu_lazy.py tests/test_gpu_gram_train.py -q --timeout=300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -25 gpurun_out/gpu_tests.log

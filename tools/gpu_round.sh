timeout 900 python -m pytest tests/test_gpu_gram_train.py -q --timeout=300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 600 python tools/train_sweep.py 1 2 4 8 16

timeout 900 python -m pytest tests/test_gpu_update.py tests/test_gpu_score.py -q --timeout=300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -30 gpurun_out/gpu_tests.log

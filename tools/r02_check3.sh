mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gram_train.py tests/test_gpu_joint.py tests/test_gpu_lazy.py tests/test_gpu_fuzz.py tests/test_gpu_update.py -q -x -rf > gpurun_out/check3.log 2>&1; echo "rc=$?" >> gpurun_out/check3.log
python tools/gram_time.py >> gpurun_out/check3.log 2>&1
tail -4 gpurun_out/check3.log

mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gram_train.py tests/test_gpu_joint.py -q -x -rf > gpurun_out/check4.log 2>&1; echo "rc=$?" >> gpurun_out/check4.log
for r in 1 2; do python tools/gram_time.py >> gpurun_out/check4.log 2>&1; FASTRON_LIB=build/variants/lib_gprev.so python tools/gram_time.py >> gpurun_out/check4.log 2>&1; done
tail -14 gpurun_out/check4.log

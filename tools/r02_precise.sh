mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_precise.py tests/test_gpu_model.py tests/test_gpu_edge.py -m gpu -q -rf -s > gpurun_out/pytest_precise.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_precise.log
timeout 1500 python tests/tools/parity_report.py gpurun_out/parity.json > gpurun_out/parity.log 2>&1
tail -3 gpurun_out/pytest_precise.log

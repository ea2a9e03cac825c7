mkdir -p gpurun_out/ds
timeout 600 python -m pytest tests/test_gpu_serving.py -q --timeout 300 --timeout-method thread 2>&1 | tail -15 > gpurun_out/ds/serving.log
cat gpurun_out/ds/serving.log

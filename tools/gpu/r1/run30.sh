timeout 900 python -m pytest tests/test_gpu_serving.py -q --timeout 600 --timeout-method thread 2>&1 | tail -25

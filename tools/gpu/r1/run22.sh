mkdir -p gpurun_out/ds
timeout 600 python -m pytest tests/test_gpu_serving.py -q --timeout 300 --timeout-method thread 2>&1 | tail -15 > gpurun_out/ds/serving2.log
timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 --timeout-method thread 2>&1 | tail -4 > gpurun_out/ds/pytest.log
timeout 120 python tools/probe_phase.py --log2n 26 --k 1024 > gpurun_out/ds/q26.log 2>&1
cat gpurun_out/ds/serving2.log gpurun_out/ds/pytest.log gpurun_out/ds/q26.log

timeout 600 python -m pytest tests/test_gpu_serving.py -q --timeout 300 --timeout-method thread 2>&1 | tail -2
timeout 120 python tools/probe_phase.py --log2n 26 --k 1024 --variant td 2>&1 | tail -1
timeout 120 python tools/probe_phase.py --log2n 26 --k 1024 2>&1 | tail -1
timeout 400 python tools/probe_mixed.py 2>&1 | tail -4

mkdir -p gpurun_out/ds
timeout 600 python -m pytest tests/test_gpu_serving.py -q --timeout 300 --timeout-method thread 2>&1 | tail -15 > gpurun_out/ds/serving3.log
cat gpurun_out/ds/serving3.log
timeout 600 python tools/stress_serving.py --runs 300 --seed 4 > gpurun_out/ds/stress4.log 2>&1; tail -1 gpurun_out/ds/stress4.log; grep FAIL gpurun_out/ds/stress4.log | head -5
timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 --timeout-method thread 2>&1 | tail -4
timeout 120 python tools/probe_phase.py --log2n 26 --k 1024 --variant td 2>&1 | tail -1
timeout 120 python tools/probe_phase.py --log2n 26 --k 1024 2>&1 | tail -1
timeout 400 python tools/probe_mixed.py 2>&1 | tail -4

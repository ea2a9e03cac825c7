# full GPU suite (incl. slow) + bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 --timeout-method thread 2>&1 | tail -8 > gpurun_out/pytest_gpu_all.log
timeout 600 python bench.py > gpurun_out/bench5.json 2> gpurun_out/bench5.err
cat gpurun_out/pytest_gpu_all.log gpurun_out/bench5.json
